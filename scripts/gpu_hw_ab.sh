# Halved upwind chains (VPFV_HALF_W): targeted 2D-2V parity tests on the
# in-tree build, stage-time A/B against exp/ builds, then the host-link probe.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "tiled or landau2d or graph_replay or medium_step or vx_sign or nonfinite or aliasing or ep2d2v or peer or range or manufactured or linear" > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
libs="main"
for f in exp/libvpfv_*.so; do libs="$libs $f"; done
: > gpurun_out/ab_stage.txt
for rep in 1 2 3; do timeout 600 python scripts/stage_ab.py --reps 20 $libs >> gpurun_out/ab_stage.txt 2>&1; done
timeout 300 python scripts/probes/pcie_bw.py > gpurun_out/pcie_bw.txt 2>&1
