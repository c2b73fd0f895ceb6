# Interleaved stage-time A/B of exp/libvpfv_*.so builds against the in-tree library (no tests).
mkdir -p gpurun_out
libs="main"
for f in exp/libvpfv_*.so; do libs="$libs $f"; done
: > gpurun_out/ab_stage.txt
for rep in 1 2 3; do timeout 600 python scripts/stage_ab.py --reps 20 $libs >> gpurun_out/ab_stage.txt 2>&1; done
