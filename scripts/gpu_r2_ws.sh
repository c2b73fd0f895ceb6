# WS-variant check: parity tests with VPFV_RB_WS=1, then the stage A/B
mkdir -p gpurun_out
VPFV_RB_WS=1 timeout 900 python -m pytest tests/test_gpu.py -x -q -k "tiled or landau2d or graph_replay or medium_step or vx_sign or nonfinite or aliasing or ep2d2v or range" > gpurun_out/ws_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ws_tests.log
bash scripts/gpu_r2_ab.sh
