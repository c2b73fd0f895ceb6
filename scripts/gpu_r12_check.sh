# 1D-2V geometry check: parity tests under each VPFV_R12_CFG, then the workload A/B
mkdir -p gpurun_out
: > gpurun_out/r12_tests.log
for cfg in 1 3 4; do
  VPFV_R12_CFG=$cfg timeout 600 python -m pytest tests/test_gpu.py tests/test_gpu_benchsize.py -x -q -k "1d2v or weibel or tiled12" >> gpurun_out/r12_tests.log 2>&1; echo "cfg=$cfg rc=$?" >> gpurun_out/r12_tests.log
done
bash scripts/gpu_wl_ab.sh weibel-256
