# Quick state check on one GPU: gpu tests, smoke, default bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g1_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g1_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g1_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err
