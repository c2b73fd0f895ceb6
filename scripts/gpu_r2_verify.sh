# After host-side changes: full -m gpu suite, smoke, default bench line.
mkdir -p gpurun_out/ver
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ver/tests.log 2>&1; echo "rc=$?" >> gpurun_out/ver/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/ver/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/ver/bench.json 2> gpurun_out/ver/bench.err
