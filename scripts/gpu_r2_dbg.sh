# Debug: one tiled 2D-2V stage launch under compute-sanitizer
mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool memcheck --show-backtrace device python -m pytest tests/test_gpu.py -x -q -k "test_tiled_stage_vs_oracle" > gpurun_out/dbg.log 2>&1; echo "rc=$?" >> gpurun_out/dbg.log
