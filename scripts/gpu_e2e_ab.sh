# HostPipeline copy paths: parity tests, then an interleaved e2e A/B at the headline and 1D-2V workloads.
mkdir -p gpurun_out/e2e
timeout 900 python -m pytest tests/test_gpu.py -x -q -m gpu -k "host_pipeline or box or cluster" > gpurun_out/e2e/tests.log 2>&1; echo "rc=$?" >> gpurun_out/e2e/tests.log
timeout 900 python scripts/probes/e2e_ab.py landau2d-128 32 3 > gpurun_out/e2e/ab_128.json 2> gpurun_out/e2e/ab_128.err
timeout 600 python scripts/probes/e2e_ab.py weibel-256 64 3 > gpurun_out/e2e/ab_weibel.json 2> gpurun_out/e2e/ab_weibel.err
