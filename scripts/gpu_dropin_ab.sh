# Drop-in host staging sweep + its parity tests.
mkdir -p gpurun_out/dropin
timeout 900 python -m pytest tests -x -q -m gpu -k "dropin or drop_in or host" > gpurun_out/dropin/tests.log 2>&1; echo "rc=$?" >> gpurun_out/dropin/tests.log
timeout 1200 python scripts/probes/dropin_ab.py landau2d-128 2 > gpurun_out/dropin/ab.json 2> gpurun_out/dropin/ab.err
nproc > gpurun_out/dropin/nproc.txt; lscpu | head -20 >> gpurun_out/dropin/nproc.txt
