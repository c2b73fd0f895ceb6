# End-of-round-2 measurement: gpu tests, smoke, default bench (both arms),
# the other workloads, launch list and a full capture of the headline kernel.
mkdir -p gpurun_out/fin
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fin/tests.log 2>&1; echo "rc=$?" >> gpurun_out/fin/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/fin/bench.json 2> gpurun_out/fin/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/fin/bench_ref.json 2> gpurun_out/fin/bench_ref.err
for wl in landau1d-128 twostream-1024 weibel-256 ep2d2v-64; do
  timeout 600 python bench.py --workload $wl --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/fin/bench_$wl.json 2> gpurun_out/fin/bench_$wl.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:stage2d2v_rb -s 4 -c 4 -o gpurun_out/fin/rb python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/fin/ncu.log 2>&1
ls -la gpurun_out/fin
