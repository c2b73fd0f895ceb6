# Round-2 measurement refresh: default bench line (both arms), launch list of
# the default bench, a full ncu capture of one RK4 step of the headline
# stage kernel (4 launches, with source), and the other workloads' bench lines.
mkdir -p gpurun_out/r2m
timeout 900 python bench.py > gpurun_out/r2m/bench.json 2> gpurun_out/r2m/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2m/bench_ref.json 2> gpurun_out/r2m/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2m/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:stage2d2v_rb -s 4 -c 4 -o gpurun_out/r2m/rb python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2m/ncu.log 2>&1
for wl in landau1d-128 twostream-1024 weibel-256 ep2d2v-64; do
  timeout 600 python bench.py --workload $wl --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2m/bench_$wl.json 2> gpurun_out/r2m/bench_$wl.err
done
ls -la gpurun_out/r2m
