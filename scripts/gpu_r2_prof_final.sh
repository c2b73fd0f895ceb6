# End-of-round-2 profiles: full capture of one RK4 step of the headline kernel,
# launch lists of the default bench and the other workloads, the 1D-2V kernel.
mkdir -p gpurun_out/r2f
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:stage2d2v_rb -s 4 -c 4 -o gpurun_out/r2f/rb python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2f/ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"stage1d2v_rb|moment_partials_row" -s 8 -c 2 -o gpurun_out/r2f/wb python bench.py --workload weibel-256 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
for wl in landau1d-128 twostream-1024 weibel-256 ep2d2v-64; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r2f/launches_$wl.csv python bench.py --workload $wl --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done
ls -la gpurun_out/r2f
