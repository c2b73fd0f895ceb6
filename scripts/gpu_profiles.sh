# End-of-round profiles: full captures of the headline stage kernel (one RK4
# step = 4 launches) and the 1D kernels, launch lists of every workload.
mkdir -p gpurun_out/prof
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:stage2d2v_rb -s 4 -c 4 -o gpurun_out/prof/rb python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"field1d_conv|stage_1d1v_march" -s 8 -c 2 -o gpurun_out/prof/ts python bench.py --workload twostream-1024 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"stage1d2v_rb|moment_partials_row" -s 8 -c 2 -o gpurun_out/prof/wb python bench.py --workload weibel-256 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
for wl in landau2d-128 landau1d-128 twostream-1024 weibel-256 ep2d2v-64; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/prof/launches_$wl.csv python bench.py --workload $wl --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done
ls -la gpurun_out/prof
