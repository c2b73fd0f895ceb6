# ncu capture of the 1D-2V stage kernel (default geometry) + moment finish, and the weibel launch list
mkdir -p gpurun_out/r2f
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"stage1d2v_rb|moment_partials_row" -s 8 -c 2 -o gpurun_out/r2f/wb python bench.py --workload weibel-256 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r2f/launches_weibel-256.csv python bench.py --workload weibel-256 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
