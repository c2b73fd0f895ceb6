# ncu source-level capture of the 1D-2V stage kernel (weibel-256, stages 1-4 of one step)
mkdir -p gpurun_out/r2prof
timeout 600 ncu --set full --import-source on --clock-control none -k regex:stage1d2v_rb -s 8 -c 4 -o gpurun_out/r2prof/w12 python bench.py --workload weibel-256 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2prof/ncu_w12.log 2>&1
