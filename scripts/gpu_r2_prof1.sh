# ncu source-level capture of one stage-1 launch of the headline kernel (quick look)
mkdir -p gpurun_out/r2prof
timeout 600 ncu --set full --import-source on --clock-control none -k regex:stage2d2v_rb -s 4 -c 1 -o gpurun_out/r2prof/${1:-cur} python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2prof/ncu_${1:-cur}.log 2>&1
