# Full ncu capture (with source) of one RK4 step of the headline stage kernel.
mkdir -p gpurun_out/r2prof
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:stage2d2v_rb -s 4 -c 4 -o gpurun_out/r2prof/rb python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2prof/ncu.log 2>&1
ls -la gpurun_out/r2prof
