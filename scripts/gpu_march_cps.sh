# march kernel: tests, then ncu launch durations at several CTAs-per-SM targets (twostream-1024)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "march or 1d1v or fused_field" > gpurun_out/t2.log 2>&1; echo "rc=$?" >> gpurun_out/t2.log
for c in 3 4 5 6 8; do
VPFV_1D1V_MARCH=1 VPFV_1D1V_CPS=$c timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:stage_1d1v -c 30 --csv --log-file gpurun_out/cps_$c.csv python bench.py --workload twostream-1024 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done
