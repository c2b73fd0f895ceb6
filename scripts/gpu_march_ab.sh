mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "march or 1d1v or fused_field or twostream or two_stream or landau" > gpurun_out/t2.log 2>&1; echo "rc=$?" >> gpurun_out/t2.log
rm -f gpurun_out/ab2.txt
for wl in twostream-1024 landau1d-128; do for m in 0 1; do
VPFV_1D1V_MARCH=$m timeout 300 python bench.py --workload $wl --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('march=$m', '$wl', round(d['ms_per_step'],4), '%.3g' % d['value'], round(d['roofline']['frac'],4), [round(x,4) for x in d['roofline']['stage_ms_per_step']])" >> gpurun_out/ab2.txt 2>&1
done; done
