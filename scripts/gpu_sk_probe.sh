# Stream-K diagnosis: single-species 64^4 with and without it; config 5 with forced CTA counts.
mkdir -p gpurun_out
: > gpurun_out/sk_probe.txt
for rep in 1 2; do for sk in 0 1 148; do
  VPFV_RB_SK=$sk timeout 300 python scripts/probes/sk_probe.py 64 >> gpurun_out/sk_probe.txt 2>&1
done; done
for sk in 0 148 74 37; do
  VPFV_RB_SK=$sk timeout 300 python bench.py --workload ep2d2v-64 --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('ep sk=$sk', round(d['ms_per_step'],4), [round(x,4) for x in r['stage_ms_per_step']])" >> gpurun_out/sk_probe.txt
done
