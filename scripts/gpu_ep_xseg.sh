# config 5 (2 x 64^4, species launched concurrently): x segments per column block
mkdir -p gpurun_out
: > gpurun_out/ep_xseg.txt
for rep in 1 2; do for xs in 0 1 2 3; do
  VPFV_XSEG=$xs timeout 300 python bench.py --workload ep2d2v-64 --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('xseg=$xs', round(d['ms_per_step'],4), round(sum(r['stage_ms_per_step']),4), round(r['frac'],4))" >> gpurun_out/ep_xseg.txt
done; done
