# Programmatic launches through the 2D field chain and into the 2D-2V stage
# kernel: full -m gpu suite, then VPFV_PDL=0/1 interleaved on the chain probe
# and the 2D bench workloads.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pdl2d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pdl2d_tests.log
: > gpurun_out/pdl2d_ab.txt
for rep in 1 2 3; do for pdl in 0 1; do
  echo "pdl=$pdl $(VPFV_PDL=$pdl timeout 300 python scripts/probes/chain_probe.py 128 2>&1 | tail -1)" >> gpurun_out/pdl2d_ab.txt
  echo "pdl=$pdl $(VPFV_PDL=$pdl timeout 300 python scripts/probes/chain_probe.py 64 2>&1 | tail -1)" >> gpurun_out/pdl2d_ab.txt
  for wl in landau2d-128 ep2d2v-64; do
    VPFV_PDL=$pdl timeout 300 python bench.py --workload $wl --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$pdl $wl', round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4), d['clocks']['sm_mhz'])" >> gpurun_out/pdl2d_ab.txt
  done
done; done
