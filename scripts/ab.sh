#!/bin/bash
# A/B of library variants on the GPU box: one short bench line per variant
# usage: scripts/ab.sh OUT WORKLOAD variant...   (variant = NAME for exp/libvpfv_NAME.so, or "main")
out=$1; wl=$2; shift 2
for v in "$@"; do
  if [ "$v" = main ]; then lib=""; else lib="VPFV_LIB=exp/libvpfv_$v.so"; fi
  env $lib timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$wl', round(d['ms_per_step'],3), '%.3g' % d['value'], round(d['roofline']['frac'],4), [round(v,3) for v in d['roofline']['stage_ms_per_step']])" >> $out 2>&1
done
