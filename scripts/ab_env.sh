#!/bin/bash
# one short bench line with extra environment (A/B of runtime switches)
# usage: scripts/ab_env.sh OUT WORKLOAD LABEL VAR=VALUE...
out=$1; wl=$2; label=$3; shift 3
env "$@" timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | \
  python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', '$wl', round(d['ms_per_step'],3), '%.3g' % d['value'], round(d['roofline']['frac'],4), [round(v,3) for v in d['roofline']['stage_ms_per_step']], d['parity']['rel_l2'] if d.get('parity') else None)" >> $out 2>&1
