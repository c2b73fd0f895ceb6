#!/bin/bash
# quick A/B on the GPU box: tiled-kernel tests + short bench lines
# usage: scripts/quickperf.sh OUT "ENV=.. ENV2=.." [workloads...]
out=$1; shift
envs=$1; shift
wl=${@:-landau2d-128 weibel-256}
timeout 300 python -m pytest tests/test_gpu.py -q -x -k "tiled or fused_path" 2>&1 | tail -1 >> $out
for w in $wl; do
  env $envs timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs', '$w', round(d['ms_per_step'],3), '%.3g' % d['value'], round(d['roofline']['frac'],4), [round(v,3) for v in d['roofline']['stage_ms_per_step']])" >> $out 2>&1
done
