# GPU check of the 1D field path: tests, then split-vs-fused A/B lines and the step-overhead probe
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q ${TESTK:+-k "$TESTK"} > gpurun_out/t1.log 2>&1; echo "tests rc=$?" >> gpurun_out/t1.log
rm -f gpurun_out/ab1.txt
for wl in landau1d-128 twostream-1024 weibel-256; do
 for sp in 0 1; do
  VPFV_FIELD_SPLIT=$sp timeout 300 python bench.py --workload $wl --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split=$sp', '$wl', round(d['ms_per_step'],4), '%.3g' % d['value'], d.get('gpu_launches'), round(d['roofline']['frac'],4), d['roofline']['timing'][-40:])" >> gpurun_out/ab1.txt 2>&1
 done
done
for w in landau1d-128 twostream-1024; do python scripts/probes/step_overhead.py $w; done > gpurun_out/ovh.txt 2>&1
