mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "fused_field or 1d1v or graph or protocol" > gpurun_out/t1.log 2>&1; echo "tests rc=$?" >> gpurun_out/t1.log
for wl in landau1d-128 twostream-1024 weibel-256; do
 for sp in 0 1; do
  VPFV_FIELD_SPLIT=$sp timeout 300 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split=$sp', '$wl', round(d['ms_per_step'],4), '%.3g' % d['value'], d.get('gpu_launches'), round(d['roofline']['frac'],4))" >> gpurun_out/ab1.txt 2>&1
 done
done
