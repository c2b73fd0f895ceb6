# A/B: preferred max-shared carveout on the small kernels next to the stage kernels
rm -f gpurun_out/carve.txt
for v in main nocarve; do
  if [ $v = main ]; then lib=""; else lib="VPFV_LIB=exp/libvpfv_$v.so"; fi
  for wl in twostream-1024 landau1d-128 weibel-256; do
    env $lib timeout 300 python bench.py --workload $wl --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$wl', round(d['ms_per_step'],4), '%.3g' % d['value'])" >> gpurun_out/carve.txt
  done
done
