# A/B of library variants on two workloads, interleaved: scripts/gpu_variant_ab2.sh NAME...
rm -f gpurun_out/var.txt
for rep in 1 2; do for wl in landau2d-128 weibel-256; do for v in main "$@"; do
  if [ "$v" = main ]; then lib=""; else lib="VPFV_LIB=exp/libvpfv_$v.so"; fi
  env $lib timeout 300 python bench.py --workload $wl --steps 12 --warmup 4 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', '$wl', round(d['ms_per_step'],4), [round(x,4) for x in r['stage_ms_per_step']], round(r['frac'],3), d['clocks']['sm_mhz'], r['clocks_roofline_pass']['sm_mhz'])" >> gpurun_out/var.txt
done; done; done
