# A/B of library builds on bench workloads (stage-kernel ms per step from the
# bench's in-graph events), interleaved: scripts/gpu_wl_ab.sh WORKLOAD...
mkdir -p gpurun_out
: > gpurun_out/wl_ab.txt
libs="main"
for f in exp/libvpfv_*.so; do libs="$libs $f"; done
for rep in 1 2; do for wl in "$@"; do for v in $libs; do
  if [ "$v" = main ]; then lib=""; else lib="VPFV_LIB=$v"; fi
  env $lib timeout 300 python bench.py --workload $wl --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$wl', '$v', round(d['ms_per_step'],4), round(sum(r['stage_ms_per_step']),4), round(r['frac'],4), d['clocks']['sm_mhz'], (d.get('parity') or {}).get('ok'))" >> gpurun_out/wl_ab.txt
done; done; done
