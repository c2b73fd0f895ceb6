# A/B: programmatic dependent launch on the 1D chain (VPFV_PDL=0 disables)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "1d1v or march or fused_field or two_stream or twostream or landau or graph or cfl" > gpurun_out/t6.log 2>&1; echo rc=$? >> gpurun_out/t6.log
rm -f gpurun_out/pdl.txt
for rep in 1 2; do for p in 1 0; do for wl in landau1d-128 twostream-1024; do
  VPFV_PDL=$p timeout 300 python bench.py --workload $wl --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$p', '$wl', round(d['ms_per_step'],4), '%.3g' % d['value'])" >> gpurun_out/pdl.txt
done; done; done
