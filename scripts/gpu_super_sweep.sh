# CTA-order sweep for the 2D-2V stage kernel: VPFV_SUPER=sj,sk super-tiles, VPFV_XSEG x segments
rm -f gpurun_out/super.txt
for cfg in "4,8 0" "2,8 0" "8,8 0" "4,4 0" "16,8 0" "1,1 0" "4,8 2" "8,4 0" "4,8 0"; do
  set -- $cfg
  VPFV_SUPER=$1 VPFV_XSEG=$2 timeout 300 python bench.py --steps 12 --warmup 4 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('super=$1 xseg=$2', round(d['ms_per_step'],3), [round(x,3) for x in r['stage_ms_per_step']], round(r['frac'],3), d['clocks']['sm_mhz'], r['clocks_roofline_pass']['sm_mhz'])" >> gpurun_out/super.txt
done
