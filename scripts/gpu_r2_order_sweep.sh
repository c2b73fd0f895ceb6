# CTA order / x-segment sweep on the warp-specialised kernel (stage_ab, interleaved)
mkdir -p gpurun_out
: > gpurun_out/sweep.txt
for rep in 1 2; do
  for cfg in "4,8 0" "16,1 0" "8,2 0" "2,8 0" "16,8 0" "4,8 2"; do
    set -- $cfg
    VPFV_SUPER=$1 VPFV_XSEG=$2 timeout 300 python scripts/stage_ab.py --reps 15 main 2>&1 | sed "s/^/super=$1 xseg=$2 /" >> gpurun_out/sweep.txt
  done
done
