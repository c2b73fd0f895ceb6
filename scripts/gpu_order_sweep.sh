#!/bin/bash
# 2D-2V stage kernel: DRAM bytes (ncu, cold L2, per launch) and bench stage times
# for several CTA orders (VPFV_SUPER = super-tile rows,cols of column blocks)
mkdir -p gpurun_out/order
for sup in "4,8" "16,1" "16,8" "8,8" "2,8" "1,8" "8,2"; do
  tag=$(echo $sup | tr , x)
  VPFV_SUPER=$sup timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
      -k regex:stage2d2v_rb -s 4 -c 4 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
      > gpurun_out/order/ncu_$tag.csv 2>/dev/null
  bash scripts/ab_env.sh gpurun_out/order/bench.txt landau2d-128 super_$tag VPFV_SUPER=$sup
done
