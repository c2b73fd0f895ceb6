for v in main notma; do
  if [ $v = main ]; then lib=""; else lib="VPFV_LIB=exp/libvpfv_$v.so"; fi
  env $lib VPFV_1D1V_MARCH=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:march -c 12 --csv --log-file gpurun_out/mx_$v.csv python bench.py --workload twostream-1024 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done
