# Stream-K x split (VPFV_RB_SK): 2D-2V parity/variant tests, then config 5
# (two species on side streams) with and without it, interleaved.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu.py tests/test_gpu_benchsize.py -x -q -k "tiled or landau2d or graph_replay or medium_step or vx_sign or nonfinite or aliasing or ep2d2v or peer or range or variants or manufactured" > gpurun_out/sk_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sk_tests.log
: > gpurun_out/sk_ab.txt
for rep in 1 2 3; do for sk in 0 1; do
  VPFV_RB_SK=$sk timeout 300 python bench.py --workload ep2d2v-64 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('sk=$sk', round(d['ms_per_step'],4), round(sum(r['stage_ms_per_step']),4), round(r['frac'],4))" >> gpurun_out/sk_ab.txt
done; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 > gpurun_out/sk_landau2d.json
