# compute-sanitizer over a reduced -m gpu subset that exercises every piece of
# synchronisation code: the TMA/mbarrier rings of the tiled 2D-2V and 1D-2V
# kernels, the bulk-copy ring of the 1D-1V march kernel, the PDL field chain,
# the x-range launches, the last-CTA `done` counters, the fused moment finish
# the linked-slab peer push (system-scope signal words), and (round 2) the
# warp-specialised 2D-2V kernel's full/empty mbarrier protocol (the default).
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash scripts/gpu_sanitize.sh'
# Logs: gpurun_out/san_<tool>.log; summary: gpurun_out/san_summary.txt
mkdir -p gpurun_out
SEL='test_tiled_stage_vs_oracle and coef0-N0
  or test_tiled_stage_vs_oracle and coef3-N2
  or test_tiled_stage_wrap_reads_interior_and_fused_moment and N1
  or test_tiled12_stage_vs_oracle and coef1-N1
  or test_tiled12_wrap_and_fused_moment
  or test_1d1v_march_equals_generic and N0
  or test_fused_field_1d_equals_split_chain and two-stream-32-128
  or test_tiled_stage_x_ranges_equal_full_launch and N0
  or test_tiled_stage_nonfinite_index
  or test_landau2d_steps_fused_path_vs_c_oracle and 32
  or test_moment_partials_finish_is_the_fold_tree
  or test_peer_halo_push_linked_slabs_equal_simulation and 2
  or test_tiled_stage_vx_sign_layouts and coef1-vx0'
SEL=$(echo $SEL)
: > gpurun_out/san_summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 2400 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 200 \
      python -m pytest tests/test_gpu.py tests/test_gpu_parallel.py -m gpu -q -p no:cacheprovider -k "$SEL" \
      > gpurun_out/san_$tool.log 2>&1
  rc=$?
  echo "== $tool rc=$rc" >> gpurun_out/san_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|passed|failed|error" gpurun_out/san_$tool.log | sort | uniq -c | sort -rn | head -20 \
      >> gpurun_out/san_summary.txt
done
