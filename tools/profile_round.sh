# Profile capture for profiles/ (run under gpurun from the repo root).
#   bench     : the default bench line (not under a profiler)
#   launch list: every kernel launch of a short bench.py run with its device time
#   full sets : the heaviest kernels of C2 frame ~10, one launch each
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-configs \
  > gpurun_out/${TAG}_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'^k_(clear_walk|clear_apply|ccl_pairs|ccl_hook_bal|ccl_compress_exact|ccl_jump|ccl_flatten|poly_fused|integrate_fold|integrate_hash|integrate_fold_medium|normals|recenter|ransac_count|bitmap_count|bitmap_emit|member_scatter|refine_part0|extract_emit|step_emit)$' \
  -s 150 -c 20 -o gpurun_out/${TAG}_top python tools/frames_driver.py --frames 12 > gpurun_out/${TAG}_full.log 2>&1
ls -la gpurun_out
