# Profile capture for profiles/ (run under gpurun from the repo root).
#   launch list: every kernel launch of 4 C2 frames with its device time
#   full sets : the heaviest kernels of frame 10, one launch each
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python tools/frames_driver.py --frames 12 > gpurun_out/${TAG}_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'^k_(clear_walk|ccl_union|ccl_hook|poly_hull|integrate_fold|normals|recenter|poly_extremes|ransac_count|bitmap_count)$' \
  -s 100 -c 10 -o gpurun_out/${TAG}_top python tools/frames_driver.py --frames 12 > gpurun_out/${TAG}_full.log 2>&1
ls -la gpurun_out
