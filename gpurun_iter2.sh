cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout=600 -p no:cacheprovider -rf -x > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.log
timeout 300 python tools/frames_driver.py --frames 30 --counters > gpurun_out/counters.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_(ccl_union|poly_hull|clear_walk|normals|recenter|integrate_fold|poly_extremes)$' -s 70 -c 7 -o gpurun_out/prof_top python tools/frames_driver.py --frames 12 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/pytest.log
