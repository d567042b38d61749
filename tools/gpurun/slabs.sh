# distributed slab segmentation: virtual-slab parity tests, C5 probe (1 vs 4 slabs), C5 bench (1 slab)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_slabs.py -q -x --timeout=500 -p no:cacheprovider > gpurun_out/pytest_slabs.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_slabs.log
timeout 600 python tools/c5_probe.py --frames 6 --slabs 1 4 8 > gpurun_out/c5.log 2>&1; echo "c5 rc=$?" >> gpurun_out/c5.log
timeout 600 python bench.py --workload c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.log; echo "rc=$?" >> gpurun_out/bench_c5.log
tail -15 gpurun_out/pytest_slabs.log; tail -25 gpurun_out/c5.log; tail -3 gpurun_out/bench_c5.log; cut -c1-400 gpurun_out/bench_c5.json
