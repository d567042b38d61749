# full check: smoke, all GPU tests, C2 bench, C5 slab probe
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout=600 -p no:cacheprovider -rf > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.log; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python tools/c5_probe.py --frames 6 --slabs 1 4 > gpurun_out/c5.log 2>&1; echo "c5 rc=$?" >> gpurun_out/c5.log
tail -3 gpurun_out/smoke.log; tail -8 gpurun_out/pytest.log; tail -3 gpurun_out/bench.log; cat gpurun_out/bench.json | cut -c1-600; tail -12 gpurun_out/c5.log
