cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/c5_probe.py --frames 8 --slabs 1 4 > gpurun_out/c5.log 2>&1; echo "c5 rc=$?" >> gpurun_out/c5.log
timeout 300 python -m pytest tests/test_gpu_slabs.py -q > gpurun_out/pytest_slabs.log 2>&1
tail -20 gpurun_out/c5.log; tail -2 gpurun_out/pytest_slabs.log
