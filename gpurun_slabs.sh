cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout=600 -p no:cacheprovider -rf > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 600 python tools/c5_probe.py --frames 6 --slabs 1 4 > gpurun_out/c5.log 2>&1; echo "c5 rc=$?" >> gpurun_out/c5.log
tail -5 gpurun_out/pytest.log; tail -15 gpurun_out/c5.log
