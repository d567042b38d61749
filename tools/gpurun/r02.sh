# round-2 iteration: box facts, all GPU tests (with durations), C2 bench, reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r02a}
( nproc; free -g; lscpu | grep -i "model name\|^CPU(s)\|Socket"; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv ) > gpurun_out/${T}_box.txt 2>&1
timeout ${PYT:-1500} python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider -rf --durations=20 ${PYARGS} > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
timeout 900 python bench.py ${BARGS:---steps 5 --warmup 3 --no-configs} > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.log; echo "bench rc=$?" >> gpurun_out/${T}_bench.log
if [ -z "$NOREF" ]; then timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.log; echo "ref rc=$?" >> gpurun_out/${T}_ref.log; fi
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi
cat gpurun_out/${T}_box.txt; tail -30 gpurun_out/${T}_pytest.log; tail -3 gpurun_out/${T}_bench.log; cut -c1-1500 gpurun_out/${T}_bench.json; cat gpurun_out/${T}_ref.json 2>/dev/null | cut -c1-1200
