# iteration run: GPU tests + C2 bench (+ optional extra command in $EXTRA)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout=600 -p no:cacheprovider -rf -x > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/bench.json 2> gpurun_out/bench.log; echo "bench rc=$?" >> gpurun_out/bench.log
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi
tail -4 gpurun_out/pytest.log; tail -2 gpurun_out/bench.log
python -c "
import json;d=json.load(open('gpurun_out/bench.json'))
print('value',d['value'],'ms/frame',d['ms_per_frame'],'e2e',d['e2e']['value'])
for k,v in list(d['kernels'].items())[:12]: print(k,v)
"
