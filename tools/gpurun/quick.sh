# quick iteration: selected GPU tests ($TESTS, default the CCL/hull/parity subset) + C2 bench kernel table
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-q}
TESTS=${TESTS:-"tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_gpu_dropin.py"}
timeout ${PYT:-900} python -m pytest $TESTS -m gpu -q --timeout=600 -p no:cacheprovider -rf -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
timeout 900 python bench.py ${BARGS:---steps 5 --warmup 3 --no-cpu-baseline --no-configs} > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.log; echo "bench rc=$?" >> gpurun_out/${T}_bench.log
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi
tail -4 gpurun_out/${T}_pytest.log; tail -2 gpurun_out/${T}_bench.log
python -c "
import json;d=json.load(open('gpurun_out/${T}_bench.json'))
print('value',d['value'],'ms/frame',d['ms_per_frame'],'e2e',d['e2e']['value'],'lat p50',d.get('latency_ms_p50'))
k=d['kernels']; print('sum us/frame', round(sum(v['ms_per_step'] for v in k.values())/30*1000,1))
for n,v in list(k.items())[:16]: print(f'{n:28s} {v[\"ms_per_step\"]/30*1000:7.1f}')
"
