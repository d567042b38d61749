# A/B of library variants on the C2 bench (value, e2e, latency); 2 runs each.
# usage: VARIANTS="base lib/variants/x.so ..." bash tools/gpurun/ab.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for v in ${VARIANTS:-base}; do
  if [ "$v" = "base" ]; then unset VP_LIB; else export VP_LIB=paper_2510_01592_b200/$v; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', d['value'], d['e2e']['value'], d['latency_ms_p50'])"
done
done
