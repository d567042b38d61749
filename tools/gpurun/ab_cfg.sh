# A/B of library variants: C2 (value, e2e, latency, CCL kernels) x2 and C4/C5 (--workload) once.
# usage: VARIANTS="base lib/variants/x.so ..." WL="c4 c5" bash tools/gpurun/ab_cfg.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for v in ${VARIANTS:-base}; do
  if [ "$v" = "base" ]; then unset VP_LIB; else export VP_LIB=paper_2510_01592_b200/$v; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/ab_$(basename $v .so)_$rep.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ab_$(basename $v .so)_$rep.json'));k=d.get('kernels',{})
print('$v c2', d['value'], d['e2e']['value'], d['latency_ms_p50'], {n: round(k[n]['ms_per_step']/30*1000,1) for n in k if 'ccl' in n})"
done
done
for w in ${WL:-c5}; do
for v in ${VARIANTS:-base}; do
  if [ "$v" = "base" ]; then unset VP_LIB; else export VP_LIB=paper_2510_01592_b200/$v; fi
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/ab_$w.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ab_$w.json'));print('$v $w', d['value'], d['e2e']['value'])"
done
done
