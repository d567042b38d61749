cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for f in -1 1; do
  for rep in 1 2; do
    VP_DDA_FORCE=$f timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/abd.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/abd.json'));k=d['kernels'];print('c2 force=$f', d['value'], d['e2e']['value'], d['latency_ms_p50'], 'walk', round(k['k_clear_walk']['ms_per_step']/30*1000,1), 'apply', round(k['k_clear_apply']['ms_per_step']/30*1000,1))"
  done
  VP_DDA_FORCE=$f timeout 300 python tools/c5_probe.py --frames 8 --slabs 1 > gpurun_out/abd_c5.log 2>&1; echo "c5 force=$f"; grep -E "frame (5|6|7)" gpurun_out/abd_c5.log | sed 's/|.*broadcast/ | bci/' | cut -c1-140
done
