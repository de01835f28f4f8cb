# tools/bench_brief.sh CFG... : one short bench per config, key fields only
for cfg in "$@"; do
  timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('cfg$cfg', round(d['value']/1e9,2), 'Ggpi/s', round(d['ms_per_step'],3), 'ms', 'launch/step', d['gpu_launches_per_step'],
      'rows_ms', round(r['avg_launch_ms'],4), 'rows_share', round(r['share_of_step'],3),
      'cols', {k: (round(v,4) if isinstance(v,(int,float)) else v) for k,v in (r.get('cols_kernel') or {}).items()})"
done
