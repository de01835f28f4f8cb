# A/B helper: tools/ab_cfg.sh CFG REPS "ENV_A" "ENV_B" ...   (each ENV is a space-separated list of VAR=value)
cfg=$1; n=$2; shift 2
for i in $(seq $n); do
  for e in "$@"; do
    v=$(env $e timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,2), round(d['ms_per_step'],3), d['gpu_launches_per_step'])")
    echo "cfg$cfg [$e] $v"
  done
done
