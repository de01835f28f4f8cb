# Diagnose the config-5 T=1000 parity under engine toggles (one line per variant).
set -x
OUT=gpurun_out/diag
mkdir -p $OUT
run() { # name, env...
  name=$1; shift
  env "$@" BCCB_PARITY_OUT=$OUT/parity_$name.json timeout 600 python -m pytest tests/test_gpu_cfg5.py -q -x --timeout 600 > $OUT/pytest_$name.log 2>&1
  echo "$name rc=$? $(python - <<P
import json
try:
    d=json.load(open('$OUT/parity_$name.json'))
    print(' '.join('%.2e'%s['rel_l2'] for s in d['snapshots']), [s['top32_same_set'] for s in d['snapshots']])
except Exception as e:
    print('no report', e)
P
)" >> $OUT/summary.txt
}
run default A=1
run default_again A=1
run tc0 BCCB_ROWS_TC=0
run tc0_nosplit BCCB_ROWS_TC=0 BCCB_DEBUG=2
run barrier BCCB_DEBUG=1
run nosplit BCCB_DEBUG=2
run barrier_nosplit BCCB_DEBUG=3
run sub1 BCCB_SUBSTREAMS=1
run screen0 BCCB_SCREEN=0
run pdl0 BCCB_PDL=0
cat $OUT/summary.txt
