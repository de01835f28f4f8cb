# Round 2, last GPU call: ncu evidence of the committed code -- --set full of one late TC rows launch and
# one column-pass launch, launch list of one full config-5 solve (-> profiles/ncu_summary.json), then the
# default bench reading that summary.
set -x
OUT=gpurun_out/r2t
mkdir -p $OUT
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rows_fista_tc -s 1500 -c 1 \
    -o $OUT/cfg5_rows_tc python tools/one_solve.py 5 > $OUT/ncu_full.log 2>&1
python tools/make_profile_summary.py r2t_cfg5_rows_tc $OUT/cfg5_rows_tc.ncu-rep > /dev/null 2>&1
ncu -i $OUT/cfg5_rows_tc.ncu-rep --page source --csv --print-source=sass,cuda > $OUT/cfg5_rows_tc_source.csv 2>/dev/null
python tools/ncu_source_hot.py $OUT/cfg5_rows_tc_source.csv 60 > $OUT/cfg5_rows_tc_hot_lines.txt 2>/dev/null
python - $OUT/cfg5_rows_tc_source.csv > $OUT/cfg5_rows_tc_blackwell_sass.txt <<'P'
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = rows[2]
seen = {}
for r in rows:
    if len(r) < len(h):
        continue
    try:
        n = int(r[7])
    except ValueError:
        continue
    if r[2] and r[3]:
        seen[r[2]] = (r[3], n)
c = collections.Counter()
for ins, n in seen.values():
    t = ins.split()
    op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "?")).split(".")[0]
    if op.startswith(("UTC", "LDTM", "STTM", "LDGSTS", "SYNCS", "UTMA")):
        c[op] += n
print("warp-level executed counts of Blackwell-specific SASS in this launch:", dict(c))
P
cp profiles/r2t_cfg5_rows_tc*.txt $OUT/ 2>/dev/null
rm -f $OUT/cfg5_rows_tc.ncu-rep $OUT/cfg5_rows_tc_source.csv
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum
timeout 2400 ncu --metrics $M --clock-control none -c 9000 --csv --log-file $OUT/launches_cfg5.csv \
    python tools/one_solve.py 5 > $OUT/ncu_solve5.log 2>&1
python tools/ncu_solve_summary.py 5 $OUT/launches_cfg5.csv $OUT/r2t_cfg5_launches.txt \
    "profiles/r2/r2t_cfg5_launches.txt: ncu --metrics $M over one full tools/one_solve.py 5 (cold-cache, serialised)" > $OUT/summary5.log 2>&1
cp profiles/ncu_summary.json $OUT/
rm -f $OUT/launches_cfg5.csv
timeout 900 python bench.py > $OUT/bench_cfg5.json 2>> $OUT/bench.err
echo done
