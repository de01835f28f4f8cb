# Round 2, GPU call 11: L1/shared split A/B on the TC rows kernel.
set -x
OUT=gpurun_out/r2l
mkdir -p $OUT
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_cfg5.json 2>> $OUT/bench.err
BCCB_SCREEN=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_cfg5_screen0.json 2>> $OUT/bench.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rows_fista_tc -s 1500 -c 1 \
    -o $OUT/cfg5_rows_tc python tools/one_solve.py 5 > $OUT/ncu_full.log 2>&1
python tools/make_profile_summary.py r2l_cfg5_rows_tc $OUT/cfg5_rows_tc.ncu-rep > /dev/null 2>&1
ncu -i $OUT/cfg5_rows_tc.ncu-rep --page source --csv --print-source=sass,cuda > $OUT/cfg5_rows_tc_source.csv 2>/dev/null
python tools/ncu_source_hot.py $OUT/cfg5_rows_tc_source.csv 60 > $OUT/cfg5_rows_tc_hot_lines.txt 2>/dev/null
cp profiles/r2l_cfg5_rows_tc*.txt $OUT/ 2>/dev/null
gzip -f $OUT/cfg5_rows_tc_source.csv
rm -f $OUT/cfg5_rows_tc.ncu-rep
echo done
