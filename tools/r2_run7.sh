# Round 2, GPU call 7: un-pipelined TC tiles with prefetched band/flags and the TMEM energy screen.
set -x
OUT=gpurun_out/r2g
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for S in 1 0; do
  BCCB_SCREEN=$S timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_cfg5_screen$S.json 2>> $OUT/bench.err
done
timeout 600 python bench.py --no-cpu-baseline --steps 5 > $OUT/bench_cfg5_e2e.json 2>> $OUT/bench.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --substreams 1 > $OUT/bench_cfg5_sub1.json 2>> $OUT/bench.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --substreams 2 > $OUT/bench_cfg5_sub2.json 2>> $OUT/bench.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rows_fista_tc -s 1500 -c 1 \
    -o $OUT/cfg5_rows_tc python tools/one_solve.py 5 > $OUT/ncu_full.log 2>&1
python tools/make_profile_summary.py r2g_cfg5_rows_tc $OUT/cfg5_rows_tc.ncu-rep > /dev/null 2>&1
ncu -i $OUT/cfg5_rows_tc.ncu-rep --page source --csv --print-source=sass,cuda > $OUT/cfg5_rows_tc_source.csv 2>/dev/null
python tools/ncu_source_hot.py $OUT/cfg5_rows_tc_source.csv 60 > $OUT/cfg5_rows_tc_hot_lines.txt 2>/dev/null
cp profiles/r2g_cfg5_rows_tc*.txt $OUT/ 2>/dev/null
gzip -f $OUT/cfg5_rows_tc_source.csv
rm -f $OUT/cfg5_rows_tc.ncu-rep   # (gpurun_out is capped at 64 MiB; the text summaries are kept)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cols_kernel -s 1500 -c 1 \
    -o $OUT/cfg5_cols python tools/one_solve.py 5 > $OUT/ncu_full_cols.log 2>&1
python tools/make_profile_summary.py r2g_cfg5_cols $OUT/cfg5_cols.ncu-rep > /dev/null 2>&1
ncu -i $OUT/cfg5_cols.ncu-rep --page source --csv --print-source=sass,cuda > $OUT/cfg5_cols_source.csv 2>/dev/null
python tools/ncu_source_hot.py $OUT/cfg5_cols_source.csv 40 > $OUT/cfg5_cols_hot_lines.txt 2>/dev/null
cp profiles/r2g_cfg5_cols*.txt $OUT/ 2>/dev/null
gzip -f $OUT/cfg5_cols_source.csv
rm -f $OUT/cfg5_cols.ncu-rep   # (gpurun_out is capped at 64 MiB; the text summaries are kept)
echo done
