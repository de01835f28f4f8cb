# Round 2, GPU call 6: energy-screened level-1 inverse DFT.  Neutrality + parity tests, A/B bench
# (BCCB_SCREEN=0/1) at configs 5/4/2/3, --set full of one late TC launch.
set -x
OUT=gpurun_out/r2f
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for S in 1 0; do
  BCCB_SCREEN=$S timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_cfg5_screen$S.json 2>> $OUT/bench.err
  BCCB_SCREEN=$S timeout 600 python bench.py --config 4 --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_cfg4_screen$S.json 2>> $OUT/bench.err
  BCCB_SCREEN=$S timeout 300 python bench.py --config 2 --no-cpu-baseline --no-e2e > $OUT/bench_cfg2_screen$S.json 2>> $OUT/bench.err
  BCCB_SCREEN=$S timeout 300 python bench.py --config 3 --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_cfg3_screen$S.json 2>> $OUT/bench.err
done
BCCB_ROWS_TC=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_cfg5_cc.json 2>> $OUT/bench.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rows_fista_tc -s 1500 -c 1 \
    -o $OUT/cfg5_rows_tc python tools/one_solve.py 5 > $OUT/ncu_full.log 2>&1
python tools/make_profile_summary.py r2f_cfg5_rows_tc $OUT/cfg5_rows_tc.ncu-rep > /dev/null 2>&1
ncu -i $OUT/cfg5_rows_tc.ncu-rep --page source --csv --print-source=sass,cuda > $OUT/cfg5_rows_tc_source.csv 2>/dev/null
python tools/ncu_source_hot.py $OUT/cfg5_rows_tc_source.csv 60 > $OUT/cfg5_rows_tc_hot_lines.txt 2>/dev/null
cp profiles/r2f_cfg5_rows_tc*.txt $OUT/ 2>/dev/null
gzip -f $OUT/cfg5_rows_tc_source.csv
rm -f $OUT/cfg5_rows_tc.ncu-rep   # (gpurun_out is capped at 64 MiB; the text summaries are kept)
echo done
