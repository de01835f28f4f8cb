# Round 2, GPU call 4: TMEM-resident level-1 twiddles in the TC engine; bench per-launch timing from an extra profiled step.
# instantiations (plain passes keep their registers); A/B TC vs CUDA-core engine; ncu of TC rows.
set -x
OUT=gpurun_out/r2d
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_paths.py tests/test_gpu_solvers.py -q -x --timeout 600 \
    -k "tensor_core or tf32 or fused_objective or cfg or config" > $OUT/pytest_focus.log 2>&1; echo "rc=$?" >> $OUT/pytest_focus.log
for c in 5 4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_cfg${c}_tc.json 2>> $OUT/bench.err
  BCCB_ROWS_TC=0 timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_cfg${c}_cc.json 2>> $OUT/bench.err
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 --substreams 1 > $OUT/bench_cfg${c}_tc_sub1.json 2>> $OUT/bench.err
  BCCB_ROWS_TC=0 timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 --substreams 1 > $OUT/bench_cfg${c}_cc_sub1.json 2>> $OUT/bench.err
done
timeout 300 python bench.py --config 2 --no-cpu-baseline --no-e2e > $OUT/bench_cfg2.json 2>> $OUT/bench.err
timeout 600 python tools/one_solve.py 5 > $OUT/plain_solve5.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rows_fista_tc -s 1500 -c 1 \
    -o $OUT/cfg5_rows_tc python tools/one_solve.py 5 > $OUT/ncu_full.log 2>&1
python tools/make_profile_summary.py r2d_cfg5_rows_tc $OUT/cfg5_rows_tc.ncu-rep > /dev/null 2>&1
ncu -i $OUT/cfg5_rows_tc.ncu-rep --page source --csv --print-source=sass,cuda > $OUT/cfg5_rows_tc_source.csv 2>/dev/null
python tools/ncu_source_hot.py $OUT/cfg5_rows_tc_source.csv 40 > $OUT/cfg5_rows_tc_hot_lines.txt 2>/dev/null
cp profiles/r2d_cfg5_rows_tc*.txt $OUT/ 2>/dev/null
gzip -f $OUT/cfg5_rows_tc_source.csv
echo done
