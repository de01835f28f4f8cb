# Round 2, GPU call 12 (final code): launch list of one full config-5 solve -> profiles/ncu_summary.json,
# --set full of one late TC launch, full pytest, smoke, then the bench lines (default config 5 with e2e +
# CPU baseline, configs 4/2/3, reference arm).
set -x
OUT=gpurun_out/r2m
mkdir -p $OUT
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_cfg5_quick.json 2>> $OUT/bench.err
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
BCCB_PARITY_OUT=$OUT/parity_cfg5_t1000.json BCCB_TRAJECTORY_OUT=$OUT/parity_cfg5_trajectory.json timeout 600 python -m pytest tests/test_gpu_cfg5.py -q --timeout 600 > $OUT/pytest_cfg5.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rows_fista_tc -s 1500 -c 1 \
    -o $OUT/cfg5_rows_tc python tools/one_solve.py 5 > $OUT/ncu_full.log 2>&1
python tools/make_profile_summary.py r2m_cfg5_rows_tc $OUT/cfg5_rows_tc.ncu-rep > /dev/null 2>&1
ncu -i $OUT/cfg5_rows_tc.ncu-rep --page source --csv --print-source=sass,cuda > $OUT/cfg5_rows_tc_source.csv 2>/dev/null
python tools/ncu_source_hot.py $OUT/cfg5_rows_tc_source.csv 60 > $OUT/cfg5_rows_tc_hot_lines.txt 2>/dev/null
cp profiles/r2m_cfg5_rows_tc*.txt $OUT/ 2>/dev/null
gzip -f $OUT/cfg5_rows_tc_source.csv
rm -f $OUT/cfg5_rows_tc.ncu-rep
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum
timeout 2400 ncu --metrics $M --clock-control none -c 9000 --csv --log-file $OUT/launches_cfg5.csv \
    python tools/one_solve.py 5 > $OUT/ncu_solve5.log 2>&1
python tools/ncu_solve_summary.py 5 $OUT/launches_cfg5.csv $OUT/r2m_cfg5_launches.txt \
    "profiles/r2/r2m_cfg5_launches.txt: ncu --metrics $M over one full tools/one_solve.py 5 (cold-cache, serialised)" > $OUT/summary5.log 2>&1
cp profiles/ncu_summary.json $OUT/
rm -f $OUT/launches_cfg5.csv
timeout 900 python bench.py > $OUT/bench_cfg5.json 2>> $OUT/bench.err
timeout 600 python bench.py --config 4 --no-cpu-baseline --steps 5 > $OUT/bench_cfg4.json 2>> $OUT/bench.err
timeout 300 python bench.py --config 2 --no-cpu-baseline > $OUT/bench_cfg2.json 2>> $OUT/bench.err
timeout 300 python bench.py --config 3 --no-cpu-baseline --steps 5 > $OUT/bench_cfg3.json 2>> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2>> $OUT/bench.err
echo done
