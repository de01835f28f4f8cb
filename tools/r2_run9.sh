# Round 2, GPU call 9: second-level class screen on the TC path (256-thread tiles).  Full pytest,
# default bench (config 5: e2e + CPU baseline), configs 4/2/3, reference arm, --set full of one late
# TC launch, then the launch list of one full config-5 solve (-> profiles/ncu_summary.json).
set -x
OUT=gpurun_out/r2i
mkdir -p $OUT
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_cfg5_quick.json 2>> $OUT/bench.err
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_cfg5.json 2>> $OUT/bench.err
timeout 600 python bench.py --config 4 --no-cpu-baseline --steps 5 > $OUT/bench_cfg4.json 2>> $OUT/bench.err
timeout 300 python bench.py --config 2 --no-cpu-baseline > $OUT/bench_cfg2.json 2>> $OUT/bench.err
timeout 300 python bench.py --config 3 --no-cpu-baseline --steps 5 > $OUT/bench_cfg3.json 2>> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2>> $OUT/bench.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rows_fista_tc -s 1500 -c 1 \
    -o $OUT/cfg5_rows_tc python tools/one_solve.py 5 > $OUT/ncu_full.log 2>&1
python tools/make_profile_summary.py r2i_cfg5_rows_tc $OUT/cfg5_rows_tc.ncu-rep > /dev/null 2>&1
ncu -i $OUT/cfg5_rows_tc.ncu-rep --page source --csv --print-source=sass,cuda > $OUT/cfg5_rows_tc_source.csv 2>/dev/null
python tools/ncu_source_hot.py $OUT/cfg5_rows_tc_source.csv 60 > $OUT/cfg5_rows_tc_hot_lines.txt 2>/dev/null
cp profiles/r2i_cfg5_rows_tc*.txt $OUT/ 2>/dev/null
gzip -f $OUT/cfg5_rows_tc_source.csv
rm -f $OUT/cfg5_rows_tc.ncu-rep
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum
timeout 2400 ncu --metrics $M --clock-control none -c 9000 --csv --log-file $OUT/launches_cfg5.csv \
    python tools/one_solve.py 5 > $OUT/ncu_solve5.log 2>&1
python tools/ncu_solve_summary.py 5 $OUT/launches_cfg5.csv $OUT/r2i_cfg5_launches.txt \
    "profiles/r2/r2i_cfg5_launches.txt: ncu --metrics $M over one full tools/one_solve.py 5 (cold-cache, serialised)" > $OUT/summary5.log 2>&1
cp profiles/ncu_summary.json $OUT/
rm -f $OUT/launches_cfg5.csv
echo done
