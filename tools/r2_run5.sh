# Round 2, GPU call 5: pipelined TC engine.  Full pytest -m gpu, smoke, default bench (config 5,
# e2e + CPU baseline), A/B TC vs CUDA-core, config 4 / 2 lines, reference arm, ncu launch list of
# one full config-5 solve (-> profiles/ncu_summary.json) and --set full of one late TC launch.
set -x
OUT=gpurun_out/r2e
mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_tc.py tests/test_gpu_paths.py -q -x --timeout 600 -k "tf32 or tensor_core" > $OUT/pytest_tc.log 2>&1; echo "rc=$?" >> $OUT/pytest_tc.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_cfg5.json 2> $OUT/bench.err
BCCB_ROWS_TC=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_cfg5_cc.json 2>> $OUT/bench.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --substreams 1 > $OUT/bench_cfg5_sub1.json 2>> $OUT/bench.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --substreams 2 > $OUT/bench_cfg5_sub2.json 2>> $OUT/bench.err
timeout 600 python bench.py --config 4 --no-cpu-baseline --steps 5 > $OUT/bench_cfg4.json 2>> $OUT/bench.err
BCCB_ROWS_TC=2 timeout 600 python bench.py --config 4 --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_cfg4_tc.json 2>> $OUT/bench.err
timeout 300 python bench.py --config 2 --no-cpu-baseline > $OUT/bench_cfg2.json 2>> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2>> $OUT/bench.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum
timeout 600 python tools/one_solve.py 5 > $OUT/plain_solve5.log 2>&1 && \
timeout 2400 ncu --metrics $M --clock-control none -c 9000 --csv --log-file $OUT/launches_cfg5.csv \
    python tools/one_solve.py 5 > $OUT/ncu_solve5.log 2>&1
python tools/ncu_solve_summary.py 5 $OUT/launches_cfg5.csv $OUT/r2e_cfg5_launches.txt \
    "profiles/r2/r2e_cfg5_launches.txt: ncu --metrics $M over one full tools/one_solve.py 5 (cold-cache, serialised)" > $OUT/summary5.log 2>&1
cp profiles/ncu_summary.json $OUT/
gzip -f $OUT/launches_cfg5.csv
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rows_fista_tc -s 1500 -c 1 \
    -o $OUT/cfg5_rows_tc python tools/one_solve.py 5 > $OUT/ncu_full.log 2>&1
python tools/make_profile_summary.py r2e_cfg5_rows_tc $OUT/cfg5_rows_tc.ncu-rep > /dev/null 2>&1
ncu -i $OUT/cfg5_rows_tc.ncu-rep --page source --csv --print-source=sass,cuda > $OUT/cfg5_rows_tc_source.csv 2>/dev/null
python tools/ncu_source_hot.py $OUT/cfg5_rows_tc_source.csv 40 > $OUT/cfg5_rows_tc_hot_lines.txt 2>/dev/null
cp profiles/r2e_cfg5_rows_tc*.txt $OUT/ 2>/dev/null
gzip -f $OUT/cfg5_rows_tc_source.csv
rm -f $OUT/cfg5_rows_tc.ncu-rep   # (gpurun_out is capped at 64 MiB; the text summaries are kept)
echo done
