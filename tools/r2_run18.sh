# Round 2: launch list of one full config-4 solve (-> profiles/ncu_summary.json cfg4) and the config-4 bench line.
set -x
OUT=gpurun_out/r2v
mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum
timeout 300 python tools/one_solve.py 4 > $OUT/plain_solve4.log 2>&1 && \
timeout 2400 ncu --metrics $M --clock-control none -c 6000 --csv --log-file $OUT/launches_cfg4.csv \
    python tools/one_solve.py 4 > $OUT/ncu_solve4.log 2>&1
python tools/ncu_solve_summary.py 4 $OUT/launches_cfg4.csv $OUT/r2v_cfg4_launches.txt \
    "profiles/r2/r2v_cfg4_launches.txt: ncu --metrics $M over one full tools/one_solve.py 4 (cold-cache, serialised)" > $OUT/summary4.log 2>&1
cp profiles/ncu_summary.json $OUT/
rm -f $OUT/launches_cfg4.csv
timeout 600 python bench.py --config 4 --no-cpu-baseline --steps 5 > $OUT/bench_cfg4.json 2>> $OUT/bench.err
echo done
