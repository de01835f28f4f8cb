# Round 2, GPU call 1 (run from the repo root on the B200 via gpurun).
#  1. pytest -m gpu, smoke()
#  2. bench: default (config 5, kernel events on), config 5 without kernel events, config 5
#     with 1 sub-batch stream, config 4; config 2 sub-stream count 3 vs 4 (3 reps each)
#  3. ncu launch list (time, DRAM bytes, FP32 op counts, instructions) of one full config-5 solve
set -x
OUT=gpurun_out/r2a
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_cfg5.json 2> $OUT/bench_cfg5.err
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-kernel-events --steps 5 > $OUT/bench_cfg5_noev.json 2>> $OUT/bench.err
timeout 600 python bench.py --no-e2e --no-cpu-baseline --substreams 1 --steps 5 > $OUT/bench_cfg5_sub1.json 2>> $OUT/bench.err
timeout 600 python bench.py --no-e2e --no-cpu-baseline --substreams 1 --no-kernel-events --steps 5 > $OUT/bench_cfg5_sub1_noev.json 2>> $OUT/bench.err
timeout 600 python bench.py --config 4 --no-cpu-baseline --steps 5 > $OUT/bench_cfg4.json 2>> $OUT/bench.err
for r in 1 2 3; do
  for n in 3 4; do
    timeout 300 python bench.py --config 2 --no-e2e --no-cpu-baseline --no-kernel-events --substreams $n > $OUT/bench_cfg2_sub${n}_r$r.json 2>> $OUT/bench.err
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum
timeout 600 python tools/one_solve.py 5 > $OUT/plain_solve5.log 2>&1 && \
timeout 1800 ncu --metrics $M --clock-control none -c 5000 --csv --log-file $OUT/launches_cfg5.csv \
    python tools/one_solve.py 5 > $OUT/ncu_solve5.log 2>&1
python tools/ncu_solve_summary.py 5 $OUT/launches_cfg5.csv $OUT/r2_cfg5_launches.txt \
    "profiles/r2/r2_cfg5_launches.txt: ncu --metrics $M over one full tools/one_solve.py 5 (cold-cache, serialised)" > $OUT/summary5.log 2>&1
cp profiles/ncu_summary.json $OUT/
gzip -f $OUT/launches_cfg5.csv
du -sh $OUT
echo done
