# Round 2, GPU call 8: 128-thread (single-line) tensor-core tiles.  Quick parity subset + bench A/B.
set -x
OUT=gpurun_out/r2h
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_tc.py -q -x --timeout 600 -k "screen or tensor_core or tf32 or substream" > $OUT/pytest_quick.log 2>&1; echo "rc=$?" >> $OUT/pytest_quick.log
timeout 300 python tests/cfg5_trajectory_tool.py $OUT/traj.json > $OUT/traj.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_cfg5.json 2>> $OUT/bench.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --substreams 1 > $OUT/bench_cfg5_sub1.json 2>> $OUT/bench.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --substreams 2 > $OUT/bench_cfg5_sub2.json 2>> $OUT/bench.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rows_fista_tc -s 1500 -c 1 \
    -o $OUT/cfg5_rows_tc python tools/one_solve.py 5 > $OUT/ncu_full.log 2>&1
python tools/make_profile_summary.py r2h_cfg5_rows_tc $OUT/cfg5_rows_tc.ncu-rep > /dev/null 2>&1
ncu -i $OUT/cfg5_rows_tc.ncu-rep --page source --csv --print-source=sass,cuda > $OUT/cfg5_rows_tc_source.csv 2>/dev/null
python tools/ncu_source_hot.py $OUT/cfg5_rows_tc_source.csv 60 > $OUT/cfg5_rows_tc_hot_lines.txt 2>/dev/null
cp profiles/r2h_cfg5_rows_tc*.txt $OUT/ 2>/dev/null
gzip -f $OUT/cfg5_rows_tc_source.csv
rm -f $OUT/cfg5_rows_tc.ncu-rep
echo done
