# Round-1 evidence, session 2 (run from the repo root on the B200 via gpurun).  Every profiled
# command first runs to exit 0 without ncu.
#  1. bench lines: default (config 2 with CPU baseline + e2e), configs 1/3/4/5, reference arm
#  2. ncu launch list (time + DRAM bytes per launch) of one full solve, configs 2-5
#  3. ncu --set full of the top kernels: config 2 rows (early, late) + column pass (late),
#     config 3 rows, config 4 rows, config 5 rows
set -x
OUT=${OUT:-gpurun_out/ev}
mkdir -p $OUT
python bench.py > $OUT/bench_r1.json 2> $OUT/bench.err
for c in 1 3 4 5; do python bench.py --config $c --steps 3 --warmup 3 > $OUT/bench_r1_cfg$c.json 2>> $OUT/bench.err; done
python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_ref_r1.json 2>> $OUT/bench.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in 2 3 4 5; do
  python tools/one_solve.py $c > $OUT/plain_solve$c.log 2>&1 && \
  ncu --metrics $M --clock-control none -c 7000 --csv --log-file $OUT/launches_cfg$c.csv \
      python tools/one_solve.py $c > $OUT/ncu_solve$c.log 2>&1
  python tools/make_profile_summary.py s2_cfg${c}_launches $OUT/launches_cfg$c.csv > /dev/null 2>&1
  python tools/ncu_bytes_per_gpi.py $c profiles/s2_cfg${c}_launches_launches.json \
      "profiles/s2_cfg${c}_launches.txt: ncu --metrics $M over one full tools/one_solve.py $c (cold-cache, serialised)" >> $OUT/bpg.log 2>&1
done
cap() {  # name cfg kernel-regex skip
  ncu --set full --clock-control none --import-source on -k regex:"$3" -s $4 -c 1 -o $OUT/$1 \
      python tools/one_solve.py $2 > $OUT/ncu_$1.log 2>&1
  ncu -i $OUT/$1.ncu-rep --page source --csv --print-source=sass,cuda > $OUT/$1_source.csv 2>/dev/null
  python tools/ncu_source_hot.py $OUT/$1_source.csv 30 > $OUT/$1_hot_lines.txt 2>/dev/null
}
cap cfg2_rows_early 2 rows_fista_fast 9
cap cfg2_rows_late 2 rows_fista_fast 1500
cap cfg2_cols_late 2 cols_warp_kernel 1500
cap cfg3_rows 3 rows_admm_split 600
cap cfg4_rows 4 rows_fista_fast 600
cap cfg5_rows 5 rows_fista_fast 600
python tools/make_profile_summary.py s2_top_kernels $OUT/cfg2_rows_early.ncu-rep $OUT/cfg2_rows_late.ncu-rep \
    $OUT/cfg2_cols_late.ncu-rep $OUT/cfg3_rows.ncu-rep $OUT/cfg4_rows.ncu-rep $OUT/cfg5_rows.ncu-rep > /dev/null 2>&1
cp profiles/s2_*.txt profiles/s2_*_launches.json profiles/ncu_summary.json $OUT/ 2>/dev/null
rm -f $OUT/*.ncu-rep $OUT/*_source.csv
du -sh $OUT
echo done
