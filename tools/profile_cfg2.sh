# config-2 top kernels: --set full captures (sparse late iteration) of the rows and column
# passes + the launch list of one full solve.  Run from the repo root on the B200 via gpurun.
set -x
OUT=${OUT:-gpurun_out/p}
mkdir -p $OUT
python tools/rows_variants.py 2 300 > $OUT/plain_rv.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rows_fista_fast" -s 600 -c 1 -o $OUT/cfg2_rows_late \
    python tools/rows_variants.py 2 300 > $OUT/ncu_rows.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"cols_kernel" -s 600 -c 1 -o $OUT/cfg2_cols_late \
    python tools/rows_variants.py 2 300 > $OUT/ncu_cols.log 2>&1
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 7000 --csv \
    --log-file $OUT/launches_cfg2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_b.log 2>&1
for r in cfg2_rows_late cfg2_cols_late; do
  ncu -i $OUT/$r.ncu-rep --page source --csv --print-source=sass,cuda > $OUT/${r}_source.csv 2>/dev/null
  ncu -i $OUT/$r.ncu-rep --page raw --csv > $OUT/${r}_raw.csv 2>/dev/null
done
python tools/make_profile_summary.py s2_cfg2_kernels $OUT/cfg2_rows_late.ncu-rep $OUT/cfg2_cols_late.ncu-rep > /dev/null 2>&1
python tools/make_profile_summary.py s2_cfg2_launches $OUT/launches_cfg2.csv > /dev/null 2>&1
cp profiles/s2_cfg2_kernels.txt profiles/s2_cfg2_launches.txt profiles/s2_cfg2_launches_launches.json $OUT/ 2>/dev/null
rm -f $OUT/*.ncu-rep
du -sh $OUT
