# Session-3 refresh: launch list of one full config-2 solve with the final round-1 code
# (PDL mode 2, four sub-batch streams).  Run from the repo root on the B200 via gpurun.
set -x
OUT=${OUT:-gpurun_out/s3}
mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
python tools/one_solve.py 2 > $OUT/plain_solve2.log 2>&1 && \
ncu --metrics $M --clock-control none -c 7000 --csv --log-file $OUT/launches_cfg2.csv \
    python tools/one_solve.py 2 > $OUT/ncu_solve2.log 2>&1
python tools/make_profile_summary.py s3_cfg2_launches $OUT/launches_cfg2.csv > /dev/null 2>&1
cp profiles/s3_cfg2_launches.txt profiles/s3_cfg2_launches_launches.json $OUT/ 2>/dev/null
ls $OUT
