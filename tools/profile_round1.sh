# Round-1 evidence (run from the repo root on the B200 via gpurun).  Every profiled command
# first runs to exit 0 without ncu.
#  1. bench lines: default (config 2, with CPU baseline and e2e), configs 1/3/4/5, reference arm
#  2. ncu launch list of one full config-2 solve (time + DRAM bytes per launch)
#  3. ncu --set full of the top kernels: config 2 rows pass at a dense (early) and a sparse
#     (late) iteration, config 3 split-ADMM rows pass, config 4 rows pass
set -x
mkdir -p gpurun_out/r1
python bench.py > gpurun_out/r1/bench_r1.json 2> gpurun_out/r1/bench_r1.err
for c in 1 3 4 5; do python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/r1/bench_r1_cfg$c.json 2>> gpurun_out/r1/bench_r1.err; done
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r1/bench_ref_r1.json 2>> gpurun_out/r1/bench_r1.err
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r1/plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4300 --csv \
    --log-file gpurun_out/r1/launches_cfg2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r1/ncu_b.log 2>&1
python tools/rows_variants.py 2 300 > gpurun_out/r1/plain_rv.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rows_fista_fast" -s 6 -c 1 -o gpurun_out/r1/cfg2_early python tools/rows_variants.py 2 300 > gpurun_out/r1/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rows_fista_fast" -s 400 -c 1 -o gpurun_out/r1/cfg2_late python tools/rows_variants.py 2 300 > gpurun_out/r1/ncu2.log 2>&1
python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r1/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rows_admm_split" -s 200 -c 1 -o gpurun_out/r1/cfg3_rows python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r1/ncu3.log 2>&1
python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r1/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rows_fista_fast" -s 100 -c 1 -o gpurun_out/r1/cfg4_rows python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r1/ncu4.log 2>&1

# summaries on the box (the .ncu-rep files exceed gpurun's copy-back limit); keep the config-2
# late capture only
python tools/make_profile_summary.py r1_rows_kernels gpurun_out/r1/cfg2_early.ncu-rep gpurun_out/r1/cfg2_late.ncu-rep \
    gpurun_out/r1/cfg3_rows.ncu-rep gpurun_out/r1/cfg4_rows.ncu-rep > /dev/null 2>&1
python tools/make_profile_summary.py r1_cfg2_launches gpurun_out/r1/launches_cfg2.csv > /dev/null 2>&1
ncu -i gpurun_out/r1/cfg2_late.ncu-rep --page source --csv --print-source=sass,cuda > gpurun_out/r1/cfg2_late_source.csv 2>/dev/null
cp profiles/r1_rows_kernels.txt profiles/r1_cfg2_launches.txt profiles/r1_cfg2_launches_launches.json gpurun_out/r1/ 2>/dev/null
rm -f gpurun_out/r1/cfg2_early.ncu-rep gpurun_out/r1/cfg3_rows.ncu-rep gpurun_out/r1/cfg4_rows.ncu-rep
du -sh gpurun_out
echo done
