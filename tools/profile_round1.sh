# Round-1 evidence: full ncu capture of the headline rows kernel at a sparse (late) and a dense
# (early) iteration of config 2, plus the launch list of bench.py's timed solve.
set -x
python tools/rows_variants.py 2 300 > gpurun_out/p_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rows_fista_fast" -s 400 -c 1 -o gpurun_out/prof_r1_cfg2_late python tools/rows_variants.py 2 300 > gpurun_out/p_ncu1.log 2>&1
python tools/rows_variants.py 2 300 > gpurun_out/p_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rows_fista_fast" -s 6 -c 1 -o gpurun_out/prof_r1_cfg2_early python tools/rows_variants.py 2 300 > gpurun_out/p_ncu2.log 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/p_plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2100 --csv --log-file gpurun_out/launches_r1_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/p_ncu_b.log 2>&1
echo done
