python tools/rows_variants.py 2 300 > gpurun_out/q_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rows_fista_fast" -s 400 -c 1 -o gpurun_out/q_cfg2_late python tools/rows_variants.py 2 300 > gpurun_out/q_ncu1.log 2>&1
timeout 300 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/q_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rows_admm" -s 300 -c 1 -o gpurun_out/q_cfg3_admm python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/q_ncu3.log 2>&1
echo done
