BCCB_PERSIST=1 python tools/rows_variants.py 2 300 > gpurun_out/q_plain.log 2>&1 && \
BCCB_PERSIST=1 ncu --set full --clock-control none --import-source on -k regex:"fista_persistent" -c 1 -o gpurun_out/q3_persist python tools/rows_variants.py 2 300 > gpurun_out/q_ncu1.log 2>&1
echo done
