# Round 2, GPU call 13: config-5 parity tests with the final tolerances, CUDA-graph probe at
# config 2, compute-sanitizer memcheck over every kernel family.
set -x
OUT=gpurun_out/r2n
mkdir -p $OUT
BCCB_PARITY_OUT=$OUT/parity_cfg5_t1000.json BCCB_TRAJECTORY_OUT=$OUT/parity_cfg5_trajectory.json timeout 600 python -m pytest tests/test_gpu_cfg5.py -q --timeout 600 > $OUT/pytest_cfg5.log 2>&1
timeout 300 python tools/graph_probe.py 2 > $OUT/graph_probe_cfg2.txt 2>&1
TOOL=memcheck timeout 2400 bash tools/sanitize.sh > $OUT/sanitize_memcheck.log 2>&1
cp gpurun_out/sanitize/memcheck_summary.txt $OUT/ 2>/dev/null
echo done
