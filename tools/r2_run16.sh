# Round 2, GPU call: full verification of the committed code (pytest -m gpu, smoke, default bench, reference arm).
set -x
OUT=gpurun_out/r2s
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2>> $OUT/bench.err
timeout 900 python bench.py > $OUT/bench_cfg5.json 2>> $OUT/bench.err
echo done
