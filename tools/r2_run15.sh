# Round 2, GPU call 15: verification of the committed final code -- full pytest -m gpu, smoke, the
# driver's two bench invocations (default arm and --impl reference), launch list of bench's first steps.
set -x
OUT=gpurun_out/r2p
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2>> $OUT/bench.err
timeout 900 python bench.py > $OUT/bench_cfg5.json 2>> $OUT/bench.err
timeout 600 python bench.py --config 4 --no-cpu-baseline --steps 5 > $OUT/bench_cfg4.json 2>> $OUT/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/bench_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --iterations 20 > $OUT/ncu_bench.log 2>&1
python tools/ncu_launch_summary.py $OUT/bench_launches.csv > $OUT/bench_launches.txt 2>&1
echo done
