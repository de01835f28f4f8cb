# compute-sanitizer over every kernel family (tools/sanitize.py), ONE tool per gpurun call:
#   gpurun -- 'TOOL=memcheck bash tools/sanitize.sh'     (then racecheck, synccheck)
set -x
TOOL=${TOOL:-memcheck}
OUT=gpurun_out/sanitize
mkdir -p $OUT
python tools/sanitize.py operator > $OUT/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
for fam in operator fista tc trace cluster small admm; do
  timeout 900 compute-sanitizer --tool $TOOL --error-exitcode 9 python tools/sanitize.py $fam \
      > $OUT/${TOOL}_$fam.log 2>&1; echo "$fam rc=$?" >> $OUT/${TOOL}_summary.txt
done
BCCB_CLUSTER=0 BCCB_SMALL_GRID=0 timeout 900 compute-sanitizer --tool $TOOL --error-exitcode 9 \
    python tools/sanitize.py fused > $OUT/${TOOL}_fused.log 2>&1; echo "fused rc=$?" >> $OUT/${TOOL}_summary.txt
grep -h "ERROR SUMMARY" $OUT/${TOOL}_*.log >> $OUT/${TOOL}_summary.txt
cat $OUT/${TOOL}_summary.txt
