for e in "BCCB_FUSE_COLS=0" "BCCB_PDL=0" "BCCB_FUSE_COLS=0 BCCB_PDL=0" "BCCB_ROWS_VARIANT=1" "BCCB_COLS_WARP=0" "BCCB_ROWS_KP16=0"; do
  r=$(env BCCB_CLUSTER=0 BCCB_SMALL_GRID=0 $e timeout 300 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-120)
  echo "[$e] $r"
done
