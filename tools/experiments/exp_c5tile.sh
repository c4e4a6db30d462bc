for t in 256 128; do
  echo "== DASPMM_TILE_COLS=$t"
  DASPMM_TILE_COLS=$t timeout 900 python tools/probe.py --workload c5 --ns 256 --kernels 0,4 --no-torch --reps 3 2>/dev/null
done
