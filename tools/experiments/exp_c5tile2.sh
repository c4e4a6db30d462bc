# c5 (B 34 GB) and c4 with narrower column tiles: does halving the per-pass B slice
# (more A passes) raise the L2 hit rate on R-MAT's hot columns enough to pay?
for t in 128 64 32; do
  echo "== c5 DASPMM_TILE_COLS=$t"
  DASPMM_TILE_COLS=$t timeout 900 python tools/probe.py --workload c5 --ns 256 --kernels 4 --no-torch --reps 3 2>/dev/null
done
for t in 0 64 32 16; do
  echo "== c4 DASPMM_TILE_COLS=$t"
  DASPMM_TILE_COLS=$t timeout 900 python tools/probe.py --workload c4 --ns 16,64 --kernels 0,4 --no-torch --reps 5 2>/dev/null
done
