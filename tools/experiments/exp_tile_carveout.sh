# Tile walk (staged, wide N) under different L1/shared carveouts, twice each (variance).
for c in "" 25 50 75 100 ""; do
  echo "== DASPMM_TILE_CARVEOUT=$c"
  DASPMM_TILE_CARVEOUT=$c timeout 600 python tools/probe.py --only banded_s20_b8 --ns 32,64,128 --kernels 0 --no-torch --reps 10 2>&1 | grep banded
done
