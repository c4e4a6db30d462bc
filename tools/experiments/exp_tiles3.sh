# 64- vs 128-column y-tiles at N=128 across the suite, c3 and c4 (all four SR kernels)
set -u
o=gpurun_out
for t in 128 64; do
  echo "== tile $t" >> $o/tile_probe3.txt
  DASPMM_TILE_COLS=$t timeout 400 python tools/probe.py --ns 128 --kernels 0,2,4,6 --no-torch 2>/dev/null >> $o/tile_probe3.txt
  DASPMM_TILE_COLS=$t timeout 300 python tools/probe.py --workload c3 --ns 128 --kernels 0,4 --no-torch 2>/dev/null >> $o/tile_probe3.txt
  DASPMM_TILE_COLS=$t timeout 300 python tools/probe.py --workload c4 --ns 64,128 --kernels 0,4 --no-torch 2>/dev/null >> $o/tile_probe3.txt
done
