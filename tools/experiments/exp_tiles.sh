set -u
o=gpurun_out
for t in 256 64 32; do
  echo "== tile $t" >> $o/tile_probe.txt
  DASPMM_TILE_COLS=$t timeout 300 python tools/probe.py --only uniform_s20_d16,powerlaw_s20_d16 --ns 64,128 --kernels 0,4 --no-torch 2>/dev/null >> $o/tile_probe.txt
  DASPMM_TILE_COLS=$t timeout 300 python tools/probe.py --workload c3 --ns 128 --kernels 4 --no-torch 2>/dev/null >> $o/tile_probe.txt
done
