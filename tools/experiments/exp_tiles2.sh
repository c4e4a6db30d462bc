# column tiles vs none on the dominant call, current kernels (uniform s20 N=128, RB+RM+SR)
set -u
o=gpurun_out
for t in 128 64 32 16; do
  echo "== tile $t" >> $o/tile_probe2.txt
  DASPMM_TILE_COLS=$t timeout 300 python tools/probe.py --only uniform_s20_d16 --ns 128 --kernels 0 --no-torch 2>/dev/null >> $o/tile_probe2.txt
done
