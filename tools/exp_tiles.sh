set -u
o=gpurun_out
tools/bin/gather_bw > $o/gather_bw.json 2>&1
for t in 256 64 32 16; do
  echo "== tile $t" >> $o/tile_probe.txt
  DASPMM_TILE_COLS=$t timeout 300 python tools/probe.py --only uniform_s20_d16,powerlaw_s20_d16 --ns 32,64,128 --kernels 0,4 --no-torch >> $o/tile_probe.txt 2>&1
  DASPMM_TILE_COLS=$t timeout 300 python tools/probe.py --workload c3 --ns 128 --kernels 0,4 --no-torch >> $o/tile_probe.txt 2>&1
done
