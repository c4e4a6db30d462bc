# the tiled dominant call (uniform s20 N=128, two 64-column passes): CTA size and rows per group
set -u
o=gpurun_out/tile64_knobs.txt; : > $o
for t in 64 128 256; do
  echo "== rb_threads $t" >> $o
  DASPMM_RB_THREADS=$t timeout 200 python tools/probe.py --only uniform_s20_d16 --ns 128 --kernels 0 --no-torch 2>/dev/null >> $o
done
for r in 2 4 8 16; do
  echo "== rpg $r" >> $o
  DASPMM_RPG=$r timeout 200 python tools/probe.py --only uniform_s20_d16 --ns 128 --kernels 0 --no-torch 2>/dev/null >> $o
done
