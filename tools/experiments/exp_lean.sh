set -u
o=gpurun_out
for w in "DASPMM_LEAN=1" "DASPMM_LEAN_MIN_LANES=2" "DASPMM_LEAN_CHUNK=64" "DASPMM_LEAN_CHUNK=256"; do
  echo "== $w" >> $o/lean_probe.txt
  env $w timeout 300 python tools/probe.py --only uniform_s20_d16,powerlaw_s20_d16,banded_s20_b8 --ns 8,16,32,64,128 --kernels 0,4 --no-torch 2>/dev/null >> $o/lean_probe.txt
  env $w timeout 300 python tools/probe.py --workload c3 --ns 128 --kernels 4 --no-torch 2>/dev/null >> $o/lean_probe.txt
done
