for w in "DASPMM_LEAN=0" "DASPMM_LEAN=1"; do
  echo "== $w"
  env $w timeout 300 python tools/probe.py --only powerlaw_s17_d16,powerlaw_s20_d16,uniform_s17_d16,uniform_s20_d16,banded_s20_b8 --ns 8,16,32,64,128 --kernels 0,4 --no-torch 2>/dev/null
  env $w timeout 300 python tools/probe.py --workload c3 --ns 128 --kernels 4 --no-torch 2>/dev/null
  env $w timeout 300 python tools/probe.py --workload c4 --ns 16,64 --kernels 4 --no-torch 2>/dev/null
done
