for w in "DASPMM_THR8=0" "DASPMM_THR8=1"; do
  echo "== $w"
  env $w timeout 300 python tools/probe.py --only uniform_s20_d16,powerlaw_s20_d16,banded_s20_b8,uniform_s17_d16,powerlaw_s17_d16,powerlaw_s14_d16 --ns 8 --kernels 0,4 --no-torch 2>/dev/null
  env $w timeout 300 python tools/probe.py --workload c4 --ns 16 --kernels 4 --no-torch 2>/dev/null
done
