echo "== default"
timeout 300 python tools/probe.py --only powerlaw_s14_d16,powerlaw_s17_d16,powerlaw_s20_d16,uniform_s17_d16,uniform_s20_d16,banded_s20_b8 --ns 64,128 --kernels 4 --no-torch 2>/dev/null
timeout 300 python tools/probe.py --workload c4 --ns 64 --kernels 4 --no-torch 2>/dev/null
for r in 4 8 16 32; do
  echo "== DASPMM_RPG=$r"
  DASPMM_RPG=$r timeout 300 python tools/probe.py --only uniform_s20_d16,banded_s20_b8,uniform_s17_d16 --ns 16,32,64,128 --kernels 0 --no-torch 2>/dev/null
done
