for w in "DASPMM_LEAN_THREADS=128" "DASPMM_LEAN_THREADS=64"; do
  echo "== $w"
  env $w timeout 300 python tools/probe.py --only powerlaw_s20_d16,uniform_s20_d16,banded_s20_b8,powerlaw_s17_d16,powerlaw_s14_d16 --ns 8,16 --kernels 4 --no-torch 2>/dev/null
  env $w timeout 300 python tools/probe.py --workload c3 --ns 128 --kernels 4 --no-torch 2>/dev/null
  env $w timeout 300 python tools/probe.py --workload c4 --ns 16 --kernels 4 --no-torch 2>/dev/null
done
