for w in "DASPMM_CTA_THREADS=64 DASPMM_THR_THREADS=64" "DASPMM_CTA_THREADS=32 DASPMM_THR_THREADS=32"; do
  echo "== $w"
  env $w timeout 300 python tools/probe.py --only powerlaw_s20_d16,uniform_s20_d16,banded_s20_b8,powerlaw_s17_d16 --ns 2,4,32,64,128 --kernels 4 --no-torch 2>/dev/null
  env $w timeout 300 python tools/probe.py --workload c4 --ns 64 --kernels 4 --no-torch 2>/dev/null
done
