for c in 64 128 256; do
  echo "== DASPMM_LEAN_CHUNK=$c"
  DASPMM_LEAN_CHUNK=$c timeout 300 python tools/probe.py --only powerlaw_s20_d16,uniform_s20_d16,banded_s20_b8,powerlaw_s17_d16 --ns 8,16 --kernels 4 --no-torch 2>/dev/null
  DASPMM_LEAN_CHUNK=$c timeout 300 python tools/probe.py --workload c4 --ns 16 --kernels 4 --no-torch 2>/dev/null
done
