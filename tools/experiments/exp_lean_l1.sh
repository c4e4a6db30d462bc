for w in "DASPMM_LEAN_RB=0" "DASPMM_LEAN_RB=1 DASPMM_LEAN_MIN_LANES=1"; do
  echo "== $w"
  env $w timeout 300 python tools/probe.py --only uniform_s20_d16,banded_s20_b8,uniform_s17_d16,banded_s17_b8 --ns 2,4,8 --kernels 0 --no-torch 2>/dev/null
done
