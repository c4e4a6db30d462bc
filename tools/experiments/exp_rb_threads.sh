for w in "DASPMM_RB_THREADS=256" "DASPMM_RB_THREADS=128" "DASPMM_RB_THREADS=64"; do
  echo "== $w"
  env $w timeout 300 python tools/probe.py --only uniform_s20_d16,banded_s20_b8,uniform_s17_d16,banded_s17_b8,uniform_s14_d16 --ns 2,8,16,32,64,128 --kernels 0 --no-torch 2>/dev/null
done
