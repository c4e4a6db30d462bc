for lib in "" "DASPMM_LIB=tools/bin/libdaspmm_mb5.so" "DASPMM_LIB=tools/bin/libdaspmm_mb6.so"; do
  echo "== $lib"
  env $lib timeout 300 python tools/probe.py --only uniform_s20_d16,powerlaw_s20_d16,banded_s20_b8,uniform_s17_d16 --ns 16,32,64,128 --kernels 0,4 --no-torch 2>/dev/null
  env $lib timeout 300 python tools/probe.py --workload c4 --ns 64 --kernels 4 --no-torch 2>/dev/null
done
