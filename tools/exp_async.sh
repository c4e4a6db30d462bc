set -u
o=gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "tma" > $o/async_test.log 2>&1; echo rc=$? >> $o/async_test.log
for w in "DASPMM_ASYNC=0" "DASPMM_ASYNC=1" "DASPMM_ASYNC=1 DASPMM_ASYNC_LW=512" "DASPMM_ASYNC=1 DASPMM_ASYNC_LW=128"; do
  echo "== $w" >> $o/async_probe.txt
  env $w timeout 300 python tools/probe.py --only uniform_s20_d16,powerlaw_s20_d16 --ns 32,64,128 --kernels 4 --no-torch 2>/dev/null >> $o/async_probe.txt
  env $w timeout 300 python tools/probe.py --workload c3 --ns 128 --kernels 4 --no-torch 2>/dev/null >> $o/async_probe.txt
  env $w timeout 300 python tools/probe.py --workload c4 --ns 64 --kernels 4 --no-torch 2>/dev/null >> $o/async_probe.txt
done
