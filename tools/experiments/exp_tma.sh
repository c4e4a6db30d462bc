set -u
o=gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "tma" > $o/tma_test.log 2>&1; echo rc=$? >> $o/tma_test.log
for w in "DASPMM_TMA=0" "DASPMM_TMA=1" "DASPMM_TMA=1 DASPMM_TMA_LW=128" "DASPMM_TMA=1 DASPMM_TMA_LW=512"; do
  echo "== $w" >> $o/tma_probe.txt
  env $w timeout 300 python tools/probe.py --only uniform_s20_d16,powerlaw_s20_d16,banded_s20_b8 --ns 32,64,128 --kernels 4 --no-torch 2>/dev/null >> $o/tma_probe.txt
  env $w timeout 300 python tools/probe.py --workload c3 --ns 128 --kernels 4 --no-torch 2>/dev/null >> $o/tma_probe.txt
done
