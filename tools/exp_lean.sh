set -u
o=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $o/gpu_tests.log 2>&1; echo rc=$? >> $o/gpu_tests.log
for w in "DASPMM_LEAN=0" "DASPMM_LEAN_RW=0" "DASPMM_LEAN_RW=1"; do
  echo "== $w" >> $o/lean_probe.txt
  env $w timeout 300 python tools/probe.py --only uniform_s20_d16,powerlaw_s20_d16,banded_s20_b8,powerlaw_s17_d16 --ns 16,32,64,128 --kernels 0,4 --no-torch 2>/dev/null >> $o/lean_probe.txt
  env $w timeout 300 python tools/probe.py --workload c3 --ns 128 --kernels 4 --no-torch 2>/dev/null >> $o/lean_probe.txt
  env $w timeout 300 python tools/probe.py --workload c4 --ns 16,64 --kernels 4 --no-torch 2>/dev/null >> $o/lean_probe.txt
done
