set -u
o=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $o/gpu_tests.log 2>&1; echo rc=$? >> $o/gpu_tests.log
for w in "DASPMM_LEAN_WIN=0" "DASPMM_LEAN_WIN=1"; do
  echo "== $w" >> $o/win_probe.txt
  env $w timeout 300 python tools/probe.py --only banded_s20_b8,banded_s17_b8,banded_s14_b8 --ns 32,64,128 --kernels 0 --no-torch 2>/dev/null >> $o/win_probe.txt
done
