set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.txt 2>&1; echo pytest rc=$?
tail -3 gpurun_out/g1_pytest.txt
for cfg in "" "DASPMM_TILE_COLS=16" "DASPMM_TILE_COLS=16 DASPMM_LEAN_RB=1" "DASPMM_TILE_COLS=32 DASPMM_LEAN_RB=1" "DASPMM_LEAN_RB=1"; do
  echo "== $cfg" >> gpurun_out/g1_probe.txt
  env $cfg timeout 300 python tools/probe.py --only uniform_s20_d16,uniform_s17_d16 --ns 16,32,128 --kernels 0 --no-torch >> gpurun_out/g1_probe.txt 2>&1
done
timeout 600 bash tools/prof_one.sh k_rb_sr uniform_s20_d16 16 0 g1_rbsr_u20_N16
timeout 600 bash tools/prof_one.sh k_rb_sr uniform_s17_d16 16 0 g1_rbsr_u17_N16
cp /tmp/prof_g1_rbsr_u20_N16.ncu-rep gpurun_out/ 2>/dev/null
