# RB+CM+SR: base walk (lanes over columns) vs lanes over rows (spmm_cm.cu), suite s17/s20.
for v in 0 1; do
  echo "== DASPMM_CM_ROWS=$v"
  DASPMM_CM_ROWS=$v timeout 900 python tools/probe.py --only uniform_s17_d16,banded_s17_b8,uniform_s20_d16,powerlaw_s20_d16,banded_s20_b8 --ns 2,8,32,128 --kernels 0,2 --no-torch --reps 5 2>&1 | grep -E "_s1[0-9]|_s20"
done
