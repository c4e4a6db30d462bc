# B-row prefetch one step ahead in sr_walk (k_rb_sr, k_eb_sr_cta): off / L2 / L1
for lib in "" tools/bin/libdaspmm_bpref1.so tools/bin/libdaspmm_bpref2.so ""; do
  echo "== DASPMM_LIB=$lib"
  DASPMM_LIB=$lib timeout 600 python tools/probe.py --only uniform_s20_d16,powerlaw_s20_d16,uniform_s17_d16 --ns 8,16,32,64,128 --kernels 0,4 --no-torch --reps 10 2>&1 | grep -E "_s1[0-9]|_s20" | sed 's/torch\/cusparse 1000000000000.0us     0.0GF | //'
done
