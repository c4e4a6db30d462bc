# EB range walk (k_eb_sr_lean_rw, power-law N <= 16): quads per iteration x min CTAs/SM
for lib in "" tools/bin/libdaspmm_rw_q1_m3.so tools/bin/libdaspmm_rw_q1_m4.so tools/bin/libdaspmm_rw_q1_m5.so tools/bin/libdaspmm_rw_q2_m4.so ""; do
  echo "== DASPMM_LIB=$lib"
  DASPMM_LIB=$lib timeout 600 python tools/probe.py --only powerlaw_s17_d16,powerlaw_s20_d16 --ns 8,16 --kernels 4 --no-torch --reps 10 2>&1 | grep -E "_s1[0-9]|_s20" | sed 's/torch\/cusparse 1000000000000.0us     0.0GF | //'
done
