# EB segment walk after the per-width choice vs before: c3 at several N (long rows, all widths)
for lib in tools/bin/libdaspmm_before.so "" tools/bin/libdaspmm_before.so ""; do
  echo "== DASPMM_LIB=$lib"
  DASPMM_LIB=$lib timeout 600 python tools/probe.py --workload c3 --ns 8,16,32,64,128 --kernels 4 --no-torch --reps 5 2>&1 | grep -E "c3" | sed 's/torch\/cusparse 1000000000000.0us     0.0GF | //'
done
