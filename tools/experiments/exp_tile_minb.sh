for lib in "" tools/bin/libdaspmm_tmb6.so tools/bin/libdaspmm_tmb7.so tools/bin/libdaspmm_tmb8.so; do
  echo "== DASPMM_LIB=$lib"
  DASPMM_LIB=$lib timeout 600 python tools/probe.py --only banded_s20_b8 --ns 32,64,128 --kernels 0 --no-torch --reps 10 2>&1 | grep -v Warn
done
