# lean segment walks: quads per iteration x min CTAs/SM (EB segment walk on c3; RB lean
# one-lane walk on uniform/banded N <= 4). Library name: lean_<segQ><segMinB><rbQ><rbMinB>.
for lib in "" tools/bin/libdaspmm_lean_1424.so tools/bin/libdaspmm_lean_1524.so tools/bin/libdaspmm_lean_2315.so tools/bin/libdaspmm_lean_2316.so ""; do
  echo "== DASPMM_LIB=$lib"
  DASPMM_LIB=$lib timeout 600 python tools/probe.py --only uniform_s17_d16,uniform_s20_d16 --ns 2,4 --kernels 0 --no-torch --reps 10 2>&1 | grep -E "_s1[0-9]|_s20" | sed 's/torch\/cusparse 1000000000000.0us     0.0GF | //'
  DASPMM_LIB=$lib timeout 600 python tools/probe.py --workload c3 --ns 128 --kernels 4 --no-torch --reps 5 2>&1 | grep -E "c3" | sed 's/torch\/cusparse 1000000000000.0us     0.0GF | //'
done
