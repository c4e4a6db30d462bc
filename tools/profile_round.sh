#!/bin/bash
# Profile artifacts for one round (run under gpurun from the repo root):
#   gpurun_out/launches_<tag>.csv      ncu launch list of the bench command (cold, serialised)
#   gpurun_out/ncu_<tag>_<case>.txt    ncu --set full summaries of the top kernels
#   gpurun_out/ncu_<tag>_traffic.json  DRAM bytes per launch of those kernels
# usage: tools/profile_round.sh r01 [full]   (launch list only unless "full")
set -u
tag=${1:-r01}
out=gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $out/launches_$tag.csv \
    python bench.py --steps 1 --warmup 3 --profile-step > $out/bench_under_ncu_$tag.json 2>&1
[ "${2:-}" = "full" ] || exit 0
echo "{" > $out/ncu_${tag}_traffic.json
first=1
# kernel-regex  matrix  N  kernel-id  [workload]
for spec in "k_rb_sr uniform_s20_d16 128 0" "k_eb_sr_cta powerlaw_s20_d16 128 4" \
            "k_eb_sr_lean_rw powerlaw_s20_d16 16 4" "k_eb_sr_thr uniform_s20_d16 2 4" \
            "k_rb_sr uniform_s20_d16 16 0" "k_eb_sr_lean c3_reddit_like 128 4 c3" \
            "k_eb_prep_uniform powerlaw_s20_d16 64 4" "k_rb_sr_tile banded_s20_b8 128 0" \
            "k_rb_sr_tile_direct banded_s20_b8 16 0" "k_rb_cm_rows banded_s20_b8 32 2"; do
  set -- $spec
  wl=${5:-suite}
  case_name="$2/N$3"
  f=/tmp/prof_${tag}_$1_$2_$3
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$1<" -s 2 -c 1 -o $f \
      python tools/probe.py --workload $wl --only $2 --ns $3 --kernels $4 --no-torch --reps 1 > /dev/null 2>&1
  python tools/ncu_summary.py $f.ncu-rep --lines 16 > $out/ncu_${tag}_$1_$2_N$3.txt 2>&1
  bytes=$(ncu -i $f.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; u=r[1]; v=r[2]
def get(k):
    i=h.index(k); x=float(v[i]); s={'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}.get(u[i],1); return x*s
print(int(get('dram__bytes_read.sum')+get('dram__bytes_write.sum')))" 2>/dev/null || echo null)
  [ $first -eq 1 ] || echo "," >> $out/ncu_${tag}_traffic.json
  first=0
  printf '  "%s": %s' "$case_name" "$bytes" >> $out/ncu_${tag}_traffic.json
done
echo "" >> $out/ncu_${tag}_traffic.json
echo "}" >> $out/ncu_${tag}_traffic.json
ls -la $out
