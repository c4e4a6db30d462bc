# usage: tools/prof_one.sh <kernel-regex> <matrix> <N> <kernel-id> <tag> [workload]
f=/tmp/prof_$5
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$1<" -s 2 -c 1 -o $f python tools/probe.py --workload ${6:-suite} --only $2 --ns $3 --kernels $4 --no-torch --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py $f.ncu-rep --lines 30 > gpurun_out/ncu_$5.txt 2>&1
