f=/tmp/prof_u32
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_rb_sr<" -s 2 -c 1 -o $f python tools/probe.py --only uniform_s20_d16 --ns 32 --kernels 0 --no-torch --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py $f.ncu-rep --lines 25 > gpurun_out/ncu_u32.txt 2>&1
f=/tmp/prof_p32
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_eb_sr_lean_rw<" -s 2 -c 1 -o $f python tools/probe.py --only powerlaw_s20_d16 --ns 32 --kernels 4 --no-torch --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py $f.ncu-rep --lines 25 > gpurun_out/ncu_p32.txt 2>&1
