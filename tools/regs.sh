#!/bin/bash
# Per-kernel registers / spills for one TU: tools/regs.sh spmm_rb_sr.cu [filter]
f=$1; flt=${2:-.}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v -c /root/repo/paper_2202_08556_b200/csrc/$f -o /tmp/regs.o 2>&1 \
 | awk '/Compiling entry function/ {match($0, /_Z[^'"'"']*/); name=substr($0, RSTART, RLENGTH)} /spill stores/ {sp=$0} /Used [0-9]+ registers/ {match($0,/Used [0-9]+ registers/); print name, substr($0,RSTART,RLENGTH), sp}' \
 | c++filt | sed 's/daspmm:://g; s/(SpmmArgs<float>)//; s/(SpmmArgs<double>)//; s/ptxas info    ://' | grep -E "$flt"
