# c1 (uniform 4096^2, 1%, N = 32): every design point, and the RB+RM+SR knobs, against
# the 5.7 us empty-launch floor of the same protocol.
P="python tools/probe.py --workload c1 --ns 32 --no-torch --reps 20"
echo "== all design points"; $P --kernels 0,1,2,3,4,5,6,7 2>/dev/null
for r in 1 2 4 8; do echo "== DASPMM_RPG=$r"; DASPMM_RPG=$r $P --kernels 0 2>/dev/null; done
for t in 64 256; do echo "== DASPMM_RB_THREADS=$t"; DASPMM_RB_THREADS=$t $P --kernels 0 2>/dev/null; done
echo "== DASPMM_LEAN_RB=1"; DASPMM_LEAN_RB=1 $P --kernels 0 2>/dev/null
echo "== DASPMM_EB_CTA=0"; DASPMM_EB_CTA=0 $P --kernels 4 2>/dev/null
for c in 32 64 128; do echo "== DASPMM_LEAN_CHUNK=$c"; DASPMM_LEAN_CHUNK=$c $P --kernels 4 2>/dev/null; done
