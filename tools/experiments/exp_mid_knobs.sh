# Re-tune after the quad-per-iteration EB walks: lean EB chunk / walk kind for power-law
# s20 N = 8, 16, 32 (k4), and RB rows per group / CTA size for uniform s20 N = 8, 16, 32 (k0).
P="python tools/probe.py --workload suite --no-torch --reps 10"
echo "== power-law s20, EB+RM+SR: default"
$P --only powerlaw_s20_d16 --ns 8,16,32 --kernels 4 2>/dev/null
for rw in 0 1; do for c in 64 128 256 512; do
  echo "== power-law s20 DASPMM_LEAN_RW=$rw DASPMM_LEAN_CHUNK=$c"
  DASPMM_LEAN_RW=$rw DASPMM_LEAN_CHUNK=$c $P --only powerlaw_s20_d16 --ns 8,16,32 --kernels 4 2>/dev/null
done; done
echo "== uniform s20, RB+RM+SR: default"
$P --only uniform_s20_d16 --ns 8,16,32 --kernels 0 2>/dev/null
for r in 1 2 4; do
  echo "== uniform s20 DASPMM_RPG=$r"
  DASPMM_RPG=$r $P --only uniform_s20_d16 --ns 8,16,32 --kernels 0 2>/dev/null
done
for t in 64 256; do
  echo "== uniform s20 DASPMM_RB_THREADS=$t"
  DASPMM_RB_THREADS=$t $P --only uniform_s20_d16 --ns 8,16,32 --kernels 0 2>/dev/null
done
echo "== uniform s20 DASPMM_LEAN_RB=1"
DASPMM_LEAN_RB=1 $P --only uniform_s20_d16 --ns 8,16,32 --kernels 0 2>/dev/null
