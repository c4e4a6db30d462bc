# Shared-memory carveout of the smem-sized kernels: driver default (3 fresh processes, to
# see its variance) vs explicit percentages. Kernels: k_eb_sr_thr (EB+SR, N <= 4),
# k_eb_sr_cta (EB+SR, N >= 32), tile walk (RB+SR banded).
run() { timeout 600 python tools/probe.py --only uniform_s20_d16,powerlaw_s20_d16,banded_s20_b8 --ns 2,4,32,128 --kernels 0,4 --no-torch --reps 10 2>&1 | grep -E "s20"; }
for i in 1 2 3; do echo "== default $i"; run; done
for c in 25 50 100; do echo "== THR/CTA_CARVEOUT=$c"; DASPMM_THR_CARVEOUT=$c DASPMM_CTA_CARVEOUT=$c run; done
