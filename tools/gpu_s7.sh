for v in 0 1; do echo "== DASPMM_PDL=$v"; DASPMM_PDL=$v timeout 600 python tools/probe.py --only powerlaw_s14_d16,uniform_s14_d16,powerlaw_s17_d16,powerlaw_s20_d16 --ns 2,8,16,64 --kernels 4 --no-torch --reps 20 2>&1 | grep -v Warn | grep -v "At ="; done > gpurun_out/s7_pdl_probe.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s7_pytest.txt 2>&1; echo pytest rc=$?; tail -3 gpurun_out/s7_pytest.txt
cat gpurun_out/s7_pdl_probe.txt
