timeout 300 python tools/probe.py --only powerlaw_s14_d16,powerlaw_s17_d16,uniform_s17_d16,powerlaw_s20_d16 --ns 32,64,128 --kernels 4 --no-torch 2>/dev/null
