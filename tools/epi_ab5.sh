for d in 1 3 4 5; do SPHEMU_TC_DBG=$d SPHEMU_TC_CG=2 python tools/epi_probe.py 98304 dpsphp bf16; done
for d in 3 4 5; do SPHEMU_TC_DBG=$d python tools/epi_probe.py 32400 dpsp fp16; done
