for d in 0 1 3 4; do SPHEMU_TC_DBG=$d python tools/epi_probe.py 98304 dpsphp bf16; done
for d in 0 1; do SPHEMU_TC_CG=2 SPHEMU_TC_DBG=$d python tools/epi_probe.py 98304 dpsphp bf16; done
for d in 0 1 3 4; do SPHEMU_TC_DBG=$d python tools/epi_probe.py 32400 dpsp fp16; done
