# INT8-emulated DP updates: correctness vs DMMA, then C2/C3 timings both ways
timeout 900 python tools/oz_check.py 4096 512 2>&1 | tail -20
timeout 300 python tools/ab.py 32400 dpsp fp16 4
SPHEMU_DP_EMU=0 timeout 300 python tools/ab.py 32400 dpsp fp16 4
timeout 300 python tools/timeline_gaps.py 32400 dpsp
timeout 300 python tools/chol_timeline.py 32400 512 dpsp | head -8
timeout 300 python tools/ab.py 129600 dpsphp bf16 2
timeout 300 python tools/ab.py 32400 dp fp16 2
SPHEMU_DP_EMU=0 timeout 300 python tools/ab.py 32400 dp fp16 2
