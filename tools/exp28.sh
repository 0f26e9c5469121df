timeout 300 python tools/ab.py 32400 dpsp fp16 4
timeout 300 python tools/ab.py 129600 dpsphp bf16 2
SPHEMU_RESERVE_EARLY=8 timeout 300 python tools/ab.py 129600 dpsphp bf16 2
timeout 300 python tools/ab.py 64800 dpsp fp16 2
timeout 300 python tools/chol_timeline.py 32400 512 dpsp 2>/dev/null | head -9
timeout 300 python tools/timeline_gaps.py 32400 dpsp
