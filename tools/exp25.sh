timeout 300 python tools/chol_timeline.py 32400 512 dpsp 2>/dev/null | head -9
for r in 8 16 24 32; do echo "early $r"; SPHEMU_RESERVE_EARLY=$r timeout 300 python tools/ab.py 32400 dpsp fp16 3; done
for t in 16 48 64; do echo "tail $t"; SPHEMU_RESERVE_TAIL=$t timeout 300 python tools/ab.py 32400 dpsp fp16 3; done
SPHEMU_MERGE=0 timeout 300 python tools/ab.py 32400 dpsp fp16 3
