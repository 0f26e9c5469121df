for t in 512 768 1024; do timeout 300 python tools/ab.py 32400 dpsp fp16 3 $t; done
timeout 300 python tools/chol_timeline.py 32400 512 dpsp 2>/dev/null | head -9
timeout 300 python tools/timeline_gaps.py 32400 dpsp
for r in 8 12 16; do echo "reserve $r"; SPHEMU_RESERVE_EARLY=$r timeout 300 python tools/ab.py 32400 dpsp fp16 3; done
