for pd in 0 1; do for r in 8 16; do echo "pair_dyn $pd reserve $r"; SPHEMU_TC_PAIR_DYN=$pd SPHEMU_RESERVE_EARLY=$r timeout 300 python tools/ab.py 32400 dpsp fp16 3; done; done
for pd in 0 1 2; do echo "pair_dyn $pd"; SPHEMU_TC_PAIR_DYN=$pd timeout 300 python tools/ab.py 129600 dpsphp bf16 2; SPHEMU_TC_PAIR_DYN=$pd timeout 300 python tools/ab.py 64800 dpsp fp16 2; done
SPHEMU_TC_PAIR_DYN=1 timeout 300 python tools/chol_timeline.py 32400 512 dpsp 2>/dev/null | head -9
