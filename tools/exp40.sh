for o in 0 4 16 32 1; do echo "opt $o"; SPHEMU_TC_OPT=$o timeout 300 python tools/ab.py 32400 dpsp fp16 3; SPHEMU_TC_OPT=$o timeout 300 python tools/ab.py 64800 dpsp fp16 2; done
for o in 0 16; do echo "opt $o C3"; SPHEMU_TC_OPT=$o timeout 300 python tools/ab.py 129600 dpsphp bf16 2; done
