for o in 0 1 33; do echo "opt $o C3"; SPHEMU_TC_OPT=$o timeout 300 python tools/ab.py 129600 dpsphp bf16 2; SPHEMU_TC_OPT=$o timeout 300 python tools/ab.py 64800 dpsphp bf16 2; done
echo "opt 33 C2"; SPHEMU_TC_OPT=33 timeout 300 python tools/ab.py 32400 dpsp fp16 3
