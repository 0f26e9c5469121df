timeout 900 python tools/oz_check.py 4096 512 2>&1 | tail -12
SPHEMU_TC_CG_SP=2 timeout 300 python tools/ab.py 32400 dpsp fp16 4
timeout 300 python tools/ab.py 32400 dpsp fp16 4
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
