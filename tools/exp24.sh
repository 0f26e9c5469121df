for cg in 1 2; do
SPHEMU_TC_CG_SP=$cg timeout 300 python tools/ab.py 32400 dpsp fp16 4
SPHEMU_TC_CG_SP=$cg timeout 300 python tools/ab.py 129600 dpsphp bf16 2
SPHEMU_TC_CG_SP=$cg timeout 300 python tools/ab.py 64800 dpsp fp16 2
done
SPHEMU_TC_CG_SP=2 SPHEMU_YIELD=0 timeout 300 python tools/ab.py 32400 dpsp fp16 4
SPHEMU_TC_CG_SP=2 timeout 300 python tools/timeline_gaps.py 32400 dpsp
SPHEMU_TC_CG_SP=2 timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
