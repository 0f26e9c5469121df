# C2 chain/bulk timeline after merging + tile-size sweep + panel/reserve A/B
set -x
timeout 300 python tools/timeline_gaps.py 32400 dpsp
timeout 300 python tools/chol_timeline.py 32400 512 dpsp > gpurun_out/tl_c2.txt; head -12 gpurun_out/tl_c2.txt
for t in 256 512 768 1024; do timeout 300 python tools/ab.py 32400 dpsp fp16 4 $t; done
SPHEMU_PANEL_F16X3=1 timeout 300 python tools/ab.py 32400 dpsp fp16 4
SPHEMU_RESERVE_EARLY=16 timeout 300 python tools/ab.py 32400 dpsp fp16 4
SPHEMU_RESERVE_TAIL=16 timeout 300 python tools/ab.py 32400 dpsp fp16 4
SPHEMU_RESERVE_TAIL=48 timeout 300 python tools/ab.py 32400 dpsp fp16 4
SPHEMU_MERGE=0 timeout 300 python tools/ab.py 32400 dpsp fp16 4
