./tools/micro/pc_pieces
timeout 60 ./tools/micro/potrf_trace | head -8
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or potrf or chol" 2>&1 | tail -2
timeout 300 python tools/ab.py 32400 dpsp fp16 3
timeout 300 python tools/ab.py 129600 dpsphp bf16 2
timeout 300 python tools/chol_timeline.py 32400 512 dpsp 2>/dev/null | head -9
