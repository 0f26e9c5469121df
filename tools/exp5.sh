for fk in 256 512 1024 2048 8192; do SPHEMU_TRMM_FLUSH_K=$fk timeout 300 python tools/trmm_probe.py 4096 512 512; done
timeout 900 python -m pytest tests/test_gpu_emulate_chol.py -q -p no:cacheprovider 2>&1 | tail -15
