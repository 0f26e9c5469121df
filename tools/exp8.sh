timeout 1500 python -m pytest tests/test_gpu_pipeline.py -q -p no:cacheprovider -x 2>&1 | tail -25
