OUT=gpurun_out; mkdir -p $OUT
timeout 1800 python -m pytest tests/test_gpu_multirank.py -q -x > $OUT/pytest_multirank.log 2>&1
