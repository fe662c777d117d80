OUT=gpurun_out; mkdir -p $OUT
R=3 OUT=$OUT/ab_pair.txt ARGS="--precision fast" timeout 1200 bash tools/ab.sh base0 pair > $OUT/ab_pair.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
