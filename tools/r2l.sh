OUT=gpurun_out; mkdir -p $OUT
R=2 OUT=$OUT/ab_probe.txt ARGS="--precision fast" timeout 1200 bash tools/ab.sh base probe_norng > $OUT/ab_probe.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
