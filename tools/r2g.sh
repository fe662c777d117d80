OUT=gpurun_out; mkdir -p $OUT
R=3 OUT=$OUT/ab_fast3.txt ARGS="--precision fast" timeout 1200 bash tools/ab.sh one nb nb2 > $OUT/ab_fast3.log 2>&1
R=2 OUT=$OUT/ab_fast3_ctr.txt ARGS="--precision fast --rng counter" timeout 1200 bash tools/ab.sh one nb2 > $OUT/ab_fast3_ctr.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
