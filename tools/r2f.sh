OUT=gpurun_out; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
R=2 OUT=$OUT/ab_exact2.txt ARGS="--precision exact" timeout 1200 bash tools/ab.sh mk one > $OUT/ab_exact2.log 2>&1
R=2 OUT=$OUT/ab_exact2_ctr.txt ARGS="--precision exact --rng counter" timeout 1200 bash tools/ab.sh mk one > $OUT/ab_exact2_ctr.log 2>&1
R=2 OUT=$OUT/ab_fast2.txt ARGS="--precision fast" timeout 1200 bash tools/ab.sh mk one > $OUT/ab_fast2.log 2>&1
