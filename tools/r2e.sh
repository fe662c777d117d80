OUT=gpurun_out; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
R=3 OUT=$OUT/ab_exact.txt ARGS="--precision exact" timeout 1200 bash tools/ab.sh base0 mk > $OUT/ab_exact.log 2>&1
R=2 OUT=$OUT/ab_exact64.txt ARGS="--precision exact --met-store f64" timeout 1200 bash tools/ab.sh mk > $OUT/ab_exact64.log 2>&1
R=2 OUT=$OUT/ab_exact_ctr.txt ARGS="--precision exact --rng counter" timeout 1200 bash tools/ab.sh base0 mk > $OUT/ab_exact_ctr.log 2>&1
