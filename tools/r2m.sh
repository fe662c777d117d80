OUT=gpurun_out; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
R=2 OUT=$OUT/ab_tx.txt ARGS="--precision exact" timeout 1200 bash tools/ab.sh prev base > $OUT/ab_tx.log 2>&1
R=2 OUT=$OUT/ab_tx_ctr.txt ARGS="--precision exact --rng counter" timeout 1200 bash tools/ab.sh prev base > $OUT/ab_tx_ctr.log 2>&1
