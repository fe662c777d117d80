OUT=gpurun_out; mkdir -p $OUT
R=2 OUT=$OUT/ab_ex3b.txt ARGS="--precision exact" timeout 1200 bash tools/ab.sh base ex3 > $OUT/ab_ex3b.log 2>&1
R=2 OUT=$OUT/ab_ex3b_ctr.txt ARGS="--precision exact --rng counter" timeout 1200 bash tools/ab.sh base ex3 > $OUT/ab_ex3b_ctr.log 2>&1
