OUT=gpurun_out; mkdir -p $OUT
R=3 OUT=$OUT/ab_levc.txt ARGS="--precision fast" timeout 1200 bash tools/ab.sh base levc > $OUT/ab_levc.log 2>&1
R=2 OUT=$OUT/ab_levc_ctr.txt ARGS="--precision fast --rng counter" timeout 1200 bash tools/ab.sh base levc > $OUT/ab_levc_ctr.log 2>&1
