OUT=gpurun_out; mkdir -p $OUT
R=2 OUT=$OUT/ab_walk.txt ARGS="--precision exact" timeout 1200 bash tools/ab.sh base walk > $OUT/ab_walk.log 2>&1
R=2 OUT=$OUT/ab_walk_ctr.txt ARGS="--precision exact --rng counter" timeout 1200 bash tools/ab.sh base walk > $OUT/ab_walk_ctr.log 2>&1
for v in base r1; do
  if [ "$v" = base ]; then lib=paper_2211_12616_b200/_lib/liblagtrans_b200.so; else lib=build/$v/liblagtrans_b200.so; fi
  LAGTRANS_B200_LIB=$lib timeout 900 python bench.py --workload cfg5 --steps 10 --alt-steps 0 --e2e-steps 0 --no-cpu > $OUT/cfg5_$v.log 2>&1
done
