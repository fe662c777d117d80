OUT=gpurun_out; mkdir -p $OUT
R=2 OUT=$OUT/ab_cb.txt ARGS="--precision exact" timeout 1200 bash tools/ab.sh base nowalk cur > $OUT/ab_cb.log 2>&1
R=2 OUT=$OUT/ab_cb_ctr.txt ARGS="--precision exact --rng counter" timeout 1200 bash tools/ab.sh base nowalk cur > $OUT/ab_cb_ctr.log 2>&1
R=2 OUT=$OUT/ab_cb_fast.txt ARGS="--precision fast" timeout 1200 bash tools/ab.sh base cur > $OUT/ab_cb_fast.log 2>&1
for v in base cur; do
  if [ "$v" = base ]; then lib=paper_2211_12616_b200/_lib/liblagtrans_b200.so; else lib=build/$v/liblagtrans_b200.so; fi
  LAGTRANS_B200_LIB=$lib timeout 900 python bench.py --workload cfg5 --steps 10 --alt-steps 0 --e2e-steps 0 --no-cpu > $OUT/cfg5b_$v.log 2>&1
done
