OUT=gpurun_out; mkdir -p $OUT
for v in r1 settle cur branchy; do
  lib=build/$v/liblagtrans_b200.so
  LAGTRANS_B200_LIB=$lib timeout 900 python bench.py --workload cfg5 --steps 10 --alt-steps 0 --e2e-steps 0 --no-cpu > $OUT/cfg5c_$v.log 2>&1
done
