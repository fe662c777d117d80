OUT=gpurun_out; mkdir -p $OUT
for v in cur sout; do
  LAGTRANS_B200_LIB=build/$v/liblagtrans_b200.so timeout 900 python bench.py --workload cfg5 --steps 10 --alt-steps 0 --e2e-steps 0 --no-cpu > $OUT/cfg5d_$v.log 2>&1
done
R=2 OUT=$OUT/ab_sout.txt ARGS="--precision fast" timeout 1200 bash tools/ab.sh cur sout > $OUT/ab_sout.log 2>&1
