OUT=gpurun_out; mkdir -p $OUT
R=3 OUT=$OUT/ab_exact3.txt ARGS="--precision exact" timeout 1200 bash tools/ab.sh nb2 enb > $OUT/ab_exact3.log 2>&1
R=2 OUT=$OUT/ab_exact3_ctr.txt ARGS="--precision exact --rng counter" timeout 1200 bash tools/ab.sh nb2 enb > $OUT/ab_exact3_ctr.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
for prec in fast exact; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 \
    -f -o $OUT/r02_step_${prec} python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 0 --alt-steps 0 \
    --precision $prec > $OUT/ncu_${prec}.log 2>&1
done
