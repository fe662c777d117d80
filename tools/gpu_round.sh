#!/bin/bash
# One evidence pass on a gpurun box (round 2): smoke, GPU tests, the bench
# line, the other BASELINE workloads, fast-vs-exact error distribution, the
# ncu launch list and full captures of the step kernel (both precisions).
# Everything lands in gpurun_out/ (copy what is judged into profiles/).
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1
timeout 900 python bench.py ${BENCH_ARGS} > $OUT/bench.log 2>&1
if [ -z "$NO_WORKLOADS" ]; then
  for wl in cfg1 cfg2 cfg4; do
    timeout 900 python bench.py --workload $wl > $OUT/bench_$wl.log 2>&1
  done
  timeout 1500 python bench.py --workload cfg5 --steps 10 --alt-steps 10 --e2e-steps 1 > $OUT/bench_cfg5.log 2>&1
fi
for r in counter philox; do timeout 600 python tools/fast_error.py $r cfg3 >> $OUT/fast_error.log 2>&1; done
if [ -z "$NO_NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 14 --warmup 3 --no-cpu --e2e-steps 0 --alt-steps 0 > $OUT/ncu_launch_run.log 2>&1
  for prec in fast exact; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 \
      -f -o $OUT/step_${prec} python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 0 --alt-steps 0 \
      --precision $prec > $OUT/ncu_${prec}.log 2>&1
  done
fi
ls -la $OUT
