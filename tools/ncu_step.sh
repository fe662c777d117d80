#!/bin/bash
# full ncu capture of the production step kernel, exact and fast precision
OUT=gpurun_out
for prec in exact fast; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 \
    -f -o $OUT/step_${prec} python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 0 --precision $prec \
    > $OUT/ncu_${prec}.log 2>&1
done
