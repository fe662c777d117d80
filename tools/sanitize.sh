#!/bin/bash
# compute-sanitizer over the GPU suites (memcheck everywhere; racecheck where
# shared memory is used).  Output: gpurun_out/sanitizer.txt
OUT=gpurun_out; mkdir -p $OUT; F=$OUT/sanitizer.txt
: > $F
run() {  # tool, -k expression, files...
  local tool=$1 k=$2; shift 2
  echo "$tool: $* ${k:+-k \"$k\"}" >> $F
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest "$@" -m gpu -q -x \
    -p no:cacheprovider ${k:+-k "$k"} 2>&1 | grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Error" | tail -5 >> $F
  echo >> $F
}
run memcheck "" tests/test_gpu_parity.py tests/test_gpu_cells.py tests/test_gpu_edge.py tests/test_gpu_output.py
run memcheck "not 24h and not full_grid" tests/test_gpu_engine.py tests/test_gpu_runtime.py tests/test_gpu_acceptance.py tests/test_gpu_hires.py
run racecheck "" tests/test_gpu_output.py
