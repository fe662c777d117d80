OUT=gpurun_out; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q -x -k "sort or permutation or cells or box" > $OUT/pytest_keys.log 2>&1
bash tools/sanitize.sh
R=2 OUT=$OUT/ab_keys.txt ARGS="--precision fast" timeout 1200 bash tools/ab.sh sout fkeys > $OUT/ab_keys.log 2>&1
