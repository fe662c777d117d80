OUT=gpurun_out; mkdir -p $OUT
R=2 OUT=$OUT/ab_plev.txt ARGS="--precision fast" timeout 1200 bash tools/ab.sh base probe_lev > $OUT/ab_plev.log 2>&1
