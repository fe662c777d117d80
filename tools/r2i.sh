OUT=gpurun_out; mkdir -p $OUT
R=2 OUT=$OUT/ab_exact4.txt ARGS="--precision exact" timeout 1200 bash tools/ab.sh base ex3 ex2 > $OUT/ab_exact4.log 2>&1
R=2 OUT=$OUT/ab_exact4_ctr.txt ARGS="--precision exact --rng counter" timeout 1200 bash tools/ab.sh base ex3 ex2 > $OUT/ab_exact4_ctr.log 2>&1
if [ -d .refsuite ]; then
  (cd .refsuite && PYTHONPATH=$PWD:$GRAFT_REPO_ROOT timeout 1800 python -m pytest tests -q -p no:cacheprovider -rf > ../$OUT/r02_reference_suite.txt 2>&1)
fi
