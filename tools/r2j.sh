OUT=gpurun_out; mkdir -p $OUT
if [ -d .refsuite ]; then
  (cd .refsuite && PYTHONPATH=$PWD:$GRAFT_REPO_ROOT timeout 1800 python -m pytest tests -q -p no:cacheprovider -rfE > ../$OUT/r02_reference_suite.txt 2>&1)
else
  echo "no .refsuite staged" > $OUT/r02_reference_suite.txt
fi
