OUT=gpurun_out; mkdir -p $OUT
(cd .refsuite && PYTHONPATH=$PWD:$GRAFT_REPO_ROOT timeout 1800 python -m pytest tests -q -p no:cacheprovider -rfE > ../$OUT/r02_reference_suite.txt 2>&1)
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
