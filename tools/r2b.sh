OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x -k "hires or broadcast or sbr or cells or parity" > $OUT/pytest_gpu_new.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1
