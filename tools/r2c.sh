OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
R=3 OUT=$OUT/ab_blocks.txt ARGS="--precision fast" timeout 1200 bash tools/ab.sh base b128m9 b128m10 b64m18 > $OUT/ab_blocks.log 2>&1
timeout 900 python bench.py > $OUT/bench.log 2>&1
timeout 900 python bench.py --gpus 2 --steps 10 > $OUT/bench_g2.log 2>&1
timeout 900 python bench.py --impl reference --steps 10 > $OUT/bench_ref.log 2>&1
