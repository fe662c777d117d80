#!/bin/bash
# interleaved A/B timing of library builds (min and median kernel ms over R
# rounds): R=3 WL=cfg3 ARGS="--precision fast" tools/ab.sh base mb4 ...
WL=${WL:-cfg3}; R=${R:-3}
OUT=${OUT:-gpurun_out/ab.txt}; mkdir -p $(dirname $OUT); : > $OUT
for i in $(seq $R); do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=paper_2211_12616_b200/_lib/liblagtrans_b200.so; else lib=build/$v/liblagtrans_b200.so; fi
    LAGTRANS_B200_LIB=$lib python bench.py --workload $WL --steps 10 --no-cpu --e2e-steps 0 --alt-steps 0 $ARGS 2>&1 |
      python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): print('$v', json.loads(l)['roofline']['kernel_ms'])
" >> $OUT
  done
done
python - "$OUT" <<'PY'
import sys, collections, statistics
d = collections.defaultdict(list)
for l in open(sys.argv[1]):
    v, t = l.split(); d[v].append(float(t))
for v, ts in d.items():
    print(f"{v:12s} min {min(ts):.3f} median {statistics.median(ts):.3f} all {' '.join(f'{t:.3f}' for t in ts)}")
PY
