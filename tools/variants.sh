#!/bin/bash
# time the step kernel of several library builds on the same workload:
#   WL=cfg3 ARGS="--precision fast" tools/variants.sh base mb4 ...
# "base" is the in-tree library; other names are build/<name>/ (see _build.py --out).
WL=${WL:-cfg3}
for v in "$@"; do
  if [ "$v" = base ]; then lib=paper_2211_12616_b200/_lib/liblagtrans_b200.so; else lib=build/$v/liblagtrans_b200.so; fi
  LAGTRANS_B200_LIB=$lib python bench.py --workload $WL --steps 10 --no-cpu --e2e-steps 0 $ARGS 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v', '$ARGS', 'value %.3e'%d['value'], 'kernel_ms %.3f'%d['roofline']['kernel_ms'], 'ms/step %.3f'%d['ms_per_step'], d['clocks'])
    elif 'Error' in l or 'error' in l: print(l.strip())
"
done
