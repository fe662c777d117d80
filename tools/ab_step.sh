# interleaved ms/step (sorts included) of library builds
for i in 1 2; do for v in "$@"; do
  if [ "$v" = base ]; then lib=paper_2211_12616_b200/_lib/liblagtrans_b200.so; else lib=build/$v/liblagtrans_b200.so; fi
  LAGTRANS_B200_LIB=$lib python bench.py --no-cpu --e2e-steps 0 --alt-steps 0 $ARGS 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('$v', 'ms/step %.3f'%d['ms_per_step'], 'kernel %.3f'%d['roofline']['kernel_ms'])
"; done; done
