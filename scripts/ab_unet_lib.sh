for lib in "$@"; do
  VB_LIBRARY=$lib python bench.py --stage unet --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib'.split('/')[-1], round(d['value']), d['ms_per_step'])"
done
