for lib in "$@"; do
  VB_LIBRARY=$lib python bench.py --frames 4000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-dropin 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernel_ms_per_step']
print('$lib'.split('/')[-1], round(d['value']), 'fps', ' '.join('%s %.3f' % (n, v) for n, v in k.items()))"
done
