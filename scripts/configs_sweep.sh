#!/usr/bin/env bash
# Stage throughput on every BASELINE.json config (shortened recordings; runs under gpurun):
# device frames/s, search-kernel FP32 fraction, per-kernel ms per step, and the C-ABI host-to-host e2e.
for spec in "c1 1000" "c2 4000" "c3 2000" "c4 2048" "c5 1000"; do
  set -- $spec
  python bench.py --config $1 --frames $2 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernel_ms_per_step']
print(json.dumps({'config': '$1', 'workload': d['config']['workload'], 'fps': round(d['value']), 'e2e_fps': round(d['e2e']['value']), 'dropin_fps': round(d['e2e_dropin']['value']),
  'frac': round(d['roofline']['frac'], 3), 'kernel': d['roofline']['kernel'], 'ms_per_step': {n: round(v, 3) for n, v in k.items()}}))"
done
