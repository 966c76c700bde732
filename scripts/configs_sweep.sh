#!/usr/bin/env bash
# Stage throughput on every BASELINE.json config (shortened recordings; runs under gpurun).
for spec in "c1 1000" "c2 4000" "c3 2000" "c4 2048" "c5 1000"; do
  set -- $spec
  python bench.py --config $1 --frames $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernel_ms_per_step']
print('$1', d['config']['workload'][:60], round(d['value']), 'fps', 'frac %.3f' % d['roofline']['frac'], d['roofline']['plan'], ' '.join('%s %.2f' % (n, v) for n, v in k.items()))"
done
