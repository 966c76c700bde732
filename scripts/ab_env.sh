#!/usr/bin/env bash
# A/B of experiment knobs on the short bench (runs under gpurun).
# Usage: scripts/ab_env.sh "VB_FPI=1" "VB_FPI=2" ...
for envs in "$@"; do
  env $envs python bench.py --frames 4000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernel_ms_per_step']
print('$envs', round(d['value']), 'fps', ' '.join('%s %.2f' % (n, v) for n, v in k.items()), 'frac %.3f' % d['roofline']['frac'])"
done
