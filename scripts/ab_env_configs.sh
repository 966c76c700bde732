#!/usr/bin/env bash
# A/B env knobs across configs (runs under gpurun).  Usage: ab_env_configs.sh "ENV=.." ...
for envs in "$@"; do
  for spec in "c2 4000" "c3 2000" "c5 1000"; do
    set -- $spec
    env $envs python bench.py --config $1 --frames $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernel_ms_per_step']
print('$envs', '$1', round(d['value']), 'frac %.3f' % d['roofline']['frac'], 'zncc %.2f' % k['zncc_group'])"
  done
done
