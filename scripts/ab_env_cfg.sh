#!/usr/bin/env bash
# Experiment-build A/B on one config: scripts/ab_env_cfg.sh CONFIG FRAMES "ENV=.." "ENV=.." ...
export VB_LIBRARY=$PWD/paper_2403_16438_b200/libvoltb200_exp.so
cfg=$1; nfr=$2; shift 2
for envs in "$@"; do
  env $envs python bench.py --config $cfg --frames $nfr --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-dropin 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernel_ms_per_step']
print('$cfg', '$envs', round(d['value']), 'fps', 'frac %.3f' % d['roofline']['frac'], ' '.join('%s %.2f' % (n, v) for n, v in k.items()))"
done
