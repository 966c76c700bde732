#!/usr/bin/env bash
# A/B of experiment switches on the short bench (runs under gpurun).  The
# switches are read only by the experiment build (build.py --experiments).
# Usage: scripts/ab_env.sh "VB_FPI=1" "VB_FPI=2" ...
python -m paper_2403_16438_b200.build --experiments > /dev/null 2>&1
export VB_LIBRARY=$PWD/paper_2403_16438_b200/libvoltb200_exp.so
for envs in "$@"; do
  env $envs python bench.py --frames 4000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-dropin 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernel_ms_per_step']
print('$envs', round(d['value']), 'fps', ' '.join('%s %.2f' % (n, v) for n, v in k.items()), 'frac %.3f' % d['roofline']['frac'])"
done
