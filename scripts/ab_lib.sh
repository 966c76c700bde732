#!/usr/bin/env bash
# A/B library builds (runs under gpurun): scripts/ab_lib.sh <lib.so> ...;
# CONFIGS="c2:4000 c3:2000" selects the workloads (default C2, 4000 frames).
for spec in ${CONFIGS:-c2:4000}; do
  cfg=${spec%%:*}; nfr=${spec##*:}
  for lib in "$@"; do
    VB_LIBRARY=$lib python bench.py --config $cfg --frames $nfr --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-dropin 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernel_ms_per_step']
print('$cfg', '$lib'.split('/')[-1], round(d['value']), 'fps', 'frac %.3f' % d['roofline']['frac'], ' '.join('%s %.3f' % (n, v) for n, v in k.items()))"
  done
done
