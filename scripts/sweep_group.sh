#!/usr/bin/env bash
# Group-size sweep of the ZNCC kernels (experiment; runs under gpurun).
for g in ${@:-4 6 8 10 12}; do
  VB_GROUP=$g python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernel_ms_per_step']
print('G=$g', round(d['value']), 'fps', 'zncc %.2f stats+mean %.2f' % (k['zncc_group'], k['other']))"
done
