#!/usr/bin/env bash
# A/B two library builds (libvoltb200_<tag>.so) on several configs (runs under gpurun).
for v in "$@"; do
  cp paper_2403_16438_b200/libvoltb200_$v.so paper_2403_16438_b200/libvoltb200.so
  for spec in "c2 4000" "c3 2000" "c5 1000"; do
    set -- $spec
    python bench.py --config $1 --frames $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernel_ms_per_step']
print('$v', '$1', round(d['value']), 'fps', 'frac %.3f' % d['roofline']['frac'], 'zncc %.2f' % k['zncc_group'])"
  done
done
