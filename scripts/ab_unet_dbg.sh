#!/usr/bin/env bash
# U-Net A/B of experiment switches (experiment build): bench line + per-layer launch times.
# Usage: scripts/ab_unet_dbg.sh "VB_UNET_THREADS=128" "VB_UNET_THREADS=288" ...
export VB_LIBRARY=$PWD/paper_2403_16438_b200/libvoltb200_exp.so
for envs in "$@"; do
  env $envs python bench.py --stage unet --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$envs', round(d['value']), d['ms_per_step'])"
done
if [ -n "$UNET_NCU" ]; then
for envs in "$@"; do
env $envs ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv3x3 -c 10 --csv --log-file "gpurun_out/unet_ab_$envs.csv" python bench.py --stage unet --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python - "$envs" <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/unet_ab_{sys.argv[1]}.csv")))
hdr, out = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        out.append(int(float(dict(zip(hdr, r))["Metric Value"]) / 1000))
print(sys.argv[1], "per-layer us", out, sum(out))
PY
done
fi
