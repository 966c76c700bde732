#!/usr/bin/env bash
# GPU-side profiling recipe (runs under gpurun).  Usage: scripts/gpu_profile.sh TAG
# Then here: python scripts/make_profiles.py TAG
set -u
TAG=${1:-r01}
OUT=gpurun_out
CMD="python bench.py --frames 2000 --steps 2 --warmup 1 --no-e2e --no-dropin --no-cpu-baseline"
$CMD > $OUT/prof_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
$CMD > $OUT/prof_plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"zncc|smooth|correct_rows|median|block_mean" -s 6 -c 6 \
    -o $OUT/prof_$TAG -f $CMD > $OUT/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
