#!/usr/bin/env bash
# Focused ncu capture of one kernel (regex $2) of the short bench command.  Usage: TAG REGEX
set -u
TAG=$1; RE=$2
CMD="python bench.py --frames 2000 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof1_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$RE" -s 2 -c 1 -o gpurun_out/prof1_$TAG -f $CMD > gpurun_out/ncu1_$TAG.log 2>&1
echo "rc=$?"
