#!/bin/bash
# compute-sanitizer over scripts/sanitize_c1.py (one GPU): memcheck, racecheck,
# synccheck, initcheck on the single-process workload; memcheck on the
# two-process CUDA-IPC exchange.  Summaries -> gpurun_out/sanitize_*.log
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # name, extra args...
  local name=$1; shift
  timeout 1500 $CS --print-limit 50 --error-exitcode 9 "$@" > gpurun_out/sanitize_$name.log 2>&1
  echo "$name rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$name.log >> gpurun_out/sanitize_summary.txt
}
: > gpurun_out/sanitize_summary.txt
run memcheck --tool memcheck python scripts/sanitize_c1.py
run racecheck --tool racecheck --racecheck-report analysis python scripts/sanitize_c1.py
run synccheck --tool synccheck python scripts/sanitize_c1.py
run initcheck --tool initcheck python scripts/sanitize_c1.py
run memcheck_ipc --tool memcheck --target-processes all python scripts/sanitize_c1.py --ipc
