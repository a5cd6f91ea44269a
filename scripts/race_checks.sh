#!/bin/bash
# Race evidence for the lock-free claim / steal / publish / pop protocol.
# Run on a GPU box from the repo root; logs go to gpurun_out/ (summaries are copied to profiles/).
#   1. compute-sanitizer memcheck and synccheck over scripts/sanitize_run.py (C1 + random graphs,
#      steal-one / steal-half / deferred check / small launch / shared counter with overflow relaunch)
#   2. a race-stress build (MBE_DEBUG_DELAYS=1: random __nanosleep at every synchronisation point)
#      running the same workload many times, every result compared with the oracle
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
G=${SAN_GRAPHS:-50}
for tool in memcheck synccheck; do
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
    python scripts/sanitize_run.py --graphs $G > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
done
bash scripts/build_variant.sh delays MBE_DEBUG_DELAYS=1 > /dev/null
MBE_LIB_PATH=variants/delays.so timeout 2400 python scripts/sanitize_run.py --graphs ${STRESS_GRAPHS:-200} \
  --reps ${STRESS_REPS:-5} > gpurun_out/stress_delays.log 2>&1
echo "stress rc=$?" >> gpurun_out/sanitize_summary.txt
tail -2 gpurun_out/sanitize_*.log gpurun_out/stress_delays.log
