#!/bin/bash
# Memory check of every kernel at small sizes (run under gpurun from the repo root).
# compute-sanitizer is closed on this pool ("runs under it have left GPUs needing
# a reset"), so this is the library's guard-band mode (PASD_B200_GUARD=1, see
# tools/sanitize_run.py); summary to gpurun_out/san_guard.txt.
mkdir -p gpurun_out
start=$(date +%s)
PASD_B200_GUARD=1 timeout 900 python tools/sanitize_run.py > gpurun_out/san_guard.log 2>&1
rc=$?
{ echo "# PASD_B200_GUARD=1 python tools/sanitize_run.py"
  echo "# exit $rc after $(( $(date +%s) - start )) s"
  grep -E "guard|iters|sanitize_run done|Error|error" gpurun_out/san_guard.log | head -60
} > gpurun_out/san_guard.txt
echo "guard rc=$rc"
