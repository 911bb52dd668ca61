#!/bin/bash
# compute-sanitizer memcheck and racecheck on the small target (default path, pair-stored M2L, hybrid solver)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python tools/sanitize_target.py > gpurun_out/sanitize_plain_r2.log 2>&1; echo "plain rc=$?"
for TOOL in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $TOOL --error-exitcode 3 python tools/sanitize_target.py > gpurun_out/sanitize_${TOOL}_r2.log 2>&1; echo "$TOOL rc=$?"
done
