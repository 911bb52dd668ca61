#!/bin/bash
# compute-sanitizer (one tool per call) on the small sanitizer target, then a bench run.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-rXX}
TOOL=${2:-memcheck}
python tools/sanitize_target.py > gpurun_out/sanitize_plain_$TAG.log 2>&1 && \
timeout 900 compute-sanitizer --tool $TOOL --error-exitcode 3 python tools/sanitize_target.py > gpurun_out/sanitize_${TOOL}_$TAG.log 2>&1; echo "sanitize rc=$?"
timeout 900 python bench.py --no-gmres > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
