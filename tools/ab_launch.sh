#!/bin/bash
# A/B: per-kernel launch times (ncu gpu__time_duration, serialised) and a short bench for each
# library named on the command line (DAFMM_LIB_NAME).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=$1; shift
for LIBN in "$@"; do
  export DAFMM_LIB_NAME=$LIBN
  timeout 600 python bench.py --no-gmres --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/ab_${TAG}_${LIBN}.json 2>&1
  python tools/ncu_target.py c4 3 > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_${TAG}_${LIBN}.csv \
      python tools/ncu_target.py c4 3 > /dev/null 2>&1
done
echo done
