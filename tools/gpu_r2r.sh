#!/bin/bash
# r2r: ncu of the warp-pair pair-stored M2L at C4 (source-level stalls)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export DAFMM_OPTS=symmetric_pivots=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"m2l_pairw" -s 0 -c 1 \
  -o gpurun_out/r2r_pairw -f python tools/ncu_target.py c4 1 2 > gpurun_out/r2r_ncu.log 2>&1; echo "ncu rc=$?"
