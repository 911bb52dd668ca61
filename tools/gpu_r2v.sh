#!/bin/bash
# r2v: ncu of the column-major translation kernel at C4 (7 launches of one matvec)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"translate" -s 0 -c 7 \
  -o gpurun_out/r2v_translate -f python tools/ncu_target.py c4 1 > gpurun_out/r2v_ncu.log 2>&1; echo "ncu rc=$?"
