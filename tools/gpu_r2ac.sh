#!/bin/bash
# r2ac: P2P register cap 88 (two P2P CTAs + two stored-M2L CTAs fill the register file exactly) vs 80
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
rm -f gpurun_out/r2ac_probe.log
export PROBE_ROWS=0 PROBE_STEPS=30
for lib in libdafmm.so libdafmm_p88.so; do
  for c in c4 c3 c5; do
    DAFMM_LIB_NAME=$lib timeout 300 python tools/mode_probe.py $c '{}' >> gpurun_out/r2ac_probe.log 2>&1
  done
done
