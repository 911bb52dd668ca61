#!/bin/bash
# r2aa: P2P held back until P2M (1) or M2M (2) has finished (DAFMM_NEAR_AFTER): C4 / C3 / C5 A/B
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
rm -f gpurun_out/r2aa_probe.log
export PROBE_ROWS=0 PROBE_STEPS=30
for lib in libdafmm.so libdafmm_na1.so libdafmm_na2.so; do
  for c in c4 c3 c5; do
    DAFMM_LIB_NAME=$lib timeout 300 python tools/mode_probe.py $c '{}' >> gpurun_out/r2aa_probe.log 2>&1
  done
done
