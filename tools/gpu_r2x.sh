#!/bin/bash
# r2x: stored-M2L CTAs per SM at C5 (P2P is the critical path there) and C4
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
rm -f gpurun_out/r2x_probe.log
export PROBE_ROWS=0 PROBE_STEPS=20
for k in 2 1 3; do
  echo "== DAFMM_MS_PER_SM_RT=$k" >> gpurun_out/r2x_probe.log
  DAFMM_MS_PER_SM_RT=$k timeout 300 python tools/mode_probe.py c5 '{}' >> gpurun_out/r2x_probe.log 2>&1
done
for k in 2 1; do
  echo "== DAFMM_MS_PER_SM_RT=$k" >> gpurun_out/r2x_probe.log
  DAFMM_MS_PER_SM_RT=$k timeout 300 python tools/mode_probe.py c3 '{}' >> gpurun_out/r2x_probe.log 2>&1
done
