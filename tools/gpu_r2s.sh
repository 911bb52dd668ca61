#!/bin/bash
# r2s: warp-pair pair-stored M2L: polling vs sleeping mbarrier waits; ncu of the sleeping build
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
rm -f gpurun_out/r2s_probe.log
export PROBE_ROWS=0 PROBE_STEPS=20
for lib in libdafmm.so libdafmm_spin.so; do
  DAFMM_LIB_NAME=$lib timeout 200 python tools/mode_probe.py c4 '{"symmetric_pivots": 1, "m2l_store": 2}' >> gpurun_out/r2s_probe.log 2>&1
done
export DAFMM_OPTS=symmetric_pivots=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"m2l_pairw" -s 0 -c 1 \
  -o gpurun_out/r2s_pairw -f python tools/ncu_target.py c4 1 2 > gpurun_out/r2s_ncu.log 2>&1; echo "ncu rc=$?"
