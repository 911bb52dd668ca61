#!/bin/bash
# r2t: L2 prefetch of the operator rows in the translation kernels (DAFMM_TPF rows ahead): C4 A/B
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
rm -f gpurun_out/r2t_probe.log
export PROBE_ROWS=64 PROBE_STEPS=30
for lib in libdafmm.so libdafmm_tpf0.so libdafmm_tpf16.so; do
  DAFMM_LIB_NAME=$lib timeout 200 python tools/mode_probe.py c4 '{}' >> gpurun_out/r2t_probe.log 2>&1
done
