#!/bin/bash
# r2p: M2M on a side stream beside the deepest level's stored M2L (flag handshake): C4 A/B against the
# serial far chain, parity of the default path, C3/C5 A/B
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
rm -f gpurun_out/r2p_probe.log
export PROBE_ROWS=64 PROBE_STEPS=30
for lib in libdafmm.so libdafmm_noside.so; do
  DAFMM_LIB_NAME=$lib timeout 300 python tools/mode_probe.py c4 '{}' >> gpurun_out/r2p_probe.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r2p_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_parity.log
export PROBE_ROWS=32
for lib in libdafmm.so libdafmm_noside.so; do
  DAFMM_LIB_NAME=$lib timeout 300 python tools/mode_probe.py c3 '{}' >> gpurun_out/r2p_probe.log 2>&1
  DAFMM_LIB_NAME=$lib timeout 400 python tools/mode_probe.py c5 '{}' >> gpurun_out/r2p_probe.log 2>&1
done
