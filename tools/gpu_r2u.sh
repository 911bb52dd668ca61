#!/bin/bash
# r2u: column-major translation items (translate_cm_kernel, lane per row) against the row-major warp-per-row
# kernels (DAFMM_OPS_ROWMAJOR=1): C4 / C3 / C5 A/B, then the parity tests on the new default
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
rm -f gpurun_out/r2u_probe.log
export PROBE_ROWS=64 PROBE_STEPS=30
timeout 200 python tools/mode_probe.py c4 '{}' >> gpurun_out/r2u_probe.log 2>&1
DAFMM_OPS_ROWMAJOR=1 timeout 200 python tools/mode_probe.py c4 '{}' >> gpurun_out/r2u_probe.log 2>&1
export PROBE_ROWS=32
timeout 200 python tools/mode_probe.py c3 '{}' >> gpurun_out/r2u_probe.log 2>&1
DAFMM_OPS_ROWMAJOR=1 timeout 200 python tools/mode_probe.py c3 '{}' >> gpurun_out/r2u_probe.log 2>&1
timeout 300 python tools/mode_probe.py c5 '{}' >> gpurun_out/r2u_probe.log 2>&1
DAFMM_OPS_ROWMAJOR=1 timeout 300 python tools/mode_probe.py c5 '{}' >> gpurun_out/r2u_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r2u_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_parity.log
