#!/bin/bash
# r2y: host part of the C4 setup after the parallel M2L stream fill (DAFMM_SETUP_TRACE), parity subset
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export PROBE_ROWS=64 PROBE_STEPS=5
DAFMM_SETUP_TRACE=1 timeout 300 python tools/mode_probe.py c4 '{}' '{}' > gpurun_out/r2y_trace.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "test_gpu_matches_oracle or pair_stored_m2l_wide or store" -p no:cacheprovider > gpurun_out/r2y_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2y_parity.log
