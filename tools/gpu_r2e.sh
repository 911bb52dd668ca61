#!/bin/bash
# r2e: first GPU cycle of the device setup (F2), device HODLR (F3) and streamed translations
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nproc > gpurun_out/r2e_host.txt; lscpu | grep "Model name" >> gpurun_out/r2e_host.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --durations=15 -k "matches_oracle or device_aca or pair" > gpurun_out/r2e_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_parity.log
timeout 600 python -m pytest tests/test_gpu_hodlr.py -q --durations=10 > gpurun_out/r2e_hodlr.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_hodlr.log
export PROBE_ROWS=64 PROBE_STEPS=20
timeout 400 python tools/mode_probe.py c4 '{}' > gpurun_out/r2e_probe.log 2>&1
timeout 300 python tools/mode_probe.py c4 '{"symmetric_pivots": 1, "m2l_store": 2}' >> gpurun_out/r2e_probe.log 2>&1
DAFMM_TRANSLATE_ROWMAJOR=1 timeout 300 python tools/mode_probe.py c4 '{}' >> gpurun_out/r2e_probe.log 2>&1
echo done
