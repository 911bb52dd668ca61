#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "pair" > gpurun_out/pytest_pair.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pair.log
export PROBE_ROWS=0
timeout 900 python tools/mode_probe.py c4 '{}' '{"symmetric_pivots": 1, "m2l_store": 2}' > gpurun_out/probe_r2c.log 2>&1
DAFMM_LIB_NAME=libdafmm_pc128.so timeout 900 python tools/mode_probe.py c4 '{"symmetric_pivots": 1, "m2l_store": 2}' >> gpurun_out/probe_r2c.log 2>&1
echo done
