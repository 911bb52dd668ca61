#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2d_gpu.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2d_pytest.log
export PROBE_ROWS=64
timeout 1200 python tools/mode_probe.py c4 '{}' '{"symmetric_pivots": 1, "m2l_store": 1}' '{"symmetric_pivots": 1, "m2l_store": 2}' > gpurun_out/r2d_probe.log 2>&1
echo done
