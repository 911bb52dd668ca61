#!/bin/bash
# r2f: row-major translations with device-formed operators, the GPU test suite with per-test timings
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export PROBE_ROWS=64 PROBE_STEPS=20
timeout 300 python tools/mode_probe.py c4 '{}' '{"symmetric_pivots": 1, "m2l_store": 2}' > gpurun_out/r2f_probe.log 2>&1
timeout 900 python tools/hybrid_probe.py c3 '[[50, 0], [50, 8], [50, 16], [200, 16]]' > gpurun_out/r2f_hybrid.log 2>&1
timeout 900 python tools/hybrid_probe.py c5 '[[50, 16], [50, 24]]' >> gpurun_out/r2f_hybrid.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -v --timeout=600 --durations=30 > gpurun_out/r2f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_pytest.log
echo done
