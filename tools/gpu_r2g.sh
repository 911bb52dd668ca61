#!/bin/bash
# r2g: pair-M2L barrier fix, HODLR plane layout + apply kernels + HR5, narrow-item translations
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "symmetric_pivots or pair" -p no:cacheprovider > gpurun_out/r2g_pair.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_pair.log
timeout 400 python -m pytest tests/test_gpu_hodlr.py -q --durations=5 > gpurun_out/r2g_hodlr.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_hodlr.log
export PROBE_ROWS=64 PROBE_STEPS=20
timeout 200 python tools/mode_probe.py c4 '{}' > gpurun_out/r2g_probe.log 2>&1
timeout 200 python tools/mode_probe.py c4 '{"symmetric_pivots": 1, "m2l_store": 2}' >> gpurun_out/r2g_probe.log 2>&1
timeout 600 python tools/hybrid_probe.py c3 '[[50, 16], [200, 16], [50, 16, 16384]]' > gpurun_out/r2g_hybrid.log 2>&1
export PROBE_MAXIT=1500
timeout 1200 python tools/hybrid_probe.py c5 '[[200, 0], [50, 16, 4096], [50, 16, 65536], [200, 16, 16384]]' >> gpurun_out/r2g_hybrid.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q --durations=20 -p no:cacheprovider > gpurun_out/r2g_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_parity.log
echo done
