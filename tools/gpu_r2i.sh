#!/bin/bash
# r2i: HODLR from the ACA factors (no cross-matrix inverse); quality sweep
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_hodlr.py -q --durations=5 > gpurun_out/r2i_hodlr.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_hodlr.log
export PROBE_MAXIT=600
timeout 600 python tools/hybrid_probe.py c3 '[[50, 8], [50, 16], [50, 32], [200, 16]]' > gpurun_out/r2i_hybrid.log 2>&1
timeout 900 python tools/hybrid_probe.py c5 '[[200, 8], [200, 16], [200, 32], [200, 16, 16384]]' >> gpurun_out/r2i_hybrid.log 2>&1
echo done
