#!/bin/bash
# r2j: HODLR ACA-factor planes (stream-order fix), apply latency fixes, quality sweep
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_hodlr.py -q --durations=5 > gpurun_out/r2j_hodlr.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_hodlr.log
export PROBE_MAXIT=800
timeout 600 python tools/hybrid_probe.py c3 '[[50, 8], [50, 16], [50, 32], [200, 16]]' > gpurun_out/r2j_hybrid.log 2>&1
timeout 900 python tools/hybrid_probe.py c5 '[[200, 8], [200, 16], [200, 32], [50, 16, 16384]]' >> gpurun_out/r2j_hybrid.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2j_hodlr_launches.csv python tools/hodlr_kernels.py c3 16 > gpurun_out/r2j_ncu.log 2>&1
echo done
