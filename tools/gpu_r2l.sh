#!/bin/bash
# r2l: HODLR leaf / Woodbury inverses applied as GEMVs
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_hodlr.py -q --durations=5 > gpurun_out/r2l_hodlr.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_hodlr.log
export PROBE_MAXIT=1000
timeout 600 python tools/hybrid_probe.py c3 '[[50, 16], [200, 16], [50, 8]]' > gpurun_out/r2l_hybrid.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2l_hodlr_launches.csv python tools/hodlr_kernels.py c3 16 > gpurun_out/r2l_ncu.log 2>&1
export PROBE_MAXIT=6000
timeout 900 python tools/hybrid_probe.py c5 '[[200, 0]]' >> gpurun_out/r2l_hybrid.log 2>&1
echo done
