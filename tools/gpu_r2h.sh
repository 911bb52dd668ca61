#!/bin/bash
# r2h: HODLR apply launch list, preconditioner quality sweep on c5 / c3 / c2, setup breakdowns
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h_hodlr_launches.csv python tools/hodlr_kernels.py c3 16 > gpurun_out/r2h_ncu.log 2>&1
export PROBE_ROWS=0 PROBE_STEPS=10
timeout 200 python tools/mode_probe.py c4 '{}' > gpurun_out/r2h_probe.log 2>&1
timeout 200 python tools/mode_probe.py c5 '{}' >> gpurun_out/r2h_probe.log 2>&1
export PROBE_MAXIT=400
timeout 600 python tools/hybrid_probe.py c2 '[[50, 0], [50, 16]]' > gpurun_out/r2h_hybrid.log 2>&1
timeout 600 python tools/hybrid_probe.py c3 '[[50, 16], [50, 32], [50, 16, 4096]]' >> gpurun_out/r2h_hybrid.log 2>&1
timeout 900 python tools/hybrid_probe.py c5 '[[200, 32], [200, 16, 1024], [200, 8, 256], [200, 4, 0]]' >> gpurun_out/r2h_hybrid.log 2>&1
echo done
