#!/bin/bash
# r2n: ncu of the pair-stored M2L (m2l_store=2, symmetric pivots) at C4; C5 GMRES convergence probes
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export DAFMM_OPTS=symmetric_pivots=1
timeout 300 python tools/ncu_target.py c4 1 2 > gpurun_out/r2n_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"m2l_pair|m2l_slot" -s 0 -c 2 \
  -o gpurun_out/r2n_pair -f python tools/ncu_target.py c4 1 2 > gpurun_out/r2n_ncu.log 2>&1; echo "ncu rc=$?"
unset DAFMM_OPTS
export PROBE_MAXIT=3000
timeout 900 python tools/hybrid_probe.py c5 '[[200, 16, 1024], [200, 0]]' > gpurun_out/r2n_c5.log 2>&1; echo "c5 rc=$?"
