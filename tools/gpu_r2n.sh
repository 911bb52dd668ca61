#!/bin/bash
# r2n: C5 unpreconditioned GMRES(200) convergence probe (up to 8000 iterations); C4 A/B of the stored vs
# pair-stored M2L; ncu of the pair-stored M2L (m2l_store=2, symmetric pivots) at C4
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export PROBE_MAXIT=8000
timeout 900 python tools/hybrid_probe.py c5 '[[200, 0]]' > gpurun_out/r2n_c5.log 2>&1; echo "c5 rc=$?"
export PROBE_ROWS=64 PROBE_STEPS=20
timeout 300 python tools/mode_probe.py c4 '{}' '{"symmetric_pivots": 1, "m2l_store": 2}' > gpurun_out/r2n_probe.log 2>&1
export DAFMM_OPTS=symmetric_pivots=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"m2l_pair|m2l_slot" -s 0 -c 2 \
  -o gpurun_out/r2n_pair -f python tools/ncu_target.py c4 1 2 > gpurun_out/r2n_ncu.log 2>&1; echo "ncu rc=$?"
