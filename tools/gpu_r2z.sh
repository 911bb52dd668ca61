#!/bin/bash
# r2z: the round's final cycle at HEAD: all GPU tests, bench (with the reference arm), launch list,
# ncu --set full of the hot kernels
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_r2z.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2z.log
bash tools/gpu_cycle.sh r2z c4 skip-tests
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r2z.log 2>&1; echo "smoke rc=$?"
