#!/bin/bash
# First GPU pass: probe host/GPU, fp64 DFMA peak, GPU tests, smoke, quick matvec timings.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
bash tools/probe.sh > gpurun_out/probe.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for c in c1 c2 c3; do timeout 600 python tools/quick_bench.py $c 20 >> gpurun_out/quick.log 2>&1; done
timeout 1200 python tools/quick_bench.py c4 20 >> gpurun_out/quick.log 2>&1
echo done
