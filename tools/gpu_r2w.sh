#!/bin/bash
# r2w: translate_cm_kernel with lane groups for small-R batches: C4/C3/C5 probe, ncu of the 7 launches, parity
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
rm -f gpurun_out/r2w_probe.log
export PROBE_ROWS=64 PROBE_STEPS=30
timeout 200 python tools/mode_probe.py c4 '{}' >> gpurun_out/r2w_probe.log 2>&1
export PROBE_ROWS=32
timeout 200 python tools/mode_probe.py c3 '{}' >> gpurun_out/r2w_probe.log 2>&1
timeout 300 python tools/mode_probe.py c5 '{}' >> gpurun_out/r2w_probe.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"translate" -s 0 -c 7 \
  -o gpurun_out/r2w_translate -f python tools/ncu_target.py c4 1 > gpurun_out/r2w_ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r2w_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2w_parity.log
