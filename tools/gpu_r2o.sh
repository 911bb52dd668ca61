#!/bin/bash
# r2o: warp-private pair-stored M2L (m2l_pairw_kernel): parity of the pair mode, C4 A/B of its shapes
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
rm -f gpurun_out/r2o_probe.log
export PROBE_ROWS=64 PROBE_STEPS=20
for lib in libdafmm.so libdafmm_w12s3.so libdafmm_w16s2.so; do
  DAFMM_LIB_NAME=$lib timeout 300 python tools/mode_probe.py c4 '{"symmetric_pivots": 1, "m2l_store": 2}' >> gpurun_out/r2o_probe.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "symmetric_pivots or pair" -p no:cacheprovider > gpurun_out/r2o_pair.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_pair.log
