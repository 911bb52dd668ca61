#!/bin/bash
# One GPU cycle: GPU tests, bench, launch list, one full ncu capture of the hot kernels.
#   bash tools/gpu_cycle.sh <tag> [config] [skip-tests]
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-rXX}
CFG=${2:-c4}
if [ "$3" != "skip-tests" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"
fi
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/clocks_$TAG.csv &
CP=$!
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
kill $CP
python tools/ncu_target.py $CFG 3 > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python tools/ncu_target.py $CFG 3 > gpurun_out/ncu_launches_$TAG.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on \
    --metrics sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active \
    -k regex:"p2p_kernel|m2l_kernel|m2l_stored|translate|combine_kernel" -s 0 -c 20 -o gpurun_out/prof_$TAG -f \
    python tools/ncu_target.py $CFG 1 > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
# the on-the-fly M2L kernel (dafmm_options.m2l_store = 0) for comparison
ncu --set full --clock-control none --import-source on \
    --metrics sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active \
    -k regex:"m2l_kernel" -s 0 -c 1 -o gpurun_out/prof_${TAG}_fly -f \
    python tools/ncu_target.py $CFG 1 0 > gpurun_out/ncu_fly_$TAG.log 2>&1; echo "ncu fly rc=$?"
