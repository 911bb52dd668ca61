#!/bin/bash
# bench + launch list + one full ncu capture of the P2P and M2L kernels (config given as $1, default c4)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CFG=${1:-c4}
TAG=${2:-r01}
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python tools/ncu_target.py $CFG 3 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python tools/ncu_target.py $CFG 3 > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on \
    --metrics sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active \
    -k regex:"p2p_kernel|m2l_kernel|translate|combine_kernel" -s 0 -c 20 -o gpurun_out/prof_$TAG -f \
    python tools/ncu_target.py $CFG 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
