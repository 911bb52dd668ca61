#!/bin/bash
# r2bl: the ncu launch list of the bench command itself (C4 matvec steps only: no GMRES, per-config lines,
# CPU baseline or e2e), after the same command has exited 0 without ncu
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CMD="python bench.py --steps 5 --warmup 3 --no-gmres --no-configs --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/bench_r2bl.json 2> gpurun_out/bench_r2bl.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench_r2.csv $CMD > gpurun_out/ncu_bench_r2.log 2>&1; echo "ncu rc=$?"
