#!/bin/bash
# r2ab: per-plan hold of the P2P until M2M has finished: probes, GPU tests, bench, launch list of the bench command
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
rm -f gpurun_out/r2ab_probe.log
export PROBE_ROWS=0 PROBE_STEPS=30
for c in c4 c3 c5 c2 c1; do
  timeout 300 python tools/mode_probe.py $c '{}' >> gpurun_out/r2ab_probe.log 2>&1
done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_r2ab.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2ab.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/clocks_r2ab.csv &
CP=$!
timeout 900 python bench.py > gpurun_out/bench_r2ab.json 2> gpurun_out/bench_r2ab.err; echo "bench rc=$?"
kill $CP
CMD="python bench.py --steps 5 --warmup 3 --no-gmres --no-configs --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench_r2ab.csv $CMD > gpurun_out/ncu_bench_r2ab.log 2>&1; echo "ncu rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r2ab.log 2>&1; echo "smoke rc=$?"
