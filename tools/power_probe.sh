#!/bin/bash
# SM clock / power / throttle reasons sampled every 100 ms while a long matvec loop runs
#   bash tools/power_probe.sh <tag> <config> <reps> [m2l_store]
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=$1; CFG=${2:-c4}; REPS=${3:-2000}; MODE=${4:--1}
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 100 > gpurun_out/power_$TAG.csv &
P=$!
python - "$CFG" "$REPS" "$MODE" <<'PY'
import sys, time, torch
sys.path.insert(0, '.')
import paper_2204_00326_b200 as prod
from synth.configs import make_problem
P = make_problem(sys.argv[1]); reps = int(sys.argv[2]); mode = int(sys.argv[3])
op = prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"], m2l_store=mode)
x = torch.from_numpy(P["x"]).cuda(); y = torch.empty_like(x)
for _ in range(5): op.matvec(x, y)
torch.cuda.synchronize(); time.sleep(1.0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps): op.matvec(x, y)
e1.record(); e1.synchronize()
print("mode", mode, "ms per matvec", e0.elapsed_time(e1) / reps, flush=True)
time.sleep(1.0)
PY
kill $P
python - "$TAG" <<'PY'
import sys, collections
rows = [l.split(',') for l in open('gpurun_out/power_%s.csv' % sys.argv[1]) if l.strip()]
load = [r for r in rows if float(r[1].split()[0]) > 400]
c = collections.Counter((r[0].strip(), r[2].strip()) for r in load)
print("samples under load", len(load), "power W median", sorted(float(r[1].split()[0]) for r in load)[len(load)//2] if load else None)
for k, v in c.most_common(8): print(v, k)
PY
