"""Quick timing of dafmm_matvec on a config (CUDA events on the handle's stream)."""
import sys, time, json, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_00326_b200 as prod
from synth.configs import make_problem

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
P = make_problem(name)
t = time.time()
op = prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"])
setup = time.time() - t
st = op.stats()
s = torch.cuda.Stream()
op.set_stream(s)
x = torch.from_numpy(P["x"]).cuda()
y = torch.empty_like(x)
with torch.cuda.stream(s):
    for _ in range(3):
        op.matvec(x, y)
    s.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); op.matvec(x, y); e1.record(s); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
print(json.dumps(dict(config=name, n=P["points"].shape[0], setup_s=setup, ms_median=float(np.median(ts)), ms_min=min(ts),
                      unknowns_per_s=P["points"].shape[0] / (np.median(ts) * 1e-3), stats=st)))
