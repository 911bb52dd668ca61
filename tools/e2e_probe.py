"""Where the end-to-end time goes: dafmm_matvec_host (pinned host x -> device -> pinned host y)
against its parts, CUDA events on the handle's stream, C4 by default."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2204_00326_b200 as prod  # noqa: E402
from synth.configs import make_problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
P = make_problem(name)
op = prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"])
s = torch.cuda.Stream()
op.set_stream(s)
n = P["points"].shape[0]
xh = torch.from_numpy(P["x"]).pin_memory()
yh = torch.empty(n, dtype=torch.complex128).pin_memory()
xd = xh.cuda()
yd = torch.empty_like(xd)


def timed(fn):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), float(np.min(ts))


with torch.cuda.stream(s):
    for _ in range(3):
        op.matvec_host(xh.numpy(), yh.numpy())
    out = {"matvec": timed(lambda: op.matvec(xd, yd)),
           "h2d": timed(lambda: xd.copy_(xh, non_blocking=True)),
           "d2h": timed(lambda: yh.copy_(yd, non_blocking=True)),
           "matvec_host": timed(lambda: op.matvec_host(xh.numpy(), yh.numpy()))}
print(json.dumps({k: {"median_ms": v[0], "min_ms": v[1]} for k, v in out.items()}))
