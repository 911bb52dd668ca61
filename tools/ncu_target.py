"""Small program for ncu captures: build a config's plan and run a few matvecs on cuda:0."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2204_00326_b200 as prod  # noqa: E402
from synth.configs import make_problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
P = make_problem(name)
mode = int(sys.argv[3]) if len(sys.argv) > 3 else -1  # dafmm_options.m2l_store
extra = dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in os.environ.get("DAFMM_OPTS", "").split(",") if kv)
op = prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"], m2l_store=mode, **extra)
x = torch.from_numpy(P["x"]).cuda()
y = torch.empty_like(x)
for _ in range(reps):
    op.matvec(x, y)
torch.cuda.synchronize()
print("ok", name, float(y.abs().sum()))
op.close()
