"""Launch the HODLR apply a few times on a config (for an ncu launch list of its kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2204_00326_b200 as prod  # noqa: E402
from synth.configs import make_problem  # noqa: E402

P = make_problem(sys.argv[1] if len(sys.argv) > 1 else "c3")
op = prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"])
pc = prod.HODLR(op, rank=int(sys.argv[2]) if len(sys.argv) > 2 else 16)
f = torch.from_numpy(P["f"]).cuda()
x = torch.empty_like(f)
for _ in range(3):
    pc.solve(f, x)
torch.cuda.synchronize()
pc.close()
op.close()
