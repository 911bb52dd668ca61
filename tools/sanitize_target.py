"""Small run for compute-sanitizer: config-1 matvec (full, near-only, far-only), a ragged
non-lattice problem (generic band paths), a few GMRES iterations, the pair-stored M2L and the
hybrid solver."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2204_00326_b200 as prod  # noqa: E402
from synth.configs import make_problem  # noqa: E402

P = make_problem("c1")
op = prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"])
x = torch.from_numpy(P["x"]).cuda()
y = torch.empty_like(x)
for mask in (3, 1, 2):
    op.matvec(x, y, mask)
f = torch.from_numpy(P["f"]).cuda()
psi = torch.empty_like(f)
print("gmres", op.gmres(f, psi, 1e-10, 20, 8))
rng = np.random.default_rng(7)
pts = rng.uniform(-1, 1, size=(3000, 2))
op2 = prod.DAFMM(pts, np.full(3000, 4.0 / 3000), 1.0 + 0.5 * np.cos(3 * pts[:, 0]), 12.0, 64, 1e-8)
x2 = torch.from_numpy(np.exp(1j * rng.uniform(0, 6.3, 3000))).cuda()
y2 = torch.empty_like(x2)
op2.matvec(x2, y2)
# the pair-stored M2L (warp pairs, TMA rings, slot gather) on a case with two directional levels and
# on wide nodes (more than 32 pivots: the row-block path), and the HODLR preconditioner
P3 = make_problem("c2", n=64, kappa=40.0)
op3 = prod.DAFMM(P3["points"], P3["weights"], P3["q"], P3["kappa"], 64, P3["nca_tol"], symmetric_pivots=1, m2l_store=2)
x3 = torch.from_numpy(P3["x"]).cuda()
y3 = torch.empty_like(x3)
op3.matvec(x3, y3)
op4 = prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, 1e-12, symmetric_pivots=1, m2l_store=2)
op4.matvec(x, y)
pc = prod.HODLR(op, rank=8, leaf_size=64)
print("hybrid", op.gmres(f, psi, 1e-10, 20, 8, prec=pc))
torch.cuda.synchronize()
print("ok", float(y.abs().sum()), float(y2.abs().sum()), float(y3.abs().sum()))
