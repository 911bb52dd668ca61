"""Accuracy probe on adaptive trees: GPU DAFMM vs the oracle's dense rows (sampled)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2204_00326_b200 as prod  # noqa: E402
from oracle.core import Problem  # noqa: E402
from synth.configs import make_problem  # noqa: E402

cases = [tuple(float(v) if "." in v else int(v) for v in c.split(":")) for c in sys.argv[1].split(",")]
rows_n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
for depth, kappa in cases:
    P = make_problem("c5", n=depth, kappa=kappa)
    t = time.perf_counter()
    op = prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"])
    setup = time.perf_counter() - t
    x = torch.from_numpy(P["x"]).cuda()
    y = torch.empty_like(x)
    op.matvec(x, y)
    torch.cuda.synchronize()
    yg = y.cpu().numpy()
    n = P["points"].shape[0]
    idx = np.sort(np.random.default_rng(5).choice(n, size=min(rows_n, n), replace=False))
    prob = Problem(P["points"], P["weights"], P["q"], P["kappa"])
    yd = oracle.dense_matvec_rows(prob, P["x"], idx)
    xs = P["x"][idx]
    err = np.linalg.norm((yg[idx] - xs) - (yd - xs)) / np.linalg.norm(yd - xs)
    st = op.stats()
    print(json.dumps(dict(depth=depth, kappa=kappa, n=n, r16_nonleaf=os.environ.get("DAFMM_R16_NONLEAF", "0"),
                          err=err, setup_s=setup, m2l_entries=st["m2l_entries"], max_rank=st["max_rank"])),
          flush=True)
    op.close()
