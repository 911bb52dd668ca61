"""GMRES(m) convergence on a config for several restart lengths (iterations, time, true relres)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2204_00326_b200 as prod  # noqa: E402
from synth.configs import make_problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
restarts = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [50, 100, 200]
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else 3000
P = make_problem(name)
for m in restarts:
    op = prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"])
    f = torch.from_numpy(P["f"]).cuda()
    psi = torch.empty_like(f)
    torch.cuda.synchronize()
    t = time.perf_counter()
    rc, it, rr = op.gmres(f, psi, P["gmres_tol"], maxit, m)
    dt = time.perf_counter() - t
    t = time.perf_counter()  # a second solve on the same handle (workspace allocated)
    rc2, it2, rr2 = op.gmres(f, psi, P["gmres_tol"], maxit, m)
    dt2 = time.perf_counter() - t
    print(json.dumps(dict(config=name, restart=m, status=rc, iterations=it, relres=rr, solve_s=dt,
                          s_per_iter=dt / max(it, 1), second_solve_s=dt2, second_iterations=it2,
                          reorthogonalisations=op.stats()["gmres_reorth"])), flush=True)
    op.close()
