"""Hybrid-solver probe: GMRES(m) on a BASELINE config with and without the HODLR
right preconditioner of rank r; prints setup times, iterations, true residual, solve time and
the HODLR apply time (CUDA events).

    python tools/hybrid_probe.py c3 '[[50, 0], [50, 8], [50, 16, 65536]]'   # [restart, rank(, max_block)] (rank 0: none)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2204_00326_b200 as prod  # noqa: E402
from synth.configs import make_problem  # noqa: E402

name = sys.argv[1]
cases = json.loads(sys.argv[2]) if len(sys.argv) > 2 else [[50, 0], [50, 16]]
maxit = int(os.environ.get("PROBE_MAXIT", "3000"))
P = make_problem(name)
t0 = time.perf_counter()
op = prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"])
setup = time.perf_counter() - t0
st = op.stats()
print(json.dumps(dict(config=name, N=int(P["points"].shape[0]), setup_s=round(setup, 2),
                      setup_breakdown={k: round(st[k], 3) for k in ("setup_tree_s", "setup_lists_s", "setup_nca_s",
                                                                    "setup_nca_device_s", "setup_ops_s",
                                                                    "setup_upload_s", "setup_ops_device_s")})),
      flush=True)
f = torch.from_numpy(P["f"]).cuda()
for case in cases:
    restart, rank = case[0], case[1]
    max_block = case[2] if len(case) > 2 else 0
    pc, pcs, apply_ms = None, None, None
    if rank > 0:
        t0 = time.perf_counter()
        pc = prod.HODLR(op, rank=rank, leaf_size=64, max_block=max_block)
        torch.cuda.synchronize()
        pcs = dict(setup_s=round(time.perf_counter() - t0, 3), **pc.stats())
        b = torch.empty_like(f)
        for _ in range(3):
            pc.solve(f, b)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            pc.solve(f, b)
        e1.record()
        e1.synchronize()
        apply_ms = e0.elapsed_time(e1) / 10
        # quality: ||A M^{-1} b - b|| / ||b|| for a random b (0 for M = A)
        g = torch.Generator(device="cpu").manual_seed(3)
        bb = torch.randn(f.numel(), dtype=torch.complex128, generator=g).cuda()
        z = torch.empty_like(bb)
        pc.solve(bb, z)
        az = torch.empty_like(bb)
        op.matvec(z, az)
        torch.cuda.synchronize()
        pcs["precond_residual"] = (torch.linalg.norm(az - bb) / torch.linalg.norm(bb)).item()
    psi = torch.empty_like(f)
    op.gmres(f, psi, P["gmres_tol"], 2, restart, prec=pc)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc, it, rr = op.gmres(f, psi, P["gmres_tol"], maxit, restart, prec=pc)
    solve = time.perf_counter() - t0
    print(json.dumps(dict(config=name, restart=restart, rank=rank, max_block=max_block, status=rc, iterations=it, true_relres=rr,
                          solve_s=round(solve, 3), ms_per_iteration=round(1e3 * solve / max(it, 1), 3),
                          hodlr=pcs, hodlr_apply_ms=apply_ms)), flush=True)
    if pc is not None:
        pc.close()
op.close()
