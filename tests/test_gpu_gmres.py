"""GPU GMRES (ls_gmres_solve, reading R14) through the C-ABI: the solution against a
dense solve of the oracle's operator, the exit residual against a recomputed one, the A = I
special case and the residual history."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
from oracle.core import Problem
from synth.configs import make_problem

pytestmark = pytest.mark.gpu


def _prod():
    import paper_2204_00326_b200 as prod
    return prod


def test_gmres_matches_dense_solve_c1():
    P = make_problem("c1")
    op = _prod().DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"])
    f = torch.from_numpy(P["f"]).cuda()
    psi = torch.empty_like(f)
    hist = np.zeros(201)
    rc, iters, relres = op.gmres(f, psi, 1e-10, 200, 50, hist)
    assert rc == 0 and 1 <= iters <= 200
    assert relres <= 2e-10
    assert op.stats()["gmres_reorth"] == iters  # CGS2: a second pass every iteration (R20)
    # exit residual equals a recomputed one with the same operator
    y = torch.empty_like(f)
    op.matvec(psi, y)
    torch.cuda.synchronize()
    r = np.linalg.norm((y - f).cpu().numpy()) / np.linalg.norm(P["f"])
    assert abs(r - relres) <= 1e-12 + 1e-3 * relres
    # history: starts at 1, non-increasing within a cycle (GMRES minimises the residual)
    h = hist[:iters + 1]
    assert h[0] == 1.0 and np.all(np.diff(h) <= 1e-14)
    # solution against the dense oracle operator (cond ~ 6, DAFMM error <= 10 nca_tol)
    prob = Problem(P["points"], P["weights"], P["q"], P["kappa"])
    A = oracle.A_block(prob, np.arange(4096), np.arange(4096))
    psi_d = np.linalg.solve(A, P["f"])
    err = np.linalg.norm(psi.cpu().numpy() - psi_d) / np.linalg.norm(psi_d)
    assert err <= 1e-6, err


def test_gmres_identity_one_iteration():
    P = make_problem("c1", n=32)
    op = _prod().DAFMM(P["points"], P["weights"], np.zeros(1024), P["kappa"], 64, 1e-8)
    f = torch.from_numpy(P["x"]).cuda()
    psi = torch.empty_like(f)
    rc, iters, relres = op.gmres(f, psi, 1e-12, 10, 50)
    assert rc == 0 and iters == 1 and relres <= 1e-14
    assert torch.allclose(psi, f, rtol=0, atol=1e-14)


def test_gmres_not_converged_status_and_restart():
    """maxit reached is a positive status, not an error; restarts keep the residual decreasing."""
    P = make_problem("c3", n=128, kappa=20.0)
    op = _prod().DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"])
    f = torch.from_numpy(P["f"]).cuda()
    psi = torch.empty_like(f)
    rc, iters, relres = op.gmres(f, psi, 1e-14, 12, 5)
    assert rc == 1 and iters == 12 and 0 < relres < 1
    rc2, iters2, relres2 = op.gmres(f, psi, 1e-14, 24, 5)
    assert rc2 == 1 and relres2 <= relres


def test_gmres_zero_rhs():
    P = make_problem("c1", n=32)
    op = _prod().DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, 1e-8)
    f = torch.zeros(1024, dtype=torch.complex128, device="cuda")
    psi = torch.ones_like(f)
    rc, iters, relres = op.gmres(f, psi, 1e-8, 10, 50)
    assert rc == 0 and iters == 0 and float(psi.abs().max()) == 0.0


def test_gmres_restart_change_and_true_residual_status():
    """A handle re-sizes its GMRES workspace when the restart changes; DAFMM_OK always means the
    TRUE relative residual ||f - A psi|| / ||f|| is within tol (the stopping rule uses it)."""
    P = make_problem("c2", n=128, kappa=20.0)
    op = _prod().DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"])
    f = torch.from_numpy(P["f"]).cuda()
    y = torch.empty_like(f)
    for restart in (10, 30, 10):
        psi = torch.empty_like(f)
        rc, iters, relres = op.gmres(f, psi, 1e-9, 400, restart)
        assert rc == 0 and relres <= 1e-9
        op.matvec(psi, y)
        torch.cuda.synchronize()
        true = np.linalg.norm((y - f).cpu().numpy()) / np.linalg.norm(P["f"])
        assert true <= 1e-9 * (1 + 1e-6)


def test_binding_rejects_wrong_lengths():
    P = make_problem("c1", n=32)
    op = _prod().DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, 1e-8)
    x = torch.zeros(1024, dtype=torch.complex128, device="cuda")
    short = torch.zeros(1000, dtype=torch.complex128, device="cuda")
    with pytest.raises(ValueError):
        op.matvec(x, short)
    with pytest.raises(ValueError):
        op.gmres(short, x, 1e-8, 10)
