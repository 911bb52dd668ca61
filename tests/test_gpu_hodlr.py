"""GPU parity of the HODLR preconditioner and the hybrid solver (readings HR1-HR4):
the product's factorised device solve Ã^{-1} b against the oracle's HODLR (the same HODLR
matrix assembled densely from the product's validated pivots and solved by dense LU), and the
right-preconditioned GMRES against the unpreconditioned one."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle.core import Problem
from oracle.hodlr import HODLR, sibling_blocks
from synth.configs import make_problem

pytestmark = pytest.mark.gpu


def _prod():
    import paper_2204_00326_b200 as prod
    return prod


def _import_pivots(path):
    blocks = np.load(path / "hodlr_blocks.npy")
    ptr = np.load(path / "hodlr_piv_ptr.npy")
    I, J = np.load(path / "hodlr_I.npy"), np.load(path / "hodlr_J.npy")
    perm = np.load(path / "hodlr_perm.npy")
    r, n0, n = np.load(path / "hodlr_meta.npy")[:3]
    piv = {}
    for k, (_, a, b, c, d) in enumerate(blocks):
        piv[(int(a), int(b), int(c), int(d))] = (I[ptr[k]:ptr[k + 1]], J[ptr[k]:ptr[k + 1]])
    return piv, perm, int(r), int(n0), int(n), blocks


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("name,n,kappa,rank,n0", [("c1", None, None, 8, 64), ("c3", 64, 10.0, 12, 64),
                                                  ("c5", 5, 12.0, 6, 40), ("c1", 48, 8.0, 12, 24)])
def test_gpu_hodlr_solve_matches_oracle(name, n, kappa, rank, n0, tmp_path):
    P = make_problem(name, n=n, kappa=kappa)
    op = _prod().DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"])
    pc = _prod().HODLR(op, rank=rank, leaf_size=n0)
    st = pc.stats()
    assert st["rank"] == rank and st["leaf_size"] == n0 and 0 < st["max_rank"] <= rank
    pc.export(str(tmp_path))
    piv, perm, r, nn0, N, blocks = _import_pivots(tmp_path)
    assert (r, nn0, N) == (rank, n0, P["points"].shape[0])
    # HR1: the exported blocks are exactly the oracle's sibling blocks of the midpoint tree
    assert sorted(tuple(int(v) for v in b) for b in blocks) == sorted(sibling_blocks(N, n0))
    prob = Problem(P["points"], P["weights"], P["q"], P["kappa"])
    H = HODLR(prob, perm, n0, rank, pivots=piv)
    H.validate()
    rng = np.random.default_rng(11)
    b = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    x_ref = H.solve(b)
    xd = torch.empty(N, dtype=torch.complex128, device="cuda")
    pc.solve(_dev(b), xd)
    torch.cuda.synchronize()
    x = xd.cpu().numpy()
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 1e-10
    # in place (b and x the same vector)
    bd = _dev(b)
    pc.solve(bd, bd)
    torch.cuda.synchronize()
    assert np.array_equal(bd.cpu().numpy(), x)
    pc.close()
    op.close()


def test_gpu_hodlr_zero_contrast_is_identity():
    """q = 0: every off-diagonal block of A vanishes (rank 0) and the leaf blocks are I, so
    Ã^{-1} b = b exactly."""
    P = make_problem("c1")
    q = np.zeros_like(P["q"])
    op = _prod().DAFMM(P["points"], P["weights"], q, P["kappa"], 64, P["nca_tol"])
    pc = _prod().HODLR(op, rank=8, leaf_size=64)
    assert pc.stats()["max_rank"] == 0
    b = P["x"]
    xd = torch.empty_like(_dev(b))
    pc.solve(_dev(b), xd)
    torch.cuda.synchronize()
    assert np.array_equal(xd.cpu().numpy(), b)
    pc.close()
    op.close()


@pytest.mark.parametrize("name,n,kappa", [("c3", 128, 40.0), ("c2", 128, 40.0)])
def test_gpu_hybrid_solver_converges_faster(name, n, kappa):
    """Right preconditioning (HR4): the GMRES residual is the true residual; with Ã^{-1} the
    solve takes fewer iterations and reaches the same solution."""
    P = make_problem(name, n=n, kappa=kappa)
    op = _prod().DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"])
    f = _dev(P["f"])
    psi0 = torch.empty_like(f)
    tol = 1e-8
    rc0, it0, rr0 = op.gmres(f, psi0, tol, 3000, restart=50)
    assert rc0 == 0 and rr0 <= tol
    pc = _prod().HODLR(op, rank=16, leaf_size=64)
    psi1 = torch.empty_like(f)
    hist = np.zeros(3001)
    rc1, it1, rr1 = op.gmres(f, psi1, tol, 3000, restart=50, history=hist, prec=pc)
    assert rc1 == 0 and rr1 <= tol
    assert it1 < it0, (it1, it0)
    # the returned residual is the true one: recompute ||f - A psi|| / ||f||
    y = torch.empty_like(f)
    op.matvec(psi1, y)
    torch.cuda.synchronize()
    true = (torch.linalg.norm(f - y) / torch.linalg.norm(f)).item()
    assert abs(true - rr1) <= 1e-12 + 1e-6 * rr1
    a, b = psi0.cpu().numpy(), psi1.cpu().numpy()
    assert np.linalg.norm(a - b) / np.linalg.norm(a) <= 1e-5
    pc.close()
    op.close()


def test_gpu_hodlr_invalid_arguments():
    prod = _prod()
    P = make_problem("c1")
    op = prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"])
    for rank, n0 in [(0, 64), (33, 64), (8, 0), (8, 65)]:
        with pytest.raises(prod.DAFMMError):
            prod.HODLR(op, rank=rank, leaf_size=n0)
    op2 = prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"], kernel_mode=1)
    with pytest.raises(prod.DAFMMError):
        prod.HODLR(op2, rank=8)
    pc = prod.HODLR(op, rank=8)
    f = _dev(P["x"])
    psi = torch.empty_like(f)
    with pytest.raises(prod.DAFMMError):  # preconditioner of another handle
        prod.ls_gmres_solve_prec(op2.h, pc.p, f, psi, 1e-6, 10)
    pc.close()
    op.close()
    op2.close()


def test_gpu_hodlr_max_block_matches_oracle(tmp_path):
    """HR5 (option): with max_block the sibling blocks of more rows are dropped; the product's
    exported pivots are empty exactly there and the solve matches the oracle's HODLR."""
    P = make_problem("c1")
    op = _prod().DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"])
    pc = _prod().HODLR(op, rank=8, leaf_size=64, max_block=512)
    assert pc.stats()["max_block"] == 512
    pc.export(str(tmp_path))
    piv, perm, r, n0, N, blocks = _import_pivots(tmp_path)
    for (a, b, c, d), (I, J) in piv.items():
        assert (len(I) == 0) if b - a > 512 else True
    assert any(len(I) > 0 for I, _ in piv.values())
    prob = Problem(P["points"], P["weights"], P["q"], P["kappa"])
    H = HODLR(prob, perm, n0, r, pivots=piv)
    H.validate()
    b = np.random.default_rng(3).standard_normal(N) + 0j
    xd = torch.empty(N, dtype=torch.complex128, device="cuda")
    pc.solve(_dev(b), xd)
    torch.cuda.synchronize()
    x_ref = H.solve(b)
    assert np.linalg.norm(xd.cpu().numpy() - x_ref) / np.linalg.norm(x_ref) <= 1e-10
    pc.close()
    op.close()
