"""Pins for the oracle's HODLR preconditioner (readings HR1-HR4): against closed
cases (full rank reproduces A, q = 0 gives the identity), the HODLR rank structure, the ACA
skeleton against the SVD, and its effect as a right preconditioner on GMRES."""
import numpy as np

import oracle
from oracle.core import Problem
from oracle.gmres import gmres
from oracle.hodlr import HODLR, aca_fixed_rank, hodlr_tree, sibling_blocks
from oracle.tree import Tree
from synth.configs import make_problem


def _case(name, n, kappa):
    P = make_problem(name, n=n, kappa=kappa)
    prob = Problem(P["points"], P["weights"], P["q"], P["kappa"])
    tree = Tree(P["points"], P["weights"], P["kappa"], 64)
    perm = np.concatenate([tree.boxes[l][b] for l, b in tree.all_leaves()])
    return P, prob, perm


def test_tree_partitions_and_blocks_cover_off_diagonal():
    """HR1: the leaves partition [0, n); the diagonal leaf blocks plus the sibling blocks tile
    the whole n x n matrix exactly once."""
    n, n0 = 1000, 64
    nodes = hodlr_tree(n, n0)
    leaves = sorted((a, b) for _, a, b in nodes if b - a <= n0)
    assert leaves[0][0] == 0 and leaves[-1][1] == n
    assert all(leaves[i][1] == leaves[i + 1][0] for i in range(len(leaves) - 1))
    cover = np.zeros((n, n), dtype=np.int32)
    for a, b in leaves:
        cover[a:b, a:b] += 1
    for _, a, b, c, d in sibling_blocks(n, n0):
        cover[a:b, c:d] += 1
    assert np.all(cover == 1)


def test_aca_fixed_rank_exact_low_rank_and_cap():
    rng = np.random.default_rng(2)
    M = (rng.standard_normal((70, 4)) + 1j * rng.standard_normal((70, 4))) @ \
        (rng.standard_normal((4, 50)) + 1j * rng.standard_normal((4, 50)))
    rows, cols = aca_fixed_rank(lambda i: M[i].copy(), lambda j: M[:, j].copy(), 70, 50, 10, 0)
    assert len(rows) == 4  # a rank-4 matrix: the fifth residual row is at rounding level
    S = M[:, cols] @ np.linalg.solve(M[np.ix_(rows, cols)], M[rows, :])
    assert np.linalg.norm(S - M) / np.linalg.norm(M) < 1e-12
    rows, cols = aca_fixed_rank(lambda i: M[i].copy(), lambda j: M[:, j].copy(), 70, 50, 2, 0)
    assert len(rows) == 2  # the cap


def test_full_rank_hodlr_is_A():
    """With the rank cap above every block size the skeletons are exact: Ã = A."""
    P, prob, perm = _case("c1", 32, 8.0)
    H = HODLR(prob, perm, 64, 1024)
    A = oracle.A_block(prob, perm, perm)
    assert np.linalg.norm(H.dense() - A) / np.linalg.norm(A) < 1e-10
    b = P["f"]
    assert np.linalg.norm(H.solve(b) - np.linalg.solve(oracle.A_block(prob, np.arange(prob.n), np.arange(prob.n)), b)) \
        <= 1e-9 * np.linalg.norm(H.solve(b))


def test_zero_contrast_is_identity():
    P, prob, perm = _case("c1", 32, 8.0)
    prob0 = Problem(P["points"], P["weights"], np.zeros(prob.n), P["kappa"])
    H = HODLR(prob0, perm, 64, 5)
    assert np.array_equal(H.dense(), np.eye(prob.n))
    assert all(len(I) == 0 for I, _ in H.pivots.values())


def test_rank_structure_and_leaf_blocks():
    """Every off-diagonal sibling block of Ã has rank <= r; leaf diagonal blocks equal A."""
    P, prob, perm = _case("c3", 32, 10.0)
    r = 5
    H = HODLR(prob, perm, 64, r)
    D = H.dense()
    A = oracle.A_block(prob, perm, perm)
    for _, a, b, c, d in H.blocks:
        assert np.linalg.matrix_rank(D[a:b, c:d], tol=1e-12 * max(1.0, np.abs(D[a:b, c:d]).max())) <= r
    for _, a, b in hodlr_tree(prob.n, 64):
        if b - a <= 64:
            assert np.array_equal(D[a:b, a:b], A[a:b, a:b])
    H.validate()


def test_skeleton_error_tracks_svd():
    """HR2 on a real sibling block: the rank-r skeleton error is within a modest factor of the
    best rank-r error (the (r+1)-th singular value)."""
    P, prob, perm = _case("c2", 64, 20.0)
    n = prob.n
    a, b, c, d = 0, n // 2, n // 2, n
    blk = oracle.A_block(prob, perm[a:b], perm[c:d])
    sv = np.linalg.svd(blk, compute_uv=False)
    for r in (5, 15):
        H = HODLR(prob, perm, n // 2, r)  # one split: the two top blocks only
        I, J = H.pivots[(a, b, c, d)]
        S = oracle.A_block(prob, perm[a:b], perm[J]) @ np.linalg.solve(
            oracle.A_block(prob, perm[I], perm[J]), oracle.A_block(prob, perm[I], perm[c:d]))
        err = np.linalg.norm(blk - S, 2)
        assert len(I) == r and err <= 50 * sv[r]


def test_right_preconditioner_cuts_gmres_iterations():
    """HR4: GMRES on A Ã^{-1} u = f (psi = Ã^{-1} u) needs far fewer iterations than on A psi = f
    (Exp. 3 / 5: the HODLR preconditioner at ranks 5-25); the solution is the same."""
    P, prob, perm = _case("c3", 64, 40.0)  # 4096 points, kappa h = 1.25 (a hard high-kappa case)
    A = oracle.A_block(prob, np.arange(prob.n), np.arange(prob.n))
    f = P["f"]
    _, it0, rr0, _, conv0 = gmres(lambda v: A @ v, f, 1e-6, 50, 2000)
    H = HODLR(prob, perm, 64, 25)
    Ht = H.dense()
    Pinv = np.zeros_like(Ht)
    Pinv[np.ix_(perm, perm)] = np.linalg.inv(Ht)  # caller order
    u, it1, rr1, _, conv1 = gmres(lambda v: A @ (Pinv @ v), f, 1e-6, 50, 2000)
    psi = Pinv @ u
    assert conv0 and conv1 and it1 * 10 <= it0
    assert np.linalg.norm(A @ psi - f) / np.linalg.norm(f) <= 1.1e-6


def test_max_block_drops_top_blocks():
    """HR5: with max_block the blocks of more rows are zero in Ã (block diagonal at the top);
    the rest is the ordinary HODLR."""
    P, prob, perm = _case("c1", 32, 8.0)
    H = HODLR(prob, perm, 64, 8, max_block=256)
    Hd = H.dense()
    n = perm.size
    for _, a, b, c, d in sibling_blocks(n, 64):
        if b - a > 256:
            assert not np.any(Hd[a:b, c:d])
    full = HODLR(prob, perm, 64, 8)
    for key, (I, J) in H.pivots.items():
        if key[1] - key[0] <= 256:
            assert np.array_equal(I, full.pivots[key][0]) and np.array_equal(J, full.pivots[key][1])
