"""Pins for the oracle's tree, regimes, cones and lists (readings R2-R7)."""
import math

import numpy as np
import pytest

from oracle.tree import Tree, Lists, cone_of
from synth.configs import make_problem


def _build(name, n=None, kappa=None):
    P = make_problem(name, n=n, kappa=kappa)
    tree = Tree(P["points"], P["weights"], P["kappa"], 64)
    return P, tree, Lists(tree)


def _cover_matrix(tree, lists):
    """How often each ordered pair of leaves (target, source) is covered: by the near field of
    the target leaf, or by an interaction-list pair (level, B, A) of boxes containing them."""
    leaves = tree.all_leaves()
    idx = {k: i for i, k in enumerate(leaves)}
    under = {}
    for l in range(tree.L + 1):
        for key in tree.boxes[l]:
            under[(l, key)] = [idx[c] for c in tree.leaf_descendants(l, key)]
    cover = np.zeros((len(leaves), len(leaves)), dtype=np.int64)
    for b, near in lists.near.items():
        for a in near:
            cover[idx[b], idx[a]] += 1
    for l in range(1, tree.L + 1):
        for b, il in lists.IL[l].items():
            for a in il:
                for i in under[(l, b)]:
                    cover[i, under[(l, a)]] += 1
    return cover


@pytest.mark.parametrize("name,n,kappa", [("c1", None, None), ("c2", 128, 20.0), ("c1", 64, 3.0), ("c5", 5, 12.0),
                                          ("c5", 5, 8.0), ("c5", 6, 30.0)])
def test_pair_completeness(name, n, kappa):
    """Every ordered pair of leaves is covered exactly once: by the target leaf's near field, or
    by exactly one (level, ancestor pair) of an interaction list (FMM partition of A,
    P:643-755).  The c5 cases are adaptive trees with leaves on several levels."""
    _, tree, lists = _build(name, n, kappa)
    cover = _cover_matrix(tree, lists)
    assert cover.min() == 1 and cover.max() == 1


def test_adaptive_tree_structure():
    """Config-5 tree (scaled): leaves on levels 3-5, all LFR (rule 3), 64 points each,
    points of every box contiguous in a Morton-ordered permutation."""
    P, tree, lists = _build("c5", 5, 12.0)
    levels = sorted({l for l, _ in tree.all_leaves()})
    assert levels == [3, 4, 5]
    for l, k in tree.all_leaves():
        assert not tree.is_hfr(l) and tree.boxes[l][k].size == 64
    n = sum(tree.boxes[l][k].size for l, k in tree.all_leaves())
    assert n == P["points"].shape[0]


def test_config1_pair_counts():
    """Counts of SURVEY 8(a) for C1: 484 near leaf pairs, 2396 LFR + 76 directional IL pairs."""
    _, tree, lists = _build("c1")
    assert tree.L == 3
    assert sum(len(v) for v in lists.N[3].values()) == 484
    assert sum(len(v) for v in lists.IL[3].values()) == 2396
    assert sum(len(v) for v in lists.IL[2].values()) == 76
    assert [tree.is_hfr(l) for l in range(4)] == [True, True, True, False]


def test_lists_symmetric_and_cones_opposite():
    _, tree, lists = _build("c2", 128, 20.0)
    for l in range(1, tree.L + 1):
        for b, il in lists.IL[l].items():
            for a in il:
                assert b in lists.IL[l][a]
            for a in lists.N[l][b]:
                assert b in lists.N[l][a]
        if tree.is_hfr(l):
            n = tree.n_cones(l)
            for b, d in lists.ILdir[l].items():
                flat = sorted(a for k, v in d.items() for a, _ in v)
                assert flat == lists.IL[l][b]  # cones partition IL(B)
                for k, v in d.items():
                    for a, kp in v:
                        assert kp == (k + n // 2) % n
                        assert (b, k) in lists.ILdir[l][a][kp]


def test_cone_geometry():
    """R5: n_l = smallest power of two >= pi kb / sqrt(2); parent has twice the child's cones;
    parent cone j nests in child cone j // 2."""
    _, tree, _ = _build("c2", 128, 20.0)
    for l in range(tree.L):
        if tree.is_hfr(l) and tree.is_hfr(l + 1):
            assert tree.n_cones(l) == 2 * tree.n_cones(l + 1)
        if tree.is_hfr(l):
            n = tree.n_cones(l)
            assert math.pi / n <= math.sqrt(2) / tree.kb(l)  # half-angle <= 1/(kappa w)
            assert math.pi / (n // 2) > math.sqrt(2) / tree.kb(l)
    rng = np.random.default_rng(2)
    for _ in range(200):
        dx, dy = rng.integers(-40, 41, size=2)
        if dx == 0 and dy == 0:
            continue
        n = 32
        assert cone_of(2 * n, dx, dy) // 2 == cone_of(n, dx, dy)


def test_regimes_and_neighbours():
    _, tree, lists = _build("c2", 128, 20.0)
    for l in range(tree.L + 1):
        kb = tree.kb(l)
        assert tree.is_hfr(l) == (kb * kb > 16.0)
        for b, nb in lists.N[l].items():
            assert b in nb  # R6
            for a in nb:
                d = math.hypot(a[0] - b[0], a[1] - b[1]) * tree.width(l)
                if tree.is_hfr(l):
                    assert d < tree.kappa * (tree.width(l) / math.sqrt(2)) ** 2 + 1e-12
                else:
                    assert d < 2 * tree.width(l)


def test_root_and_leaf_level():
    P, tree, _ = _build("c1")
    assert (tree.x0, tree.y0, tree.W) == (-1.0, -1.0, 2.0)
    assert all(len(v) == 64 for v in tree.boxes[tree.L].values())
    # rule 3: leaves must be LFR even when leaf_size would stop earlier
    t2 = Tree(P["points"], P["weights"], 80.0, 4096)
    assert not t2.is_hfr(t2.L) and t2.is_hfr(t2.L - 1)


@pytest.mark.parametrize("name,n,kappa", [("c1", None, None), ("c2", 128, 40.0), ("c5", 5, 12.0)])
def test_pair_completeness_width_reading(name, n, kappa):
    """w_reading = width (w = b in P:297-303 instead of the circumradius, R4): still an exact
    partition of all leaf pairs."""
    P = make_problem(name, n=n, kappa=kappa)
    tree = Tree(P["points"], P["weights"], P["kappa"], 64, w_reading="width")
    cover = _cover_matrix(tree, Lists(tree))
    assert cover.min() == 1 and cover.max() == 1


def test_width_reading_pair_counts_and_geometry():
    """SURVEY App. A.2 (T = 16): C1 has 3612 IL box pairs over all levels with w = width against
    2472 with the circumradius; HFR neighbours lie within kappa b^2 and the cones have
    half-angle <= 1/(kappa b)."""
    P = make_problem("c1")
    counts = {}
    for wr in ("circumradius", "width"):
        tree = Tree(P["points"], P["weights"], P["kappa"], 64, w_reading=wr)
        lists = Lists(tree)
        counts[wr] = sum(len(v) for l in range(1, tree.L + 1) for v in lists.IL[l].values())
    assert counts == {"circumradius": 2472, "width": 3612}
    P, tree = make_problem("c2", n=128, kappa=40.0), None
    tree = Tree(P["points"], P["weights"], P["kappa"], 64, w_reading="width")
    lists = Lists(tree)
    for l in range(tree.L + 1):
        if not tree.is_hfr(l):
            continue
        b = tree.width(l)
        assert math.pi / tree.n_cones(l) <= 1.0 / (tree.kappa * b) + 1e-15
        for key, nb in lists.N[l].items():
            for a in nb:
                assert math.hypot(a[0] - key[0], a[1] - key[1]) * b < tree.kappa * b * b


def test_level_restricted_config5_trees():
    """the paper's adaptive tree is level restricted.  The config-5 generator balances
    its refinement (synth.configs.level_restrict); without it the same refinement rules leave
    leaves two or more levels apart across the contrast's transition layer."""
    from oracle.tree import level_restricted
    for n, kappa in [(5, 12.0), (6, 30.0)]:
        P = make_problem("c5", n=n, kappa=kappa)
        tree = Tree(P["points"], P["weights"], P["kappa"], 64)
        assert level_restricted(tree)
        P0 = make_problem("c5", n=n, kappa=kappa, balance=False)
        tree0 = Tree(P0["points"], P0["weights"], P0["kappa"], 64)
        assert not level_restricted(tree0)
