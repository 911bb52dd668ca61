"""CPU checks of the C-ABI library (no GPU, no compute calls on the device): it loads, exports
every function include/dafmm.h declares, rejects bad arguments, and its host setup (tree,
lists, cones, NCA pivots) agrees with the oracle's own construction."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle.core import Problem
from oracle.nca import NCA
from oracle.plan_io import compare_lists, load_plan, validate_pivots
from oracle.tree import Lists, Tree
from synth.configs import make_problem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _prod():
    import paper_2204_00326_b200 as prod
    return prod


def _declared():
    src = open(os.path.join(ROOT, "include", "dafmm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(?:int|void|const char\*)\s+(\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    prod = _prod()
    lib = ctypes.CDLL(prod.library_path())
    names = _declared()
    assert "dafmm_create" in names and "ls_gmres_solve" in names and "dafmm_matvec" in names
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(prod.EXPORTED) == names


def _host_plan(P, tmp_path, **opts):
    prod = _prod()
    op = prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"], host_only=1, **opts)
    op.export_plan(tmp_path / "plan")
    stats = op.stats()
    op.close()
    return load_plan(tmp_path / "plan"), stats


@pytest.mark.parametrize("name,n,kappa", [("c1", None, None), ("c2", 128, 20.0), ("c3", 128, 20.0), ("c5", 5, 12.0),
                                          ("c5", 5, 8.0), ("c5", 6, 30.0)])
def test_host_setup_matches_oracle_lists_and_pivots(name, n, kappa, tmp_path):
    P = make_problem(name, n=n, kappa=kappa)
    plan, stats = _host_plan(P, tmp_path)
    tree = Tree(P["points"], P["weights"], P["kappa"], 64)
    lists = Lists(tree)
    compare_lists(plan, tree, lists)
    if (name, n) != ("c5", 6):  # the three-level adaptive case checks tree and lists only (the pivot
        # validation of its points takes over a minute; the depth-5 adaptive cases above validate pivots)
        piv = [dict()] + [plan["levels"][l]["pivots"] for l in range(1, tree.L + 1)]
        prob = Problem(P["points"], P["weights"], P["q"], P["kappa"])
        nca = NCA(prob, tree, lists, P["nca_tol"], pivots=piv)
        validate_pivots(nca, piv)
    assert stats["p2p_pairs"] > 0 and stats["levels"] == tree.L
    assert np.array_equal(np.sort(plan["perm"]), np.arange(P["points"].shape[0]))


def test_host_setup_symmetric_pivots(tmp_path):
    """R19: with symmetric_pivots=1 the outgoing skeleton is the incoming one swapped; with 0
    (default) the two ACAs run separately.  Both pass the oracle's validation."""
    P = make_problem("c1")
    plan, _ = _host_plan(P, tmp_path, symmetric_pivots=1)
    for piv in plan["levels"][3]["pivots"].values():
        assert np.array_equal(piv["so"], piv["ti"]) and np.array_equal(piv["to"], piv["si"])
    plan2, _ = _host_plan(P, tmp_path / "b")
    tree = Tree(P["points"], P["weights"], P["kappa"], 64)
    lists = Lists(tree)
    piv = [dict()] + [plan2["levels"][l]["pivots"] for l in range(1, tree.L + 1)]
    prob = Problem(P["points"], P["weights"], P["q"], P["kappa"])
    validate_pivots(NCA(prob, tree, lists, P["nca_tol"], pivots=piv), piv)


def test_host_setup_ragged_points(tmp_path):
    rng = np.random.default_rng(7)
    pts = rng.uniform(-1, 1, size=(3000, 2))
    P = dict(points=pts, weights=np.full(3000, 4.0 / 3000), q=np.ones(3000), kappa=12.0, nca_tol=1e-8)
    plan, _ = _host_plan(P, tmp_path)
    tree = Tree(pts, P["weights"], 12.0, 64)
    compare_lists(plan, tree, Lists(tree))


@pytest.mark.parametrize("bad", ["kappa", "tol", "dup", "nan", "weight", "leaf"])
def test_invalid_arguments_rejected(bad):
    prod = _prod()
    P = make_problem("c1", n=16)
    pts, w, q, kappa, tol, leaf = P["points"].copy(), P["weights"].copy(), P["q"].copy(), 5.0, 1e-8, 64
    if bad == "kappa":
        kappa = -1.0
    elif bad == "tol":
        tol = 1.5
    elif bad == "dup":
        pts[3] = pts[2]
    elif bad == "nan":
        q[5] = np.nan
    elif bad == "weight":
        w[0] = 0.0
    elif bad == "leaf":
        leaf = 0
    with pytest.raises(prod.DAFMMError) as e:
        prod.DAFMM(pts, w, q, kappa, leaf, tol, host_only=1)
    assert e.value.code == -1
    assert prod.dafmm_last_error() != ""


def test_host_only_plan_refuses_device_calls():
    prod = _prod()
    P = make_problem("c1", n=16)
    op = prod.DAFMM(P["points"], P["weights"], P["q"], 5.0, 64, 1e-8, host_only=1)
    with pytest.raises(prod.DAFMMError):
        prod.dafmm_matvec(op.h, 1, 2)
    with pytest.raises(prod.DAFMMError):
        op.set_profiling(True)
    op.close()


def test_h0_band_table():
    """dafmm_h0_bands (host only): the near bands are (0, 7], (0, 8], (0, 12]; the data bands are
    finite positive intervals inside the generic band's (0, inf) and overlap so that every z
    beyond the near bands is covered by some data band up to the largest one's end."""
    from paper_2204_00326_b200 import binding
    bands = binding.dafmm_h0_bands()
    assert bands[0] == (0.0, float("inf"))
    assert bands[1] == (0.0, 8.0) and bands[2] == (0.0, 12.0) and bands[3] == (0.0, 7.0)
    data = sorted(bands[4:])
    assert len(data) >= 1
    for lo, hi in data:
        assert 0.0 < lo < hi < float("inf")
    reach = 12.0
    for lo, hi in data:
        if lo <= reach:
            reach = max(reach, hi)
    assert reach >= max(hi for _, hi in data) * 0.999


def test_m2l_store_option_validated():
    """dafmm_options.m2l_store takes -1 (auto), 0 or 1; anything else is DAFMM_EINVAL."""
    from paper_2204_00326_b200 import binding
    P = make_problem("c1", n=16)
    assert binding.default_options().m2l_store == -1
    with pytest.raises(binding.DAFMMError):
        binding.DAFMM(P["points"], P["weights"], P["q"], 5.0, 64, 1e-8, host_only=1, m2l_store=2)
    op = binding.DAFMM(P["points"], P["weights"], P["q"], 5.0, 64, 1e-8, host_only=1, m2l_store=1)
    st = op.stats()
    assert st["m2l_stored"] == 0 and st["m2l_store_bytes"] == 0  # host-only plan: nothing on a device


def test_symmetric_near_field_flag():
    """The symmetric near field is used exactly when every leaf has 32 or 64 points (the P2P
    CTA's slices are then whole warps); ragged leaves fall back to the one-sided near field."""
    from paper_2204_00326_b200 import binding
    P = make_problem("c1")
    op = binding.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, 1e-8, host_only=1)
    assert op.stats()["p2p_symmetric"] == 1
    rng = np.random.default_rng(7)
    pts = rng.uniform(-1, 1, size=(3000, 2))
    op = binding.DAFMM(pts, np.full(3000, 4.0 / 3000), np.ones(3000), 12.0, 64, 1e-8, host_only=1)
    assert op.stats()["p2p_symmetric"] == 0


def test_hfr_box_at_max_level_rejected():
    """Refinement rule 3: every leaf must be LFR.  A max_level that stops the tree while
    its boxes are still in the high-frequency regime is an error (it would otherwise silently
    drop the far field of such leaves); the oracle's tree refuses the same input."""
    prod = _prod()
    P = make_problem("c1", n=64, kappa=160.0)  # level-3 boxes: kappa b = 40 (HFR)
    with pytest.raises(prod.DAFMMError) as e:
        prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 4096, 1e-6, host_only=1, max_level=3)
    assert e.value.code == -1 and "max_level" in prod.dafmm_last_error()
    with pytest.raises(ValueError):
        Tree(P["points"], P["weights"], P["kappa"], 4096, max_level=3)
    # an LFR stop is fine: leaf_size 4096 holds the whole grid, kappa = 1 keeps the root LFR
    op = prod.DAFMM(P["points"], P["weights"], P["q"], 1.0, 4096, 1e-6, host_only=1, max_level=3)
    assert op.stats()["levels"] == 0
    op.close()


def test_host_setup_l_shaped_parent_search(tmp_path):
    """Reading R7b (hfr_parent_search=1) on the L-shaped random point set: the product's lists
    equal the oracle's and its pivots lie in the oracle's R7b search sets; with the option off
    the plan is the paper's (search sets of P:624-631 only)."""
    from synth.configs import l_shaped_problem
    P = l_shaped_problem()
    prod = _prod()
    for flag in (1, 0):
        op = prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], P["leaf_size"], P["nca_tol"], host_only=1,
                        hfr_parent_search=flag)
        op.export_plan(tmp_path / ("plan%d" % flag))
        op.close()
        plan = load_plan(tmp_path / ("plan%d" % flag))
        assert plan["meta"]["hfr_parent_search"] == bool(flag)
        tree = Tree(P["points"], P["weights"], P["kappa"], P["leaf_size"])
        lists = Lists(tree)
        compare_lists(plan, tree, lists)
        piv = [dict()] + [plan["levels"][l]["pivots"] for l in range(1, tree.L + 1)]
        prob = Problem(P["points"], P["weights"], P["q"], P["kappa"])
        validate_pivots(NCA(prob, tree, lists, P["nca_tol"], pivots=piv, hfr_parent_search=bool(flag)), piv)


def test_binding_rejects_bad_host_vectors():
    """dafmm_matvec_host takes C-contiguous complex128 host arrays of exactly n elements; the
    binding refuses anything else before the library could read or write past them."""
    from paper_2204_00326_b200 import binding
    P = make_problem("c1", n=16)
    op = binding.DAFMM(P["points"], P["weights"], P["q"], 5.0, 64, 1e-8, host_only=1)
    good = np.zeros(256, dtype=np.complex128)
    for bad in (np.zeros(255, dtype=np.complex128), np.zeros(512, dtype=np.complex128)[::2],
                np.zeros(256, dtype=np.float64)):
        with pytest.raises(ValueError):
            op.matvec_host(bad, good)
        with pytest.raises(ValueError):
            op.matvec_host(good, bad)
    ro = np.zeros(256, dtype=np.complex128)
    ro.flags.writeable = False
    with pytest.raises(ValueError):
        op.matvec_host(good, ro)
    op.close()


@pytest.mark.parametrize("mode,code", [("disk", 1), ("square", 2), ("zero", 0)])
def test_host_self_terms_match_oracle(mode, code, tmp_path):
    """The product's self terms D_i (exported with the plan) against the oracle's: the disk
    closed form (D1), the square-cell integral (Eq. 13's cell) and zero; ragged weights."""
    import numpy as np
    from oracle.core import self_terms
    P = make_problem("c5", n=5, kappa=12.0)  # adaptive: several cell sizes
    prod = _prod()
    op = prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"], host_only=1, self_term=code)
    op.export_plan(tmp_path / "plan")
    op.close()
    D = np.load(tmp_path / "plan" / "self.npy")
    ref = self_terms(P["weights"], P["kappa"], mode)
    if mode == "zero":
        assert np.all(D == 0)
    else:
        assert np.max(np.abs(D - ref) / np.abs(ref)) < 1e-13


@pytest.mark.parametrize("name,n,kappa", [("c1", None, None), ("c2", 128, 40.0)])
def test_host_width_reading_lists_match_oracle(name, n, kappa, tmp_path):
    """w_reading = 1 (w = b in P:297-303): the product's tree, neighbour, interaction and
    directional lists equal the oracle's under the same reading, and its pivots validate."""
    P = make_problem(name, n=n, kappa=kappa)
    plan, _ = _host_plan(P, tmp_path, w_reading=1)
    assert plan["meta"]["w_reading"] == 1
    tree = Tree(P["points"], P["weights"], P["kappa"], 64, w_reading="width")
    lists = Lists(tree)
    compare_lists(plan, tree, lists)
    piv = [dict()] + [plan["levels"][l]["pivots"] for l in range(1, tree.L + 1)]
    prob = Problem(P["points"], P["weights"], P["q"], P["kappa"])
    validate_pivots(NCA(prob, tree, lists, P["nca_tol"], pivots=piv), piv)


@pytest.mark.parametrize("balance", [True, False])
def test_host_level_restricted_flag_matches_oracle(balance):
    """dafmm_stats.level_restricted against the oracle's brute-force check."""
    from oracle.tree import level_restricted
    P = make_problem("c5", n=5, kappa=12.0, balance=balance)
    prod = _prod()
    op = prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"], host_only=1)
    flag = op.stats()["level_restricted"]
    op.close()
    tree = Tree(P["points"], P["weights"], P["kappa"], 64)
    assert flag == int(level_restricted(tree)) == int(balance)
