"""ORACLE — TEST INFRASTRUCTURE ONLY.  Reader for the plan files written by the product's
dafmm_export_plan (.npy files: tree, lists, cones, pivot index sets).

The oracle never takes the product's operators or vectors — only its *choices* (the pivot
index sets, of which several are correct), and only after checking them (``validate``).
Lists are recomputed by the oracle and compared exactly.
"""
import os

import numpy as np


def load_plan(path):
    """Return dict: meta, perm, and per level: boxes (keys), hfr, ncones, N, IL, ILdir, nodes,
    pivots {node_key: dict(ti, si, to, so)} with oracle node keys ((ix, iy) or ((ix, iy), cone))."""
    ld = lambda name: np.load(os.path.join(path, name))
    meta = ld("meta.npy")
    L = int(meta[1])
    out = dict(meta=dict(n=int(meta[0]), L=L, W=meta[2], x0=meta[3], y0=meta[4], kappa=meta[5], T=meta[6],
                         nca_tol=meta[7], hfr_parent_search=bool(meta[8]) if meta.size > 8 else False,
                         w_reading=int(meta[9]) if meta.size > 9 else 0),
               perm=ld("perm.npy"), levels=[])
    for l in range(L + 1):
        pre = "l%d_" % l
        boxes = [tuple(int(v) for v in b) for b in ld(pre + "boxes.npy").reshape(-1, 2)]
        hfr, ncones = (int(v) for v in ld(pre + "info.npy"))
        leaf = ld(pre + "leaf.npy")
        lv = dict(boxes=boxes, hfr=bool(hfr), ncones=ncones, leaves={b for b, f in zip(boxes, leaf) if f})

        def csr(name):
            ptr, idx = ld(pre + name + "_ptr.npy"), ld(pre + name + "_idx.npy")
            return {boxes[b]: sorted(boxes[a] for a in idx[ptr[b]:ptr[b + 1]]) for b in range(len(boxes))}

        lv["N"] = csr("N")
        if l >= 1:
            lv["IL"] = csr("IL")
            d = {}
            for b, k, a, kp in ld(pre + "ILdir.npy").reshape(-1, 4):
                d.setdefault(boxes[b], {}).setdefault(int(k), []).append((boxes[a], int(kp)))
            lv["ILdir"] = {b: {k: sorted(v) for k, v in dd.items()} for b, dd in d.items()}
            nodes = ld(pre + "nodes.npy").reshape(-1, 2)
            keys = [(boxes[b], int(k)) if hfr else boxes[b] for b, k in nodes]
            piv = {}
            ptrs = {s: (ld(pre + s + "_ptr.npy"), ld(pre + s + "_idx.npy")) for s in ("ti", "si", "to", "so")}
            for i, key in enumerate(keys):
                piv[key] = {s: ptrs[s][1][ptrs[s][0][i]:ptrs[s][0][i + 1]].astype(np.int64) for s in ptrs}
            lv["nodes"] = keys
            lv["pivots"] = piv
        out["levels"].append(lv)
    # near field: leaf (level, key) -> source boxes (level, key) (non-leaf boxes stand for all
    # their leaves)
    lvs = out["levels"]
    leaves = [(int(l), lvs[int(l)]["boxes"][int(b)]) for l, b in ld("leaves.npy").reshape(-1, 2)]
    ptr, src = ld("near_ptr.npy"), ld("near_src.npy").reshape(-1, 2)
    out["near"] = {leaves[i]: [(int(l), lvs[int(l)]["boxes"][int(b)]) for l, b in src[ptr[i]:ptr[i + 1]]]
                   for i in range(len(leaves))}
    return out


def compare_lists(plan, tree, lists):
    """Exact equality of the product's tree and lists with the oracle's own (raises on mismatch)."""
    assert plan["meta"]["L"] == tree.L
    assert (plan["meta"]["W"], plan["meta"]["x0"], plan["meta"]["y0"]) == (tree.W, tree.x0, tree.y0)
    for l, lv in enumerate(plan["levels"]):
        assert sorted(lv["boxes"]) == sorted(tree.boxes[l].keys()), "boxes differ at level %d" % l
        assert lv["leaves"] == tree.leaves[l], "leaves differ at level %d" % l
        assert lv["hfr"] == tree.is_hfr(l)
        if lv["hfr"]:
            assert lv["ncones"] == tree.n_cones(l)
        for b, nb in lv["N"].items():
            assert nb == lists.N[l][b], "N differs at level %d box %s" % (l, b)
        if l >= 1:
            for b, il in lv["IL"].items():
                assert il == lists.IL[l][b], "IL differs at level %d box %s" % (l, b)
            if lv["hfr"]:
                for b in tree.boxes[l]:
                    assert lv["ILdir"].get(b, {}) == lists.ILdir[l][b], "IL(B,l) differs at %d %s" % (l, b)
            assert set(lv["nodes"]) == lists.active[l], "active nodes differ at level %d" % l
    # near field: the same source leaves for every leaf (compared as sets of leaves)
    assert set(plan["near"]) == set(lists.near), "near-field leaves differ"
    for b, src in plan["near"].items():
        got = sorted(c for m, a in src for c in tree.leaf_descendants(m, a))
        assert got == sorted(lists.near[b]), "near field of leaf %s differs" % (b,)


def validate_pivots(nca_like, pivots):
    """Check imported pivots against the oracle's own search sets: containment,
    |t| = |s|, non-singular cross matrices.  ``nca_like`` is an oracle NCA built on them."""
    from .core import K_block
    for level in range(1, len(pivots)):
        for node, p in pivots[level].items():
            s = nca_like.search[level][node]
            for key in ("ti", "si", "to", "so"):
                assert np.all(np.isin(p[key], s[key])), "pivot %s outside its search set" % key
                assert len(np.unique(p[key])) == len(p[key])
            assert len(p["ti"]) == len(p["si"]) and len(p["to"]) == len(p["so"])
            for a, b in (("ti", "si"), ("to", "so")):
                if len(p[a]):
                    M = K_block(nca_like.prob, p[a], p[b])
                    assert np.linalg.matrix_rank(M) == len(p[a]), "singular cross matrix"
