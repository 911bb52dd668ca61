"""ORACLE — TEST INFRASTRUCTURE ONLY.  Quadtree, frequency regimes, cones and the
neighbour / interaction lists of the DAFMM.

Readings: R2 adaptive tree whose leaves are LFR (paper rule 3);
R3 T = 16; R4 w = circumradius b/sqrt(2) (w_reading="width": w = b, the alternative reading of
P:297-303); R5 nested cone geometry; R6 N(B) contains B.

Boxes are keyed (level, ix, iy) with integer lattice indices; only non-empty boxes exist.
Every list is a sorted Python list of keys; directional lists hold (key, cone) pairs.
"""
import math

import numpy as np

PHI0 = math.pi / 4096.0  # R5: cone boundaries at PHI0 + 2*pi*k/n (odd multiples of pi/4096)


def morton(ix, iy):
    """Interleave bits (x in even bits): Morton order of the children (0,0),(1,0),(0,1),(1,1)."""
    code = 0
    for bit in range(32):
        code |= ((ix >> bit) & 1) << (2 * bit)
        code |= ((iy >> bit) & 1) << (2 * bit + 1)
    return code


MAXL = 20  # points are binned on the 2^20 lattice once; a box at level l is that index >> (20 - l)


class Tree:
    """Adaptive quadtree over the root square of the points' quadrature cells.

    Root (R2): the smallest axis-aligned square containing every cell [x_j +- sqrt(w_j)/2]^2,
    centred on their bounding box.  A box is split while it holds more than leaf_size points
    or is in the high-frequency regime ((kappa b)^2 > T: refinement rule 3 of P:204, so every
    leaf is LFR), up to max_level.  Lattice index of a point: ix = floor(((x - x0) / W) 2^20),
    clamped; its box at level l is ix >> (20 - l).  For the uniform configs every leaf lies on
    one level L and the tree is the uniform tree.

    boxes[l]: {(ix, iy): sorted point indices} of the boxes that exist at level l (the root
    and the children of split boxes, non-empty); leaves[l]: the keys of boxes not split."""

    def __init__(self, points, weights, kappa, leaf_size, T=16.0, max_level=MAXL, w_reading="circumradius"):
        # R4: w of the HFR neighbour test and the cone angle is the box circumradius
        # b / sqrt(2); the alternative reading takes w = b, the width of P:279's regime test
        self.w_width = {"circumradius": False, "width": True}[w_reading]
        pts = np.asarray(points, dtype=np.float64).reshape(-1, 2)
        half = 0.5 * np.sqrt(np.asarray(weights, dtype=np.float64))
        lo_x, hi_x = float(np.min(pts[:, 0] - half)), float(np.max(pts[:, 0] + half))
        lo_y, hi_y = float(np.min(pts[:, 1] - half)), float(np.max(pts[:, 1] + half))
        self.W = max(hi_x - lo_x, hi_y - lo_y)
        cx, cy = 0.5 * (lo_x + hi_x), 0.5 * (lo_y + hi_y)
        self.x0, self.y0 = cx - 0.5 * self.W, cy - 0.5 * self.W
        self.kappa, self.T, self.n = float(kappa), float(T), pts.shape[0]
        self.points = pts
        self.fx, self.fy = self._lattice(pts, MAXL)
        self.boxes = [{(0, 0): np.arange(self.n)}]
        self.leaves = []
        level = 0
        while True:
            nxt, leaves = {}, set()
            for key, idx in self.boxes[level].items():
                split = (idx.size > leaf_size or self.is_hfr(level)) and level < max_level
                if not split:
                    if idx.size > leaf_size:
                        raise ValueError("leaf_size not reachable within max_level")
                    if self.is_hfr(level):  # refinement rule 3: leaves are LFR
                        raise ValueError("high-frequency box cannot be split within max_level")
                    leaves.add(key)
                    continue
                sh = MAXL - (level + 1)
                cxs, cys = self.fx[idx] >> sh, self.fy[idx] >> sh
                for c in range(4):
                    k = (2 * key[0] + (c & 1), 2 * key[1] + (c >> 1))
                    sel = idx[(cxs == k[0]) & (cys == k[1])]
                    if sel.size:
                        nxt[k] = sel
            self.leaves.append(leaves)
            if not nxt:
                break
            self.boxes.append(nxt)
            level += 1
        self.L = level  # deepest level

    def _lattice(self, pts, level):
        m = 1 << level
        ix = np.floor(((pts[:, 0] - self.x0) / self.W) * m).astype(np.int64)
        iy = np.floor(((pts[:, 1] - self.y0) / self.W) * m).astype(np.int64)
        return np.clip(ix, 0, m - 1), np.clip(iy, 0, m - 1)

    def is_leaf(self, level, key):
        return key in self.leaves[level]

    def all_leaves(self):
        """(level, key) of every leaf, coarse levels first, Morton order within a level."""
        return [(l, k) for l in range(self.L + 1) for k in self.keys(l) if k in self.leaves[l]]

    def leaf_descendants(self, level, key):
        """Leaves inside box (level, key), itself included when it is a leaf."""
        if key in self.leaves[level]:
            return [(level, key)]
        out = []
        for c in range(4):
            k = (2 * key[0] + (c & 1), 2 * key[1] + (c >> 1))
            if level + 1 <= self.L and k in self.boxes[level + 1]:
                out += self.leaf_descendants(level + 1, k)
        return out

    def width(self, level):
        return math.ldexp(self.W, -level)

    def kb(self, level):
        return self.kappa * self.width(level)

    def is_hfr(self, level):
        """a box of width w is HFR iff (kappa w)^2 > T."""
        kb = self.kb(level)
        return kb * kb > self.T

    def n_cones(self, level):
        """R5: smallest power of two n with half-angle pi/n <= 1/(kappa w), w = b/sqrt(2)."""
        x = math.pi * self.kb(level) if self.w_width else math.pi * self.kb(level) / math.sqrt(2.0)
        n = 1
        while n < x:
            n *= 2
        return n

    def keys(self, level):
        return sorted(self.boxes[level].keys(), key=lambda k: morton(*k))


def level_restricted(tree):
    """every two leaves that share a boundary (an edge or a corner) are at most one
    level apart.  Brute force over all leaf pairs by their closed squares (small trees)."""
    leaves = tree.all_leaves()
    sq = []
    for l, (i, j) in leaves:
        b = tree.width(l)
        sq.append((l, tree.x0 + i * b, tree.y0 + j * b, b))
    for p in range(len(sq)):
        lp, xp, yp, bp = sq[p]
        for q in range(len(sq)):
            lq, xq, yq, bq = sq[q]
            if lq <= lp + 1:
                continue
            touch = xp <= xq + bq + 1e-12 and xq <= xp + bp + 1e-12 and yp <= yq + bq + 1e-12 and yq <= yp + bp + 1e-12
            if touch:
                return False
    return True


def is_neighbor(tree, level, a, b):
    """N(B) membership: LFR — centres closer than 2b; HFR — centres closer than
    kappa w^2 with w = b/sqrt(2) (R4), i.e. |d| b < kappa b^2 / 2 (w = b: |d| < kappa b).
    d in lattice units."""
    dx, dy = a[0] - b[0], a[1] - b[1]
    d2 = dx * dx + dy * dy
    if tree.is_hfr(level):
        kb = tree.kb(level)
        return d2 < kb * kb if tree.w_width else 4.0 * d2 < kb * kb
    return d2 < 4


def cone_of(n, dx, dy):
    """Cone index k of the lattice offset (dx, dy): boundaries at PHI0 + 2 pi k / n (R5)."""
    a = math.atan2(dy, dx) - PHI0
    if a < 0.0:
        a += 2.0 * math.pi
    t = a * n / (2.0 * math.pi)
    k = int(math.floor(t))
    frac = t - k
    assert min(frac, 1.0 - frac) > 1e-9, "box centre on a cone boundary"
    return k % n


class Lists:
    """N(B), IL(B), IL(B,l), active nodes and the substitute lists of R7, for every level."""

    def __init__(self, tree):
        self.tree = tree
        L = tree.L
        self.N = [dict() for _ in range(L + 1)]
        self.IL = [dict() for _ in range(L + 1)]      # key -> sorted keys (LFR and HFR alike)
        self.ILdir = [dict() for _ in range(L + 1)]   # key -> {cone: sorted [(key, cone')]}
        for l in range(L + 1):
            boxes = tree.boxes[l]
            hfr = tree.is_hfr(l)
            reach = 1
            if hfr:
                reach = int(math.ceil(tree.kb(l) if tree.w_width else tree.kb(l) / 2.0)) + 1
            for b in boxes:
                nb = []
                for dx in range(-reach, reach + 1):
                    for dy in range(-reach, reach + 1):
                        a = (b[0] + dx, b[1] + dy)
                        if a in boxes and is_neighbor(tree, l, a, b):
                            nb.append(a)
                self.N[l][b] = sorted(nb)
        for l in range(1, L + 1):
            boxes = tree.boxes[l]
            for b in boxes:
                parent = (b[0] >> 1, b[1] >> 1)
                cand = set()
                for pn in self.N[l - 1][parent]:
                    for c in range(4):
                        a = (2 * pn[0] + (c & 1), 2 * pn[1] + (c >> 1))
                        if a in boxes:
                            cand.add(a)
                # P:376 / P:378: children of the parent's neighbours that are not neighbours of B
                near = set(self.N[l][b])
                il = sorted(a for a in cand if a not in near)
                self.IL[l][b] = il
                if tree.is_hfr(l):
                    n = tree.n_cones(l)
                    d = {}
                    for a in il:
                        k = cone_of(n, a[0] - b[0], a[1] - b[1])
                        kp = cone_of(n, b[0] - a[0], b[1] - a[1])
                        assert kp == (k + n // 2) % n
                        d.setdefault(k, []).append((a, kp))
                    self.ILdir[l][b] = {k: sorted(v) for k, v in d.items()}
        self._near_lists()
        self._activate()

    def _near_lists(self):
        """Near field of every leaf B at level l (R6), for an adaptive tree: the
        source leaves C whose ancestors at level min(l, l_C) are neighbours.  These are exactly
        the pairs no interaction list covers (the U, W and X lists of adaptive FMMs, all folded
        into the direct near field):
          - leaves C at a level m <= l that neighbour B's ancestor at level m (B itself included);
          - every leaf inside a non-leaf neighbour of B at level l."""
        tree = self.tree
        self.near = {}
        for l, b in tree.all_leaves():
            out = []
            for m in range(l, -1, -1):
                bm = (b[0] >> (l - m), b[1] >> (l - m))
                out += [(m, a) for a in self.N[m][bm] if a in tree.leaves[m]]
            for a in self.N[l][b]:
                if a not in tree.leaves[l]:
                    out += tree.leaf_descendants(l, a)
            self.near[(l, b)] = sorted(out)

    def _activate(self):
        """Active nodes, top-down: a node needs bases if its interaction list is non-empty or
        its parent's M2M / L2L needs it (passes run up to the coarsest level with a
        non-empty interaction list)."""
        tree = self.tree
        self.active = [set() for _ in range(tree.L + 1)]  # LFR: keys; HFR: (key, cone)
        for l in range(1, tree.L + 1):
            hfr = tree.is_hfr(l)
            parents_any = {nd[0] for nd in self.active[l - 1]} if tree.is_hfr(l - 1) else self.active[l - 1]
            for b in tree.boxes[l]:
                parent = (b[0] >> 1, b[1] >> 1)
                if hfr:
                    n = tree.n_cones(l)
                    for k in range(n):
                        need = bool(self.ILdir[l][b].get(k))
                        if l > 1 and tree.is_hfr(l - 1):
                            need = need or (parent, 2 * k) in self.active[l - 1] or \
                                (parent, 2 * k + 1) in self.active[l - 1]
                        if need:
                            self.active[l].add((b, k))
                else:
                    need = bool(self.IL[l][b])
                    if l > 1:
                        need = need or parent in parents_any
                    if need:
                        self.active[l].add(b)

    def far_list(self, level, node, parent_search=False):
        """Far-field list used for the search sets of an active node.

        It is IL(B) (LFR) or IL(B,l) (HFR).  R7: an active HFR node whose IL(B,l) is empty
        (active only because its parent needs it) uses the children, in the matching child
        cones, of its parent's IL in the two parent cones that nest in l.  R7b
        (parent_search=True): every HFR node with an HFR parent takes the union of its own
        IL(B,l) and those children."""
        tree = self.tree
        if not tree.is_hfr(level):
            return [(a, None) for a in self.IL[level][node]]
        b, k = node
        lst = self.ILdir[level][b].get(k, [])
        if lst and not (parent_search and level > 1 and tree.is_hfr(level - 1)):
            return lst
        if level <= 1 or not tree.is_hfr(level - 1):
            return lst
        parent = (b[0] >> 1, b[1] >> 1)
        sub = set(lst)
        for p in (2 * k, 2 * k + 1):
            for (a, ap) in self.ILdir[level - 1][parent].get(p, []):
                for c in range(4):
                    ac = (2 * a[0] + (c & 1), 2 * a[1] + (c >> 1))
                    if ac in tree.boxes[level]:
                        sub.add((ac, ap // 2))
        return sorted(sub)
