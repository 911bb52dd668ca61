"""Seeded workload generators for BASELINE.json configs 1-4 (plus scaled-down variants).

Grid: h = 2/n, x_ab = (-1 + (a+1/2) h, -1 + (b+1/2) h), a, b in [0, n),
row-major in b then a; weights w = h^2.  Input x_j = exp(i theta_j), theta ~ U[0, 2 pi)
from numpy default_rng(0).  Config-4 bump centres then amplitudes from default_rng(1).
Right-hand sides f = -kappa^2 q u_inc with a plane wave u_inc.
"""
import math

import numpy as np


def grid_points(n):
    h = 2.0 / n
    a = np.arange(n)
    c = -1.0 + (a + 0.5) * h
    xx, yy = np.meshgrid(c, c, indexing="xy")  # row-major in b (y) then a (x)
    pts = np.stack([xx.ravel(), yy.ravel()], axis=1)
    return pts, np.full(n * n, h * h)


def gaussian_q(pts):
    """q(x) = 1.5 exp(-160 |x|^2) (the Gaussian contrast of P:884)."""
    return 1.5 * np.exp(-160.0 * (pts[:, 0] ** 2 + pts[:, 1] ** 2))


def disk_q(pts, radius=0.5):
    """q = 1 inside the disk |x| < radius, else 0 (config 3)."""
    return (pts[:, 0] ** 2 + pts[:, 1] ** 2 < radius * radius).astype(np.float64)


def bumps_q(pts, seed=1, count=8):
    """Sum of `count` Gaussian bumps a_m exp(-200 |x - c_m|^2), c_m ~ U([-0.7,0.7]^2),
    a_m ~ U(0.5, 2), drawn centres first then amplitudes from default_rng(seed) (config 4)."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(-0.7, 0.7, size=(count, 2))
    amps = rng.uniform(0.5, 2.0, size=count)
    q = np.zeros(pts.shape[0])
    for c, a in zip(centres, amps):
        q += a * np.exp(-200.0 * ((pts[:, 0] - c[0]) ** 2 + (pts[:, 1] - c[1]) ** 2))
    return q


def unit_phase_vector(n, seed=0):
    rng = np.random.default_rng(seed)
    theta = rng.uniform(0.0, 2.0 * math.pi, size=n)
    return np.exp(1j * theta)


def plane_wave_rhs(pts, q, kappa, angle_deg=0.0):
    """f = -kappa^2 q exp(i kappa d.x), d = (cos a, sin a)."""
    a = math.radians(angle_deg)
    phase = kappa * (pts[:, 0] * math.cos(a) + pts[:, 1] * math.sin(a))
    return -kappa * kappa * q * np.exp(1j * phase)


def smoothed_disk_q(pts, radius=0.5, sharpness=200.0):
    """q = (1 + tanh(sharpness (radius - r))) / 2 (config 5; SURVEY A15 reading)."""
    r = np.sqrt(pts[:, 0] ** 2 + pts[:, 1] ** 2)
    return 0.5 * (1.0 + np.tanh(sharpness * (radius - r)))


def adaptive_leaves(kappa, max_depth, tol=1e-3, T=16.0, qfun=smoothed_disk_q, balance=True):
    """Leaves (level, i, j) of the config-5 quadtree on [-1,1]^2: split a box while
    max over its corners |q(corner) - q(centre)| > tol, up to max_depth, and (refinement rule 3,
    P:204) while it is in the high-frequency regime (kappa b)^2 > T, so every leaf is LFR; then
    (balance=True, the paper's level-restricted tree) level_restrict."""
    leaves, stack = [], [(0, 0, 0)]
    while stack:
        level, i, j = stack.pop()
        b = 2.0 / (1 << level)
        x0, y0 = -1.0 + i * b, -1.0 + j * b
        c = np.array([[x0, y0], [x0 + b, y0], [x0, y0 + b], [x0 + b, y0 + b]])
        qc = qfun(c)
        qm = qfun(np.array([[x0 + 0.5 * b, y0 + 0.5 * b]]))[0]
        split = level < max_depth and (np.max(np.abs(qc - qm)) > tol or (kappa * b) ** 2 > T)
        if split:
            stack += [(level + 1, 2 * i + di, 2 * j + dj) for dj in (1, 0) for di in (1, 0)]
        else:
            leaves.append((level, i, j))
    if balance:
        leaves = level_restrict(leaves)
    return sorted(leaves)


def _deepest_leaf(leafset, level, i, j):
    """Level of the deepest leaf inside box (level, i, j), or of the leaf covering it."""
    key = (level, i, j)
    if key in leafset:
        return level
    lv, a, b = level, i, j
    while lv > 0:  # a coarser leaf covers the box
        lv, a, b = lv - 1, a >> 1, b >> 1
        if (lv, a, b) in leafset:
            return lv
    best, stack = -1, [key]
    while stack:
        lv, a, b = stack.pop()
        for c in ((lv + 1, 2 * a + da, 2 * b + db) for db in (0, 1) for da in (0, 1)):
            if c in leafset:
                best = max(best, c[0])
            elif c[0] < 31:
                stack.append(c)
    return best


def level_restrict(leaves):
    """Level-restricted tree ("any two boxes that share a boundary are not more than
    one level apart"): split every leaf that touches (edge or corner) a leaf more than one level
    finer, until none does.  Splits only add resolution, so the refinement rules still hold."""
    leafset = set(leaves)
    changed = True
    while changed:
        changed = False
        for (level, i, j) in sorted(leafset):
            if (level, i, j) not in leafset:
                continue
            n = 1 << level
            deep = max((_deepest_leaf(leafset, level, i + di, j + dj)
                        for di in (-1, 0, 1) for dj in (-1, 0, 1)
                        if (di or dj) and 0 <= i + di < n and 0 <= j + dj < n), default=-1)
            if deep > level + 1:
                leafset.remove((level, i, j))
                leafset.update((level + 1, 2 * i + di, 2 * j + dj) for dj in (0, 1) for di in (0, 1))
                changed = True
    return sorted(leafset)


def adaptive_grid(leaves, per_side=8):
    """per_side x per_side cell-centred points in every leaf; weight = leaf area / per_side^2."""
    pts, w = [], []
    for level, i, j in leaves:
        b = 2.0 / (1 << level)
        h = b / per_side
        c = (np.arange(per_side) + 0.5) * h
        xx, yy = np.meshgrid(-1.0 + i * b + c, -1.0 + j * b + c, indexing="xy")
        pts.append(np.stack([xx.ravel(), yy.ravel()], axis=1))
        w.append(np.full(per_side * per_side, h * h))
    return np.concatenate(pts), np.concatenate(w)


# name -> (grid n, kappa, contrast, nca_tol, rhs angle, gmres tol)
CONFIGS = {
    "c1": dict(n=64, kappa=10.0, contrast="gaussian", nca_tol=1e-8, angle=0.0, gmres_tol=1e-8),
    "c2": dict(n=256, kappa=40.0, contrast="gaussian", nca_tol=1e-8, angle=0.0, gmres_tol=1e-8),
    "c3": dict(n=512, kappa=80.0, contrast="disk", nca_tol=1e-7, angle=30.0, gmres_tol=1e-6),
    "c4": dict(n=1024, kappa=160.0, contrast="bumps", nca_tol=1e-6, angle=0.0, gmres_tol=1e-6),
    # adaptive (n = max depth): q = smoothed disk, plane wave along x1, nca_tol unstated (1e-6)
    "c5": dict(n=10, kappa=200.0, contrast="smoothed_disk", nca_tol=1e-6, angle=0.0, gmres_tol=1e-6),
}


def l_shaped_problem(n=4000, kappa=40.0, seed=7, nca_tol=1e-8):
    """Seeded random points in the L-shaped domain [-1,1]^2 minus the quadrant x1, x2 > 0 (no
    lattice structure, ragged leaves, a re-entrant corner): the geometry on which directional
    nodes can be active only through their parent (reading R7).  Weights = area / n, q = 1 +
    0.5 cos(3 x1), x = unit-modulus seeded phases."""
    rng = np.random.default_rng(seed)
    pts = rng.uniform(-1.0, 1.0, size=(3 * n, 2))
    pts = pts[~((pts[:, 0] > 0) & (pts[:, 1] > 0))][:n]
    w = np.full(n, 3.0 / n)
    q = 1.0 + 0.5 * np.cos(3.0 * pts[:, 0])
    x = unit_phase_vector(n, seed=seed + 1)
    return dict(name="lshape", points=pts, weights=w, q=q, kappa=kappa, nca_tol=nca_tol, leaf_size=32, x=x,
                f=plane_wave_rhs(pts, q, kappa), gmres_tol=1e-8, n_grid=None)


def make_problem(name, n=None, kappa=None, balance=True):
    """Return dict(points, weights, q, kappa, nca_tol, leaf_size, x, f, gmres_tol) for a config.
    `n` / `kappa` override the grid size (the maximum depth for the adaptive config 5) and the
    wavenumber, for scaled-down variants; balance=False skips config 5's level restriction."""
    cfg = dict(CONFIGS[name])
    if n is not None:
        cfg["n"] = n
    if kappa is not None:
        cfg["kappa"] = kappa
    if cfg["contrast"] == "smoothed_disk":
        pts, w = adaptive_grid(adaptive_leaves(cfg["kappa"], cfg["n"], balance=balance))
    else:
        pts, w = grid_points(cfg["n"])
    q = {"gaussian": gaussian_q, "disk": disk_q, "bumps": bumps_q,
         "smoothed_disk": smoothed_disk_q}[cfg["contrast"]](pts)
    x = unit_phase_vector(pts.shape[0], seed=0)
    f = plane_wave_rhs(pts, q, cfg["kappa"], cfg["angle"])
    return dict(name=name, points=pts, weights=w, q=q, kappa=cfg["kappa"], nca_tol=cfg["nca_tol"],
                leaf_size=64, x=x, f=f, gmres_tol=cfg["gmres_tol"], n_grid=cfg["n"])
