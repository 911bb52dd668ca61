"""Pins for the oracle's dense product (P:251-263 point form + D1) and GMRES (R14)."""
import math

import mpmath as mp
import numpy as np
import scipy.sparse.linalg as spla

import oracle
from oracle.core import Problem
from oracle.gmres import gmres
from synth.configs import make_problem


def test_dense_two_points_closed_form():
    """N = 2: y_0 = x_0 + k^2 q_0 [ (i/4) H0(k r) w_1 x_1 + D_0 x_0 ] with H0 from mpmath."""
    pts = np.array([[0.1, -0.2], [0.4, 0.2]])
    w = np.array([0.01, 0.02])
    q = np.array([0.7, 1.3])
    kappa = 7.0
    x = np.array([1.0 + 2.0j, -0.5 + 0.25j])
    prob = Problem(pts, w, q, kappa)
    y = oracle.dense_matvec(prob, x)
    r = 0.5
    with mp.workdps(30):
        G = complex(0.25j * mp.hankel1(0, kappa * r))
        R0 = math.sqrt(w[0] / math.pi)
        D0 = complex(0.5j * mp.pi * mp.quad(lambda rho: mp.hankel1(0, kappa * rho) * rho, [0, R0]))
    y0 = x[0] + kappa ** 2 * q[0] * (G * w[1] * x[1] + D0 * x[0])
    assert abs(y[0] - y0) / abs(y0) < 1e-13


def test_dense_zero_contrast_is_identity_and_linear():
    P = make_problem("c1", n=24, kappa=6.0)
    prob0 = Problem(P["points"], P["weights"], np.zeros(576), P["kappa"])
    assert np.array_equal(oracle.dense_matvec(prob0, P["x"]), P["x"])
    prob = Problem(P["points"], P["weights"], P["q"], P["kappa"])
    A = np.stack([oracle.dense_matvec(prob, e) for e in np.eye(576, dtype=complex)[:40]], axis=1)
    Ablk = oracle.A_block(prob, np.arange(576), np.arange(40))
    assert np.allclose(A, Ablk, rtol=1e-14, atol=1e-16)


def test_gmres_identity_one_iteration():
    f = np.exp(1j * np.arange(50))
    psi, it, rr, hist, conv = gmres(lambda v: v, f, 1e-12)
    assert it == 1 and conv and np.allclose(psi, f, rtol=1e-15)


def test_gmres_manufactured_solution_dense_ls():
    """Manufactured psi* on the dense LS operator (N = 1024): f = A psi*, recover psi*; the
    residual history is non-increasing; exit relres equals the recomputed one;
    the solution agrees with scipy's independent GMRES."""
    P = make_problem("c1", n=32, kappa=5.0)
    prob = Problem(P["points"], P["weights"], P["q"], P["kappa"])
    A = oracle.A_block(prob, np.arange(1024), np.arange(1024))
    rng = np.random.default_rng(4)
    psi_star = rng.standard_normal(1024) + 1j * rng.standard_normal(1024)
    f = A @ psi_star
    psi, it, rr, hist, conv = gmres(lambda v: A @ v, f, 1e-12, restart=50, maxit=500)
    assert conv and rr <= 1e-11
    assert np.all(np.diff(hist) <= 1e-15)
    assert np.linalg.norm(psi - psi_star) / np.linalg.norm(psi_star) <= np.linalg.cond(A) * 1e-11
    assert abs(np.linalg.norm(f - A @ psi) / np.linalg.norm(f) - rr) < 1e-15
    ref, info = spla.gmres(A, f, rtol=1e-12, restart=50, maxiter=50)
    assert info == 0 and np.linalg.norm(psi - ref) / np.linalg.norm(ref) < 1e-9
