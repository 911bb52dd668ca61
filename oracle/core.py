"""ORACLE — TEST INFRASTRUCTURE ONLY.  ctypes front end of oracle/src/oracle_core.c.

The C file holds the special functions and the entries of A; this module only marshals
arguments.  The library is compiled by __graft_entry__.build() (or on first use here with
gcc), never by the product build.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "src", "oracle_core.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build_library(force=False):
    """Compile oracle/src/oracle_core.c -> oracle/liboracle.so with gcc (OpenMP over rows)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB_PATH, _SRC, "-lm"])
    return _LIB_PATH


def load_library():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_library())
        vp, i64, dbl, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        _lib.oracle_h0.argtypes = [vp, i64, vp]
        _lib.oracle_h1_small.argtypes = [vp, i64, vp]
        _lib.oracle_self_terms.argtypes = [vp, i64, dbl, i32, vp]
        _lib.oracle_A_block.argtypes = [vp, i64, vp, i64, vp, vp, vp, vp, dbl, vp]
        _lib.oracle_K_block.argtypes = [vp, i64, vp, i64, vp, vp, vp, dbl, vp]
        _lib.oracle_dense_matvec_rows.argtypes = [vp, i64, vp, vp, vp, vp, dbl, i64, vp, vp]
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def h0(z):
    """H0^(1)(z) for an array of z > 0 (three bands, see oracle_core.c)."""
    z = _f64(np.atleast_1d(z))
    out = np.empty(z.size, dtype=np.complex128)
    load_library().oracle_h0(_p(z), z.size, _p(out))
    return out


def h1_small(z):
    """H1^(1)(z) by its ascending series (small z only; used for the self term)."""
    z = _f64(np.atleast_1d(z))
    out = np.empty(z.size, dtype=np.complex128)
    load_library().oracle_h1_small(_p(z), z.size, _p(out))
    return out


SELF_TERM_MODES = {"zero": 0, "disk": 1, "square": 2}


def self_term_square(w, kappa):
    """D_i = integral of G(0, y) = (i/4) H0(kappa |y|) over the square cell of side h = sqrt(w_i)
    centred on the point (Eq. 13 integrates G over the cell).  By symmetry the square is
    8 triangles 0 <= theta <= pi/4, 0 <= rho <= R(theta) = h / (2 cos theta); the radial integral
    is exact, int_0^R H0(k rho) rho d rho = (k R H1(k R) + 2i/pi) / k^2 (d/dz [z H1(z)] = z H0(z),
    z H1(z) -> -2i/pi as z -> 0), and the smooth angular one is Gauss-Legendre (40 nodes)."""
    w = _f64(np.atleast_1d(w))
    k = float(kappa)
    x, gw = np.polynomial.legendre.leggauss(40)
    theta = (x + 1.0) * (np.pi / 8.0)
    out = np.empty(w.size, dtype=np.complex128)
    for i, wi in enumerate(w):
        z = k * np.sqrt(wi) / (2.0 * np.cos(theta))
        radial = (z * h1_small(z) + 2j / np.pi) / (k * k)
        out[i] = 0.25j * 8.0 * (np.pi / 8.0) * np.dot(gw, radial)
    return out


def self_terms(weights, kappa, mode="disk"):
    """D_i of reading D1: integral of G over the equal-area disk of weight w_i (mode 'disk'),
    over the square cell of side sqrt(w_i) (mode 'square', self_term_square), or 0 (mode
    'zero', the point-kernel N-body of Experiment 1)."""
    w = _f64(weights)
    if mode == "square":
        return self_term_square(w, kappa)
    out = np.empty(w.size, dtype=np.complex128)
    load_library().oracle_self_terms(_p(w), w.size, float(kappa), SELF_TERM_MODES[mode], _p(out))
    return out


class Problem:
    """The discrete operator's data: points (N,2), weights w, contrast q, kappa, self terms D."""

    def __init__(self, points, weights, q, kappa, self_term="disk"):
        self.points = _f64(points).reshape(-1, 2)
        self.w = _f64(weights)
        self.q = _f64(q)
        self.kappa = float(kappa)
        self.n = self.points.shape[0]
        self.D = self_terms(self.w, self.kappa, self_term)


def A_block(prob, rows, cols):
    """A[rows, cols] (P:251-263 in point form; diagonal per D1), complex (len(rows), len(cols))."""
    rows, cols = _i64(rows), _i64(cols)
    out = np.empty((rows.size, cols.size), dtype=np.complex128)
    if rows.size and cols.size:
        load_library().oracle_A_block(_p(rows), rows.size, _p(cols), cols.size, _p(prob.points), _p(prob.w),
                                      _p(prob.q), _p(prob.D), prob.kappa, _p(out))
    return out


def K_block(prob, rows, cols):
    """K[rows, cols]: the discretised volume potential V of Eq. 5 that the DAFMM
    compresses (R9): K_ij = G(x_i,x_j) w_j for i != j, K_ii = D_i;  A = I + kappa^2 diag(q) K."""
    rows, cols = _i64(rows), _i64(cols)
    out = np.empty((rows.size, cols.size), dtype=np.complex128)
    if rows.size and cols.size:
        load_library().oracle_K_block(_p(rows), rows.size, _p(cols), cols.size, _p(prob.points), _p(prob.w),
                                      _p(prob.D), prob.kappa, _p(out))
    return out


def dense_matvec_rows(prob, x, rows):
    """(A x)[rows] by direct summation over all N columns."""
    rows, x = _i64(rows), _c128(x)
    out = np.empty(rows.size, dtype=np.complex128)
    load_library().oracle_dense_matvec_rows(_p(rows), rows.size, _p(prob.points), _p(prob.w), _p(prob.q),
                                            _p(prob.D), prob.kappa, prob.n, _p(x), _p(out))
    return out


def dense_matvec(prob, x):
    """A x by direct summation: the plain definition of the product (O(N^2))."""
    return dense_matvec_rows(prob, x, np.arange(prob.n))
