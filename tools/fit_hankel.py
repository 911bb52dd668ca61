#!/usr/bin/env python3
"""Generate paper_2204_00326_b200/csrc/hankel_coeffs.h — the product's H0^(1) approximations.

PRODUCT TOOLING (not the oracle; the oracle evaluates H0 by its own series / Miller /
asymptotic bands and never reads this header).  Fits are Chebyshev interpolants computed in
multi-digit arithmetic with mpmath, converted to monomial form and checked in fp64 Horner
arithmetic against mpmath before being written.

All evaluators take z2 = (kappa r)^2 (the kernels store kappa-scaled coordinates).

  near-type band Zn (z <= Zn):   H0 = J0 + i [ (1/pi) ln(u) J0 + R ],  u = z2/4,
        J0 and R (the regular part of Y0) polynomials in t = 2u/U - 1, U = Zn^2/4.
  far-type band, z in [zlo, zhi]:   H0 = sqrt(2/(pi z)) (P + i Q) e^{i (z - pi/4)},
        P, Q polynomials in x = A s + B, s = 1/z mapped from [1/zhi, 1/zlo] onto [-1, 1].
        The generic band [8, inf) sits in PolyTable; 29 narrower bands form the FarBand table.
  sincos on |rho| <= pi/4: sin(rho)/rho and cos(rho) polynomials in rho^2.
  ln u = e ln2 + ln c_i + log1p(m/c_i - 1), u = 2^e m, with a 2^8-entry table (rcp_i, ln c_i)
        indexed by the top mantissa bits and a degree-6 log1p.

Fixed-degree polynomials (near bands, generic far band, sincos, log1p) are emitted as lane-
blocked Horner evaluators with literal coefficients: each literal becomes a uniform-register
immediate shared by the TB lanes of a block (on sm_100a DFMA takes no constant-bank operand).
Data that is selected at run time is emitted as tables the kernels copy to shared memory: the
log table (PolyTable) and the FarBand table of data bands (coefficient pairs, padded to an odd
count so the Horner loop runs in pairs).
"""
import math
import os
import sys

import mpmath as mp
import numpy as np

mp.mp.dps = 32
NEAR_BANDS = [7.0, 8.0, 12.0]       # near-type bands z <= Zn
GENERIC_FAR = (8.0, float("inf"))   # far-type band emitted as code (generic per-lane path)
TOL_FAR = 3.0e-16                   # max abs error of P, Q (|P| ~ 1)
TOL_NEAR = 3.2e-15                  # max abs error of J0, R


def far_menu():
    """Far-type data bands: ratio-2 and ratio-4 bands on a sqrt(2) grid from 2.5, and tails."""
    g = [2.5 * math.sqrt(2.0) ** k for k in range(13)]
    bands = [(a, 2 * a) for a in g] + [(a, 4 * a) for a in g[:11]]
    bands += [(a, float("inf")) for a in (16.0, 32.0, 64.0, 128.0, 256.0)]
    return bands


def cheb_coeffs(f, deg):
    n = deg + 1
    nodes = [mp.cos(mp.pi * (k + mp.mpf(1) / 2) / n) for k in range(n)]
    vals = [f(x) for x in nodes]
    c = []
    for j in range(n):
        s = mp.fsum(vals[k] * mp.cos(mp.pi * j * (k + mp.mpf(1) / 2) / n) for k in range(n))
        c.append(2 * s / n)
    c[0] /= 2
    return c


def cheb_to_monomial(c, a=1, b=0):
    """Chebyshev series in w on [-1,1] -> monomial coefficients (ascending) in y, w = a y + b."""
    n = len(c)
    T = [[mp.mpf(0)] * n for _ in range(n)]
    T[0][0] = mp.mpf(1)
    if n > 1:
        T[1][1] = mp.mpf(1)
    for k in range(2, n):
        for j in range(n):
            T[k][j] = (2 * T[k - 1][j - 1] if j > 0 else 0) - T[k - 2][j]
    mono_w = [mp.fsum(c[k] * T[k][j] for k in range(n)) for j in range(n)]
    out = [mp.mpf(0)] * n
    for j, cw in enumerate(mono_w):
        for i in range(j + 1):
            out[i] += cw * mp.binomial(j, i) * mp.mpf(a) ** i * mp.mpf(b) ** (j - i)
    return out


def horner(coef, x):
    acc = np.float64(coef[-1])
    for a in reversed(coef[:-1]):
        acc = np.float64(acc * np.float64(x) + np.float64(a))
    return acc


def j0_of_u(u):
    return mp.besselj(0, 2 * mp.sqrt(u)) if u > 0 else mp.mpf(1)


def r_of_u(u):
    """Regular part of Y0: Y0 - (1/pi) ln(u) J0 with u = z^2/4 (limit 2 gamma / pi at 0)."""
    if u == 0:
        return 2 * mp.euler / mp.pi
    z = 2 * mp.sqrt(u)
    return mp.bessely(0, z) - (1 / mp.pi) * mp.log(u) * mp.besselj(0, z)


def pq(z):
    h = mp.hankel1(0, z) * mp.exp(-1j * (z - mp.pi / 4)) * mp.sqrt(mp.pi * z / 2)
    return h.real, h.imag


def fit_near(zn):
    U = zn * zn / 4
    for deg in range(12, 30):
        cj = cheb_to_monomial(cheb_coeffs(lambda t: j0_of_u((t + 1) / 2 * U), deg))
        cr = cheb_to_monomial(cheb_coeffs(lambda t: r_of_u((t + 1) / 2 * U), deg))
        err = 0.0
        for u in np.linspace(0, U, 241):
            t = np.float64(u / U * 2 - 1)
            err = max(err, abs(horner(cj, t) - float(j0_of_u(mp.mpf(u)))),
                      abs(horner(cr, t) - float(r_of_u(mp.mpf(u)))))
        if err < TOL_NEAR:
            print("near z <= %g: degree %d, max abs err %.2e" % (zn, deg, err), file=sys.stderr)
            return cj, cr, deg, err
    raise RuntimeError("near fit failed")


def band_map(zlo, zhi):
    slo = mp.mpf(0) if zhi == float("inf") else mp.mpf(1) / zhi
    shi = mp.mpf(1) / zlo
    return slo, shi, 2 / (shi - slo), -(shi + slo) / (shi - slo)


def fit_far(zlo, zhi, start=4):
    slo, shi, A, B = band_map(zlo, zhi)

    def s_of(x):
        return slo + (shi - slo) * (x + 1) / 2

    def fp(x):
        return pq(1 / s_of(x))[0] if s_of(x) > 0 else mp.mpf(1)

    def fq(x):
        return pq(1 / s_of(x))[1] if s_of(x) > 0 else mp.mpf(0)

    checks = [mp.mpf(x) for x in np.linspace(-1, 1, 121)]
    ref = [pq(1 / s_of(x)) if s_of(x) > 0 else (mp.mpf(1), mp.mpf(0)) for x in checks]
    for deg in range(start, 34):
        cp = cheb_to_monomial(cheb_coeffs(fp, deg))
        cq = cheb_to_monomial(cheb_coeffs(fq, deg))
        err = 0.0
        for x, (P, Q) in zip(checks, ref):
            err = max(err, abs(horner(cp, float(x)) - float(P)), abs(horner(cq, float(x)) - float(Q)))
        if err < TOL_FAR:
            print("far band [%g, %g]: degree %d, max abs err %.2e" % (zlo, zhi, deg, err), file=sys.stderr)
            return cp, cq, deg, err, float(A), float(B)
    raise RuntimeError("far fit failed for [%g, %g]" % (zlo, zhi))


def fit_sincos():
    r2max = (mp.pi / 4) ** 2
    for deg in range(5, 14):
        fs = lambda w: (mp.sin(mp.sqrt((w + 1) / 2 * r2max)) / mp.sqrt((w + 1) / 2 * r2max)) if w > -1 else mp.mpf(1)
        fc = lambda w: mp.cos(mp.sqrt((w + 1) / 2 * r2max))
        a, b = 2 / r2max, -1  # w = 2 rho^2 / r2max - 1  ->  monomials in rho^2
        cs = cheb_to_monomial(cheb_coeffs(fs, deg), a, b)
        cc = cheb_to_monomial(cheb_coeffs(fc, deg), a, b)
        err = 0.0
        for rho in np.linspace(-float(mp.pi / 4), float(mp.pi / 4), 513):
            r2 = np.float64(rho * rho)
            err = max(err, abs(rho * horner(cs, r2) - np.sin(rho)), abs(horner(cc, r2) - np.cos(rho)))
        if err < 2.3e-16:
            print("sincos: degree %d, max abs err %.2e" % (deg, err), file=sys.stderr)
            return cs, cc, deg, err
    raise RuntimeError("sincos fit failed")


def cody_waite():
    """pi/2 = C1 + C2 (+ C3): C1 with 33 significant bits (m C1 exact for m < 2^20), C2 the
    rounded remainder; C3 (< 1e-20) is below the fp64 resolution of rho for z < 1e4."""
    half_pi = mp.pi / 2

    def trunc(x, bits):
        e = int(mp.floor(mp.log(abs(x), 2)))
        scale = mp.mpf(2) ** (bits - 1 - e)
        return mp.floor(x * scale) / scale
    c1 = trunc(half_pi, 33)
    return float(c1), float(half_pi - c1)


def log_table(bits=8):
    """(rcp_i, ln c_i) with rcp_i = fp64(1 / (1 + (i + 1/2) / 2^bits)) and ln c_i = -ln(rcp_i)
    exactly for the stored rcp_i, so ln(m) = log1p(m rcp_i - 1) + ln c_i is an identity."""
    out = []
    for i in range(1 << bits):
        rcp = float(1 / (1 + (mp.mpf(i) + mp.mpf(1) / 2) / (1 << bits)))
        out.append((rcp, float(-mp.log(mp.mpf(rcp)))))
    return out


def log1p_coeffs():
    """log1p(r) = r + r^2 q(r), q(r) = sum_{k>=0} (-1)^(k+1) r^k / (k+2), split into even and odd
    parts q = qe(r^2) + r qo(r^2) (degree 6 overall: |r| <= 2^-9 leaves a tail < 2e-19)."""
    q = [mp.mpf((-1) ** (k + 1)) / (k + 2) for k in range(5)]
    return q[0::2], q[1::2]


def h2_function(name, ca, cb, doc, template="template <int TB>", prefix="DAFMM_HD void"):
    """A lane-blocked pair-Horner evaluator with literal coefficients:
    a[i] = sum_k ca[k] x[i]^k, b[i] = sum_k cb[k] x[i]^k for i < TB."""
    n = max(len(ca), len(cb))
    ca = [float(v) for v in ca] + [0.0] * (n - len(ca))
    cb = [float(v) for v in cb] + [0.0] * (n - len(cb))
    out = ["// %s" % doc, template, "%s %s(const double* x, double* a, double* b) {" % (prefix, name),
           "  DAFMM_H2_INIT(%.17e, %.17e)" % (ca[-1], cb[-1])]
    for k in range(n - 2, -1, -1):
        out.append("  DAFMM_H2_STEP(%.17e, %.17e)" % (ca[k], cb[k]))
    out.append("}")
    return "\n".join(out)


def main(out_path):
    nears = [fit_near(zn) for zn in NEAR_BANDS]
    gfar = fit_far(*GENERIC_FAR)
    menu = far_menu()
    fars = [fit_far(zlo, zhi) for zlo, zhi in menu]
    cs, cc, sc_deg, sc_err = fit_sincos()
    c1, c2 = cody_waite()
    qe, qo = log1p_coeffs()
    lt = log_table()
    maxn = max(f[2] for f in fars) + 2
    L = []
    w = L.append
    w("// GENERATED by tools/fit_hankel.py — do not edit.  Product-side H0^(1) fits (DESIGN.md §6).")
    for zn, f in zip(NEAR_BANDS, nears):
        w("// near band z <= %g: degree %d, fp64 Horner max abs err %.2e" % (zn, f[2], f[3]))
    w("// generic far band [%g, inf): degree %d, %.2e;  sincos degree %d, %.2e" % (GENERIC_FAR[0], gfar[2], gfar[3],
                                                                                  sc_deg, sc_err))
    w("// %d far-type data bands, degrees %d..%d, max abs err <= %.1e" % (len(fars), min(f[2] for f in fars),
                                                                         max(f[2] for f in fars), TOL_FAR))
    w("#pragma once")
    w('#include "common.h"')
    w("namespace dafmm_fit {")
    w("constexpr double INV_PI = %.17e;" % float(1 / mp.pi))
    w("constexpr double TWO_OVER_PI = %.17e;" % float(2 / mp.pi))
    w("constexpr double SQRT_2_OVER_PI = %.17e;" % float(mp.sqrt(2 / mp.pi)))
    w("constexpr double LN2 = %.17e;" % float(mp.log(2)))
    w("constexpr double PIO2_1 = %.17e;\nconstexpr double PIO2_2 = %.17e;" % (c1, c2))
    w("constexpr int LOG_BITS = 8;")
    w("struct alignas(16) Pair {\n  double a, b;\n};")
    # fixed-degree polynomials: pairs in one table (copied to shared memory by the kernels)
    def pairlist(ca, cb):
        n = max(len(ca), len(cb))
        ca = [float(v) for v in ca] + [0.0] * (n - len(ca))
        cb = [float(v) for v in cb] + [0.0] * (n - len(cb))
        return n, "{" + ", ".join("{%.17e, %.17e}" % (x, y) for x, y in zip(ca, cb)) + "}"
    n7, near7 = pairlist(nears[0][0], nears[0][1])
    n8, near8 = pairlist(nears[1][0], nears[1][1])
    n12, near12 = pairlist(nears[2][0], nears[2][1])
    ngf, gf = pairlist(gfar[0], gfar[1])
    nsc, sc = pairlist(cs, cc)
    nlp, lp = pairlist(qe, qo)
    w("// near-type bands: (J0, R) polynomials in t = z2 * T_SCALE - 1")
    for zn, n in zip(NEAR_BANDS, (n7, n8, n12)):
        U = zn * zn / 4
        w("constexpr double NEAR%d_Z2_MAX = %.17g;  // z^2 <= Z2_MAX" % (int(zn), zn * zn))
        w("constexpr double NEAR%d_T_SCALE = %.17g;  // t = z2 * T_SCALE - 1 = 2 (z2/4) / U - 1" % (int(zn), 0.5 / U))
        w("constexpr int NEAR%d_N = %d;" % (int(zn), n))
    w("constexpr double GENERIC_FAR_ZLO = %.17g;" % GENERIC_FAR[0])
    w("constexpr double GENERIC_FAR_A = %.17e, GENERIC_FAR_B = %.17e;" % (gfar[4], gfar[5]))
    w("constexpr int GENERIC_FAR_N = %d, SC_N = %d, LOG1P_N = %d;" % (ngf, nsc, nlp))
    w("#define DAFMM_H2_INIT(ca, cb)                 \\")
    w("  _Pragma(\"unroll\") for (int i = 0; i < TB; ++i) { \\")
    w("    a[i] = ca;                                \\")
    w("    b[i] = cb;                                \\")
    w("  }")
    w("#define DAFMM_H2_STEP(ca, cb)                 \\")
    w("  _Pragma(\"unroll\") for (int i = 0; i < TB; ++i) { \\")
    w("    a[i] = fma(a[i], x[i], ca);               \\")
    w("    b[i] = fma(b[i], x[i], cb);               \\")
    w("  }")
    w("// Fixed-degree polynomials with their coefficients as immediates (uniform-register operands")
    w("// of DFMA, shared by the TB lanes of a block); measured faster than shared-memory coefficient")
    w("// tables for both the P2P and the M2L kernel (DESIGN.md §6, profiles/ab_r20_*).")
    w(h2_function("near7_imm", nears[0][0], nears[0][1], "(J0, R), z <= 7"))
    w(h2_function("near8_imm", nears[1][0], nears[1][1], "(J0, R), z <= 8"))
    w(h2_function("near12_imm", nears[2][0], nears[2][1], "(J0, R), z <= 12"))
    w(h2_function("generic_far_imm", gfar[0], gfar[1], "(P, Q) of the generic far band [8, inf)"))
    w(h2_function("sincos_imm", cs, cc, "(sin(rho)/rho, cos(rho)) in rho^2"))
    w(h2_function("log1p_imm", qe, qo, "(qe, qo) in r^2"))
    w("// The log table (per-lane indexed: data, copied to shared memory by the kernels).")
    w("struct PolyTable {")
    w("  Pair log_tab[1 << LOG_BITS];    // (rcp_i, ln c_i), i = top LOG_BITS mantissa bits")
    w("};")
    lt_init = "{" + ", ".join("{%.17e, %.17e}" % t for t in lt) + "}"
    init = "{\n%s}" % lt_init
    w("#if defined(__CUDACC__)")
    w("static __constant__ PolyTable kPolyDev = %s;" % init)
    w("#endif")
    w("static const PolyTable kPolyHost = %s;" % init)
    w("// far-type data bands: x = A / z + B; pq[k] = (P_k, Q_k), k < n")
    w("constexpr int NUM_FAR = %d;" % len(fars))
    w("constexpr int FAR_MAXN = %d;" % maxn)
    w("struct FarBand {\n  double zlo, zhi, A, B;\n  int n, pad;\n  Pair pq[FAR_MAXN];\n};")
    rows = []
    for (zlo, zhi), f in zip(menu, fars):
        n = f[2] + 1
        if n % 2 == 0:  # pad to an odd coefficient count with a zero leading (highest) coefficient:
            # the kernels' Horner loop then runs in coefficient pairs without a remainder
            f = (list(f[0]) + [mp.mpf(0)], list(f[1]) + [mp.mpf(0)]) + tuple(f[2:])
            n += 1
        pqs = ", ".join("{%.17e, %.17e}" % (float(a), float(b)) for a, b in zip(f[0], f[1]))
        pqs += "".join(", {0.0, 0.0}" for _ in range(maxn - n))
        rows.append("{%.17g, %s, %.17e, %.17e, %d, 0, {%s}}" % (zlo, "1e308" if zhi == float("inf") else
                                                                "%.17g" % zhi, f[4], f[5], n, pqs))
    init = "{\n" + ",\n".join(rows) + "}"
    w("#if defined(__CUDACC__)")
    w("static __constant__ FarBand kFarBandsDev[NUM_FAR] = %s;" % init)
    w("#endif")
    w("static const FarBand kFarBandsHost[NUM_FAR] = %s;" % init)
    w("}  // namespace dafmm_fit")
    with open(out_path, "w") as f:
        f.write("\n".join(L) + "\n")


if __name__ == "__main__":
    here = os.path.dirname(os.path.abspath(__file__))
    main(os.path.join(here, "..", "paper_2204_00326_b200", "csrc", "hankel_coeffs.h"))
