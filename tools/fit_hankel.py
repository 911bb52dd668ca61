#!/usr/bin/env python3
"""Generate paper_2204_00326_b200/csrc/hankel_coeffs.h — the product's H0^(1) approximations.

PRODUCT TOOLING (not the oracle; the oracle evaluates H0 by its own series / Miller /
asymptotic bands and never reads this header).  Fits are Chebyshev interpolants computed in
40-digit arithmetic with mpmath, converted to monomial form in a scaled variable and checked
in fp64 Horner arithmetic against mpmath before being written.

Bands:
  near  z <  Z_NEAR:  H0 = J0(u) + i [ (1/pi) ln(u) J0(u) + R(u) ],  u = z^2/4,
        J0 and R (the regular part of Y0) as polynomials in t = u / U_MAX * 2 - 1.
  far   z >= Z_FAR:   H0 = sqrt(2/(pi z)) (P + i Q) e^{i (z - pi/4)},
        P(s), Qt(s) polynomials in v = 2 s - 1, s = (Z_FAR / z)^2, Q = Qt * Z_FAR / z.
  sincos on |rho| <= pi/4: sin(rho)/rho and cos(rho) as polynomials in rho^2.
"""
import os
import sys

import mpmath as mp
import numpy as np

mp.mp.dps = 45
Z_NEAR = 8.0
U_MAX = Z_NEAR * Z_NEAR / 4.0
Z_FAR = 8.0


def cheb_coeffs(f, deg, a, b):
    n = deg + 1
    nodes = [mp.cos(mp.pi * (k + mp.mpf(1) / 2) / n) for k in range(n)]
    vals = [f(mp.mpf(a) + (mp.mpf(b) - a) * (x + 1) / 2) for x in nodes]
    c = []
    for j in range(n):
        s = mp.fsum(vals[k] * mp.cos(mp.pi * j * (k + mp.mpf(1) / 2) / n) for k in range(n))
        c.append(2 * s / n)
    c[0] /= 2
    return c


def cheb_to_monomial(c):
    """Chebyshev series on [-1,1] -> monomial coefficients (ascending)."""
    n = len(c)
    T = [[mp.mpf(0)] * n for _ in range(n)]
    T[0][0] = mp.mpf(1)
    if n > 1:
        T[1][1] = mp.mpf(1)
    for k in range(2, n):
        for j in range(n):
            T[k][j] = (2 * T[k - 1][j - 1] if j > 0 else 0) - T[k - 2][j]
    return [mp.fsum(c[k] * T[k][j] for k in range(n)) for j in range(n)]


def horner(coef, x):
    acc = np.float64(coef[-1])
    for a in reversed(coef[:-1]):
        acc = acc * x + np.float64(a)
    return acc


def j0_of_u(u):
    return mp.besselj(0, 2 * mp.sqrt(u)) if u > 0 else mp.mpf(1)


def r_of_u(u):
    if u == 0:
        return 2 / mp.pi * mp.euler
    z = 2 * mp.sqrt(u)
    return mp.bessely(0, z) - (1 / mp.pi) * mp.log(u) * mp.besselj(0, z)


def pq(z):
    h = mp.hankel1(0, z) * mp.exp(-1j * (z - mp.pi / 4)) * mp.sqrt(mp.pi * z / 2)
    return h.real, h.imag


def fit_near(deg):
    cj = cheb_to_monomial(cheb_coeffs(lambda t: j0_of_u((t + 1) / 2 * U_MAX), deg, -1, 1))
    cr = cheb_to_monomial(cheb_coeffs(lambda t: r_of_u((t + 1) / 2 * U_MAX), deg, -1, 1))
    return cj, cr


def fit_far(deg):
    def fp(v):
        s = (v + 1) / 2
        return pq(Z_FAR / mp.sqrt(s))[0] if s > 0 else mp.mpf(1)

    def fq(v):
        s = (v + 1) / 2
        if s == 0:
            return mp.mpf(-1) / (8 * Z_FAR)
        z = Z_FAR / mp.sqrt(s)
        return pq(z)[1] * z / Z_FAR

    return (cheb_to_monomial(cheb_coeffs(fp, deg, -1, 1)), cheb_to_monomial(cheb_coeffs(fq, deg, -1, 1)))


def fit_sincos(deg):
    r2max = (mp.pi / 4) ** 2
    fs = lambda v: (mp.sin(mp.sqrt((v + 1) / 2 * r2max)) / mp.sqrt((v + 1) / 2 * r2max)) if v > -1 else mp.mpf(1)
    fc = lambda v: mp.cos(mp.sqrt((v + 1) / 2 * r2max))
    return cheb_to_monomial(cheb_coeffs(fs, deg, -1, 1)), cheb_to_monomial(cheb_coeffs(fc, deg, -1, 1)), r2max


def emit(name, coef):
    """An inline Horner evaluator with the coefficients as literals (folded into DFMA operands)."""
    expr = "%.17e" % float(coef[-1])
    for a in reversed(coef[:-1]):
        expr = "fma(%s, x, %.17e)" % (expr, float(a))
    return "DAFMM_HD double %s(double x) {\n  return %s;\n}\n" % (name, expr)


def cody_waite():
    """pi/2 split into C1 (33 significant bits), C2 (33 bits), C3 (53 bits)."""
    half_pi = mp.pi / 2
    def trunc(x, bits):
        e = int(mp.floor(mp.log(abs(x), 2)))
        scale = mp.mpf(2) ** (bits - 1 - e)
        return mp.floor(x * scale) / scale
    c1 = trunc(half_pi, 33)
    c2 = trunc(half_pi - c1, 33)
    c3 = half_pi - c1 - c2
    return float(c1), float(c2), float(c3)


def main(out_path):
    # --- near band ---
    for deg in range(12, 26):
        cj, cr = fit_near(deg)
        err = 0.0
        for u in np.linspace(0, U_MAX, 257):
            t = np.float64(u / U_MAX * 2 - 1)
            ej = abs(horner(cj, t) - float(j0_of_u(mp.mpf(u))))
            er = abs(horner(cr, t) - float(r_of_u(mp.mpf(u))))
            err = max(err, ej, er)
        print("near deg", deg, "max abs err", err, file=sys.stderr)
        if err < 4e-16 * 8:
            break
    near_deg, near_err = deg, err
    # --- far band ---
    for deg in range(8, 30):
        cp, cq = fit_far(deg)
        err = 0.0
        for s in np.linspace(0, 1, 257):
            v = np.float64(2 * s - 1)
            if s == 0:
                continue
            z = Z_FAR / mp.sqrt(mp.mpf(s))
            P, Q = pq(z)
            err = max(err, abs(horner(cp, v) - float(P)), abs(horner(cq, v) - float(Q * z / Z_FAR)))
        print("far deg", deg, "max abs err", err, file=sys.stderr)
        if err < 3e-16:
            break
    far_deg, far_err = deg, err
    for deg in range(5, 14):
        cs, cc, r2max = fit_sincos(deg)
        err = 0.0
        for rho in np.linspace(-float(mp.pi / 4), float(mp.pi / 4), 513):
            v = np.float64(rho * rho / float(r2max) * 2 - 1)
            err = max(err, abs(rho * horner(cs, v) - np.sin(rho)), abs(horner(cc, v) - np.cos(rho)))
        print("sincos deg", deg, "max abs err", err, file=sys.stderr)
        if err < 2.3e-16:
            break
    with open(out_path, "w") as f:
        f.write("// GENERATED by tools/fit_hankel.py — do not edit.  Product-side H0^(1) fits\n")
        f.write("// (near band: fp64 Horner max abs err %.2e at degree %d; far band %.2e at degree %d).\n"
                % (near_err, near_deg, far_err, far_deg))
        f.write("#pragma once\n#include \"common.h\"\nnamespace dafmm_fit {\n")
        f.write("static constexpr double Z_NEAR = %.17g;\nstatic constexpr double U_MAX = %.17g;\n" % (Z_NEAR, U_MAX))
        f.write("static constexpr double Z_FAR = %.17g;\nstatic constexpr double SC_R2MAX = %.17e;\n"
                % (Z_FAR, float(r2max)))
        c1, c2, c3 = cody_waite()
        f.write("static constexpr double PIO2_1 = %.17e;\nstatic constexpr double PIO2_2 = %.17e;\n"
                "static constexpr double PIO2_3 = %.17e;\n" % (c1, c2, c3))
        f.write(emit("near_j0", cj) + emit("near_r", cr) + emit("far_p", cp) + emit("far_q", cq))
        f.write(emit("sin_over_x", cs) + emit("cos_poly", cc))
        f.write("}  // namespace dafmm_fit\n")


if __name__ == "__main__":
    here = os.path.dirname(os.path.abspath(__file__))
    main(os.path.join(here, "..", "paper_2204_00326_b200", "csrc", "hankel_coeffs.h"))
