"""GPU parity of the product's H0^(1) evaluator, band by band (dafmm_h0_eval, the lane-blocked
code the P2P and M2L kernels run), against the oracle's H0 (oracle/oracle_core.c, itself pinned
to mpmath values, the Wronskian and series/asymptotic overlap in tests/test_oracle_*.py).

Every band is swept over its whole valid interval (dafmm_h0_bands), endpoints included, with a
log-spaced grid plus seeded random points, so every coefficient of every band is exercised,
including bands the C1-C5 workloads touch only rarely.  Tolerance: |h_gpu - h_oracle| <=
2.5e-13 * max(1, z/100) * |H0(z)|.  That is the oracle's own pinned bound (2e-13 relative,
reading A2 of SURVEY 8(c), tests/test_oracle_special.py; its ascending series loses digits
towards z = 8) plus 5e-14 for the product (its fits are within 3e-15 of mpmath,
tools/fit_hankel.py); the z/100 growth is the phase's input-rounding floor z * eps."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle.core import h0 as oracle_h0

pytestmark = pytest.mark.gpu

Z_MIN = 1e-3   # below every kappa r the workloads produce (C5's smallest is kappa h / 8 ~ 0.05)
Z_MAX = 1e3    # above every kappa r the workloads produce (C5: 200 * 2 sqrt(2) = 566)


def _prod():
    import paper_2204_00326_b200 as prod
    return prod


def _sample(lo, hi, n, rng):
    lo = max(lo, Z_MIN)
    hi = min(hi, Z_MAX)
    z = np.concatenate([np.geomspace(lo, hi, n), rng.uniform(lo, hi, n), [lo, hi, np.nextafter(hi, 0.0)]])
    return np.unique(z)


def _gpu_h0(z2, band):
    prod = _prod()
    zd = torch.from_numpy(z2).cuda()
    out = torch.empty(z2.size, dtype=torch.complex128, device="cuda")
    prod.binding.dafmm_h0_eval(zd, out, band, torch.cuda.current_stream())
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _check(z, band):
    z2 = z * z
    got = _gpu_h0(z2, band)
    ref = oracle_h0(np.sqrt(z2))
    err = np.abs(got - ref) / np.abs(ref)
    tol = 2.5e-13 * np.maximum(1.0, z / 100.0)
    worst = int(np.argmax(err / tol))
    assert np.all(err <= tol), "band %d: z = %.17g rel err %.3e (tol %.1e)" % (band, z[worst], err[worst], tol[worst])
    return float(err.max())


def test_every_band_over_its_interval():
    prod = _prod()
    bands = prod.binding.dafmm_h0_bands()
    assert len(bands) >= 5
    rng = np.random.default_rng(2204)
    for code, (lo, hi) in enumerate(bands):
        _check(_sample(lo, hi, 400, rng), code)


def test_generic_band_covers_everything_and_ragged_lengths():
    # code 0 picks near-8 or the asymptotic form per element; lengths that are not a multiple of
    # the lane block (4) and n = 0 take the tail path
    rng = np.random.default_rng(7)
    for n in (1, 3, 5, 4099):
        z = np.exp(rng.uniform(np.log(Z_MIN), np.log(Z_MAX), n))
        _check(z, 0)
    _gpu_h0(np.empty(0), 0)


def test_band_choice_boundaries_agree():
    # at every band's upper end the band and the next wider evaluator agree (no seam in the
    # M2L / P2P sums where setup switches bands)
    prod = _prod()
    bands = prod.binding.dafmm_h0_bands()
    for code, (lo, hi) in enumerate(bands[1:], start=1):
        if not np.isfinite(hi) or hi > Z_MAX:
            continue
        z = np.array([hi, np.nextafter(hi, 0.0)])
        a, g = _gpu_h0(z * z, code), _gpu_h0(z * z, 0)
        assert np.all(np.abs(a - g) <= 2e-13 * np.abs(g)), code


def test_invalid_band_code_rejected():
    prod = _prod()
    nb = len(prod.binding.dafmm_h0_bands())
    z = torch.ones(4, dtype=torch.float64, device="cuda")
    out = torch.empty(4, dtype=torch.complex128, device="cuda")
    with pytest.raises(prod.binding.DAFMMError):
        prod.binding.dafmm_h0_eval(z, out, nb)
    with pytest.raises(prod.binding.DAFMMError):
        prod.binding.dafmm_h0_eval(z, out, -1)
