// H0^(1)(z) = J0(z) + i Y0(z) for the product (host setup and device kernels share this code).
//
// The paper only names the kernel G_k(x,y) = (i/4) H0^(1)(k|x-y|).  This is
// the product's own evaluator, independent of the oracle's series / Miller /
// asymptotic bands.  Every entry point takes z2 = (kappa |x - y|)^2: the kernels store
// kappa-scaled coordinates, so no per-entry multiplication by kappa is needed.
//
//   near-type band Zn in {8, 12} (z <= Zn):
//       J0 = pJ(t), Y0 = (1/pi) ln(z2/4) J0 + pR(t),  t = z2 T_SCALE - 1        (code)
//   far-type band [zlo, zhi]:
//       H0 = sqrt(2/(pi z)) (P(x) + i Q(x)) e^{i(z - pi/4)},  x = A/z + B
//       generic band [8, inf) as code; 29 narrower bands as data (FarBand, shared memory)
//   generic (any z > 0): per-lane choice of near band 8 or the generic far band.
//
// Evaluators are lane-blocked: one call evaluates TB independent entries in lockstep, so each
// coefficient (a uniform-register immediate, or one broadcast shared-memory load for data
// bands) is shared by TB FMAs and the TB Horner chains hide each other's latency.  Kernels
// pick one band per CTA-uniform work segment (setup classifies every interaction by the exact
// [z_min, z_max] of its point pairs), so the band never diverges inside a warp.
// ln u uses a 128-entry table of (1/c_i, ln c_i): device callers pass its shared-memory copy
// (load_log_table), host callers kLogTabHost.
#pragma once
#include "common.h"
#include "hankel_coeffs.h"

namespace dafmm {

constexpr double kPi = 3.14159265358979323846;
constexpr double kZ2Safe = 4.0;  // a z^2 inside every band's domain (z = 2), for masked lanes

using dafmm_fit::FarBand;
using dafmm_fit::Pair;

// Band codes of a work segment: 0 generic, 1 near z <= 8, 2 near z <= 12, 3 + b data band b.
constexpr int kBandGeneric = 0;
constexpr int kBandNear8 = 1;
constexpr int kBandNear12 = 2;
constexpr int kBandFarData = 3;
constexpr int kNumBandCodes = kBandFarData + dafmm_fit::NUM_FAR;

// ln(z2 / 4) for TB positive normal z2.
template <int TB>
DAFMM_HD void log_quarter_vec(const double* z2, double* out, const Pair* logtab) {
#ifdef __CUDA_ARCH__
  double r[TB], r2[TB], qe[TB], qo[TB], lc[TB];
  int e[TB];
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    const int hi = __double2hiint(z2[i]);
    e[i] = (hi >> 20) - 1025;  // exponent of z2 / 4
    const int ix = (hi >> (20 - dafmm_fit::LOG_BITS)) & ((1 << dafmm_fit::LOG_BITS) - 1);
    const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, __double2loint(z2[i]));  // [1, 2)
    const Pair tb = logtab[ix];
    r[i] = fma(m, tb.a, -1.0);  // |r| <= 2^-8
    lc[i] = tb.b;
    r2[i] = r[i] * r[i];
  }
  dafmm_fit::log1p_poly<TB>(r2, qe, qo);
#pragma unroll
  for (int i = 0; i < TB; ++i)
    out[i] = fma((double)e[i], dafmm_fit::LN2, lc[i] + fma(r2[i], fma(r[i], qo[i], qe[i]), r[i]));
#else
  (void)logtab;
  for (int i = 0; i < TB; ++i) out[i] = std::log(0.25 * z2[i]);
#endif
}

// Near-type band ZN (z <= ZN): valid for 0 < z2 <= ZN^2.
template <int ZN, int TB>
DAFMM_HD void h0_near_vec(const double* z2, double* re, double* im, const Pair* logtab) {
  using NB = dafmm_fit::NearJR<ZN>;
  double t[TB], j0[TB], rr[TB], lu[TB];
#pragma unroll
  for (int i = 0; i < TB; ++i) t[i] = fma(z2[i], NB::T_SCALE, -1.0);
  NB::template eval<TB>(t, j0, rr);
  log_quarter_vec<TB>(z2, lu, logtab);
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    re[i] = j0[i];
    im[i] = fma(dafmm_fit::INV_PI * lu[i], j0[i], rr[i]);
  }
}

// y = z2^(-1/4) = z^(-1/2): fp32 MUFU seed (z2 must lie in the normal fp32 range), then one
// third-order step y <- y (1 + h/4 + 5h^2/32), h = 1 - z2 y^4 (seed error 2^-22 -> ~1e-19).
DAFMM_HD double rsqrt_sqrt(double z2) {
#ifdef __CUDA_ARCH__
  float f = __double2float_rn(z2), g;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(g) : "f"(f));
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(f) : "f"(g));
  const double y = (double)f;
  const double y2 = y * y;
  const double h = fma(-z2, y2 * y2, 1.0);
  return fma(y, h * fma(h, 0.15625, 0.25), y);
#else
  return 1.0 / std::sqrt(std::sqrt(z2));
#endif
}

// Far-type evaluation with a caller-supplied (P, Q) evaluator: pq(x, P, Q) over TB lanes.
template <int TB, class PQ>
DAFMM_HD void h0_far_vec(const double* z2, double* re, double* im, double A, double B, const PQ& pq) {
  double y[TB], z[TB], x[TB], P[TB], Q[TB], rho[TB], rh2[TB], sp[TB], c[TB];
  int quad[TB];
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    y[i] = rsqrt_sqrt(z2[i]);   // z^(-1/2)
    const double iz = y[i] * y[i];
    z[i] = z2[i] * iz;
    x[i] = fma(iz, A, B);
  }
  pq(x, P, Q);
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    // theta = z - pi/4 = rho + q pi/2, m = q + 1/2, rho = z - m pi/2 (two-part Cody-Waite)
    const double qf = rint(fma(z[i], dafmm_fit::TWO_OVER_PI, -0.5));
    const double m = qf + 0.5;
    rho[i] = fma(-m, dafmm_fit::PIO2_2, fma(-m, dafmm_fit::PIO2_1, z[i]));
    rh2[i] = rho[i] * rho[i];
    quad[i] = ((int)qf) & 3;
  }
  dafmm_fit::sincos_poly<TB>(rh2, sp, c);
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    const double s = rho[i] * sp[i];
    // (cos theta, sin theta) = (c, s) rotated by quadrant * pi/2
    const bool swap = quad[i] & 1;
    double cr = swap ? s : c[i];
    double sr = swap ? c[i] : s;
    if (quad[i] == 1 || quad[i] == 2) cr = -cr;
    if (quad[i] >= 2) sr = -sr;
    const double amp = dafmm_fit::SQRT_2_OVER_PI * y[i];  // sqrt(2/(pi z))
    const double pr = amp * P[i], pi_ = amp * Q[i];
    re[i] = fma(pr, cr, -pi_ * sr);
    im[i] = fma(pr, sr, pi_ * cr);
  }
}

template <int TB>
struct GenericFarPQ {
  DAFMM_HD void operator()(const double* x, double* P, double* Q) const { dafmm_fit::generic_far_pq<TB>(x, P, Q); }
};

// (P, Q) of a data band (coefficients in shared memory on the device; n is CTA-uniform).
template <int TB>
struct DataFarPQ {
  const FarBand* band;
  DAFMM_HD void operator()(const double* x, double* P, double* Q) const {
    const int n = band->n;
    Pair c = band->pq[n - 1];
#pragma unroll
    for (int i = 0; i < TB; ++i) {
      P[i] = c.a;
      Q[i] = c.b;
    }
#pragma unroll 2
    for (int k = n - 2; k >= 0; --k) {
      c = band->pq[k];
#pragma unroll
      for (int i = 0; i < TB; ++i) {
        P[i] = fma(P[i], x[i], c.a);
        Q[i] = fma(Q[i], x[i], c.b);
      }
    }
  }
};

// Generic: any z > 0 (per-lane band choice; used where a segment straddles the bands).
template <int TB>
DAFMM_HD void h0_generic_vec(const double* z2, double* re, double* im, const Pair* logtab) {
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    if (z2[i] <= dafmm_fit::NearJR<8>::Z2_MAX)
      h0_near_vec<8, 1>(z2 + i, re + i, im + i, logtab);
    else
      h0_far_vec<1>(z2 + i, re + i, im + i, dafmm_fit::GENERIC_FAR_A, dafmm_fit::GENERIC_FAR_B, GenericFarPQ<1>());
  }
}

// Scalar host evaluation (setup: ACA entries and operators); z2 = (kappa r)^2.
inline cplx h0(double z2) {
  double re, im;
  h0_generic_vec<1>(&z2, &re, &im, dafmm_fit::kLogTabHost);
  return {re, im};
}

// Setup-side band choice for a segment whose point pairs have z in [zmin, zmax]: the
// cheapest band (estimated fp64 operations per entry) that covers the whole range.
inline int choose_band(double zmin, double zmax) {
  int best = kBandGeneric;
  double cost = 1e30;
  if (zmax <= 8.0) {
    best = kBandNear8;
    cost = 51.0;
  } else if (zmax <= 12.0) {
    best = kBandNear12;
    cost = 59.0;
  }
  for (int b = 0; b < dafmm_fit::NUM_FAR; ++b) {
    const FarBand& F = dafmm_fit::kFarBandsHost[b];
    if (zmin >= F.zlo && zmax <= F.zhi) {
      double c = 40.0 + 2.0 * F.n;
      if (c < cost) {
        cost = c;
        best = kBandFarData + b;
      }
    }
  }
  return best;
}

#ifdef __CUDACC__
// Copy the log table into shared memory (all threads; followed by a barrier).
__device__ __forceinline__ void load_log_table(Pair* dst) {
  for (int i = threadIdx.x; i < (1 << dafmm_fit::LOG_BITS); i += blockDim.x) dst[i] = dafmm_fit::kLogTabDev[i];
  __syncthreads();
}
// Copy data band b into shared memory (all threads; the caller's next barrier publishes it).
__device__ __forceinline__ void load_far_band(FarBand* dst, int b) {
  static_assert(sizeof(FarBand) % sizeof(Pair) == 0, "FarBand is copied as pairs");
  const Pair* src = reinterpret_cast<const Pair*>(&dafmm_fit::kFarBandsDev[b]);
  Pair* d = reinterpret_cast<Pair*>(dst);
  for (int i = threadIdx.x; i < (int)(sizeof(FarBand) / sizeof(Pair)); i += blockDim.x) d[i] = src[i];
}
#endif

}  // namespace dafmm
