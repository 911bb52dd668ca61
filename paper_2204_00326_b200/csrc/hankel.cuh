// H0^(1)(z) = J0(z) + i Y0(z) for the product (host setup and device kernels share this code).
//
// The paper only names the kernel G_k(x,y) = (i/4) H0^(1)(k|x-y|).  This is
// the product's own evaluator, independent of the oracle's series / Miller /
// asymptotic bands.  Every entry point takes z2 = (kappa |x - y|)^2: the kernels store
// kappa-scaled coordinates, so no per-entry multiplication by kappa is needed.
//
//   near-type band Zn in {8, 12} (z <= Zn):
//       J0 = pJ(t), Y0 = (1/pi) ln(z2/4) J0 + pR(t),  t = z2 T_SCALE - 1
//   far-type band [zlo, zhi]:
//       H0 = sqrt(2/(pi z)) (P(x) + i Q(x)) e^{i(z - pi/4)},  x = A/z + B
//       generic band [8, inf) in PolyTable; 29 narrower bands in the FarBand table
//   generic (any z > 0): per-lane choice of near band 8 or the generic far band.
//
// Evaluators are lane-blocked: one call evaluates TB independent entries in lockstep, so each
// coefficient of a fixed-degree polynomial (an immediate: a uniform-register DFMA operand) is
// shared by TB FMAs.  Data chosen at run time lives in tables that device callers pass as their
// shared-memory copies (load_poly_table: the log table; load_far_bands: the data bands) and host
// callers as kPolyHost / kFarBandsHost.  Kernels pick one band per CTA-uniform work segment (setup classifies every
// interaction by the exact [z_min, z_max] of its point pairs), so the band never diverges
// inside a warp.
#pragma once
#include "common.h"
#include "hankel_coeffs.h"

namespace dafmm {

constexpr double kPi = 3.14159265358979323846;
constexpr double kZ2Safe = 4.0;  // a z^2 inside every band's domain (z = 2), for masked lanes

using dafmm_fit::FarBand;
using dafmm_fit::Pair;
using dafmm_fit::PolyTable;

// Band codes of a work segment: 0 generic, 1 near z <= 8, 2 near z <= 12, 3 near z <= 7,
// 4 + b data band b.
constexpr int kBandGeneric = 0;
constexpr int kBandNear8 = 1;
constexpr int kBandNear12 = 2;
constexpr int kBandNear7 = 3;
constexpr int kBandFarData = 4;
constexpr int kNumBandCodes = kBandFarData + dafmm_fit::NUM_FAR;

// Fixed-degree polynomials: lane-blocked Horner with immediate coefficients (hankel_coeffs.h).
template <int ZN, int TB>
DAFMM_HD void poly_near(const double* x, double* a, double* b) {
  if constexpr (ZN == 7) dafmm_fit::near7_imm<TB>(x, a, b);
  else if constexpr (ZN == 8) dafmm_fit::near8_imm<TB>(x, a, b);
  else dafmm_fit::near12_imm<TB>(x, a, b);
}

// ln(z2 / 4) for TB positive normal z2.
template <int TB>
DAFMM_HD void log_quarter_vec(const double* z2, double* out, const PolyTable& T) {
#ifdef __CUDA_ARCH__
  double r[TB], r2[TB], qe[TB], qo[TB], lc[TB];
  int e[TB];
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    const int hi = __double2hiint(z2[i]);
    e[i] = (hi >> 20) - 1025;  // exponent of z2 / 4
    const int ix = (hi >> (20 - dafmm_fit::LOG_BITS)) & ((1 << dafmm_fit::LOG_BITS) - 1);
    const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, __double2loint(z2[i]));  // [1, 2)
    const Pair tb = T.log_tab[ix];  // per-lane index: an ordinary (gather) shared load
    r[i] = fma(m, tb.a, -1.0);      // |r| <= 2^-8
    lc[i] = tb.b;
    r2[i] = r[i] * r[i];
  }
  dafmm_fit::log1p_imm<TB>(r2, qe, qo);
#pragma unroll
  for (int i = 0; i < TB; ++i)
    out[i] = fma((double)e[i], dafmm_fit::LN2, lc[i] + fma(r2[i], fma(r[i], qo[i], qe[i]), r[i]));
#else
  (void)T;
  for (int i = 0; i < TB; ++i) out[i] = std::log(0.25 * z2[i]);
#endif
}

// Near-type band: z <= ZN for ZN in {7, 8, 12}.
template <int ZN, int TB>
DAFMM_HD void h0_near_vec(const double* z2, double* re, double* im, const PolyTable& T) {
  static_assert(ZN == 7 || ZN == 8 || ZN == 12, "near bands are z <= 7, 8 and 12");
  constexpr double ts = ZN == 7 ? dafmm_fit::NEAR7_T_SCALE : ZN == 8 ? dafmm_fit::NEAR8_T_SCALE
                                                                     : dafmm_fit::NEAR12_T_SCALE;
  double t[TB], j0[TB], rr[TB], lu[TB];
#pragma unroll
  for (int i = 0; i < TB; ++i) t[i] = fma(z2[i], ts, -1.0);
  poly_near<ZN, TB>(t, j0, rr);
  log_quarter_vec<TB>(z2, lu, T);
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

// Negate a double when `mask` (0 or 0x80000000) is set: one XOR on the high word.
DAFMM_HD double flip_sign(double v, unsigned mask) {
#ifdef __CUDA_ARCH__
  return __hiloint2double(__double2hiint(v) ^ (int)mask, __double2loint(v));
#else
  return mask ? -v : v;
#endif
}

// Far-type evaluation with a caller-supplied (P, Q) evaluator: pq(x, P, Q) over TB lanes.
template <int TB, class PQ>
DAFMM_HD void h0_far_vec(const double* z2, double* re, double* im, double A, double B, const PQ& pq,
                         const PolyTable& T) {
  double y[TB], x[TB], P[TB], Q[TB], rho[TB], rh2[TB], sp[TB], c[TB];
  int quad[TB];
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    y[i] = rsqrt_sqrt(z2[i]);  // z^(-1/2)
    x[i] = fma(y[i] * y[i], A, B);
  }
  pq(x, P, Q);
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    const double z = z2[i] * (y[i] * y[i]);
    // theta = z - pi/4 = rho + q pi/2, m = q + 1/2, rho = z - m pi/2 (two-part Cody-Waite)
    const double qf = rint(fma(z, dafmm_fit::TWO_OVER_PI, -0.5));
    const double m = qf + 0.5;
    rho[i] = fma(-m, dafmm_fit::PIO2_2, fma(-m, dafmm_fit::PIO2_1, z));
    rh2[i] = rho[i] * rho[i];
    quad[i] = (int)qf;
  }
  dafmm_fit::sincos_imm<TB>(rh2, sp, c);
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    const double s = rho[i] * sp[i];
    // (cos theta, sin theta) = (c, s) rotated by q pi/2: swap for odd q, then signs
    // cos: - for q = 1, 2 (mod 4); sin: - for q = 2, 3 (mod 4)
    const int q = quad[i];
    const bool swap = q & 1;
    const double cr = flip_sign(swap ? s : c[i], (unsigned)((q + 1) & 2) << 30);
    const double sr = flip_sign(swap ? c[i] : s, (unsigned)(q & 2) << 30);
    const double amp = dafmm_fit::SQRT_2_OVER_PI * y[i];  // sqrt(2/(pi z))
    const double pr = amp * P[i], pi_ = amp * Q[i];
    re[i] = fma(pr, cr, -pi_ * sr);
    im[i] = fma(pr, sr, pi_ * cr);
  }
}

// (P, Q) of the generic far band [8, inf).
template <int TB>
struct GenericFarPQ {
  const PolyTable& T;
  DAFMM_HD void operator()(const double* x, double* P, double* Q) const {
    dafmm_fit::generic_far_imm<TB>(x, P, Q);
  }
};

// (P, Q) of a data band (coefficients in shared memory on the device; n is odd and
// CTA-uniform, so the loop runs in coefficient pairs without a remainder).
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
#pragma unroll 1
    for (int k = n - 2; k > 0; k -= 2) {
      const Pair c1 = band->pq[k], c0 = band->pq[k - 1];
#pragma unroll
      for (int i = 0; i < TB; ++i) {
        P[i] = fma(fma(P[i], x[i], c1.a), x[i], c0.a);
        Q[i] = fma(fma(Q[i], x[i], c1.b), x[i], c0.b);
      }
    }
  }
};

// Generic: any z > 0, for segments that straddle the bands (rare).  Both the near-8 and the
// generic far evaluation run on all TB lanes (inputs clamped into each domain) and every lane
// keeps its own: twice the work, but no divergence and no extra code per lane.
template <int TB>
DAFMM_HD void h0_generic_vec(const double* z2, double* re, double* im, const PolyTable& T) {
  double zn[TB], zf[TB], nr[TB], ni[TB], fr[TB], fi[TB];
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    zn[i] = fmin(z2[i], dafmm_fit::NEAR8_Z2_MAX);
    zf[i] = fmax(z2[i], dafmm_fit::NEAR8_Z2_MAX);
  }
  h0_near_vec<8, TB>(zn, nr, ni, T);
  h0_far_vec<TB>(zf, fr, fi, dafmm_fit::GENERIC_FAR_A, dafmm_fit::GENERIC_FAR_B, GenericFarPQ<TB>{T}, T);
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    const bool near = z2[i] <= dafmm_fit::NEAR8_Z2_MAX;
    re[i] = near ? nr[i] : fr[i];
    im[i] = near ? ni[i] : fi[i];
  }
}

// Scalar host evaluation (setup: ACA entries and operators); z2 = (kappa r)^2.
inline cplx h0(double z2) {
  double re, im;
  h0_generic_vec<1>(&z2, &re, &im, dafmm_fit::kPolyHost);
  return {re, im};
}

// Setup-side band choice for a segment whose point pairs have z in [zmin, zmax]: the
// cheapest band (estimated fp64 operations per entry) that covers the whole range.  The M2L
// stream passes allow_near7 = false: one band fewer keeps the persistent kernel free of spills.
inline int choose_band(double zmin, double zmax, bool allow_near7) {
  int best = kBandGeneric;
  double cost = 1e30;
  if (allow_near7 && zmax <= 7.0) {
    best = kBandNear7;
    cost = 47.0;
  } else if (zmax <= 8.0) {
    best = kBandNear8;
    cost = 49.0;
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
// Copy the fixed-degree polynomial table into shared memory (all threads; then a barrier).
__device__ __forceinline__ void load_poly_table(PolyTable& dst) {
  static_assert(sizeof(PolyTable) % sizeof(Pair) == 0, "PolyTable is copied as pairs");
  const Pair* src = reinterpret_cast<const Pair*>(&dafmm_fit::kPolyDev);
  Pair* d = reinterpret_cast<Pair*>(&dst);
  for (int i = threadIdx.x; i < (int)(sizeof(PolyTable) / sizeof(Pair)); i += blockDim.x) d[i] = src[i];
  __syncthreads();
}
// Copy every data band into shared memory (all threads; then a barrier).
__device__ __forceinline__ void load_far_bands(FarBand* dst) {
  static_assert(sizeof(FarBand) % sizeof(Pair) == 0, "FarBand is copied as pairs");
  const Pair* src = reinterpret_cast<const Pair*>(dafmm_fit::kFarBandsDev);
  Pair* d = reinterpret_cast<Pair*>(dst);
  constexpr int n = (int)(dafmm_fit::NUM_FAR * sizeof(FarBand) / sizeof(Pair));
  for (int i = threadIdx.x; i < n; i += blockDim.x) d[i] = src[i];
  __syncthreads();
}
#endif

}  // namespace dafmm
