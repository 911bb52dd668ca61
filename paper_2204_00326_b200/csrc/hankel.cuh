// H0^(1)(z) = J0(z) + i Y0(z) for the product (host setup and device kernels share this code).
//
// The paper only names the kernel G_k(x,y) = (i/4) H0^(1)(k|x-y|).  This is
// the product's own evaluator, independent of the oracle's series / Miller /
// asymptotic bands.  Every entry point takes the squared distance r2 = |x - y|^2.
//
//   near band, z <= 8:  J0 = pJ(t), Y0 = (1/pi) ln(u) J0 + pR(t),  u = z^2/4, t = u/8 - 1
//   far-type band b, z in [ZLO_b, ZHI_b]:
//       H0 = sqrt(2/(pi z)) (P_b(x) + i Q_b(x)) e^{i(z - pi/4)},  x = A_b / z + B_b
//   generic (any z > 0): per-lane choice of the near band or far band 0 ([8, inf)).
//
// Evaluators are lane-blocked: one call evaluates TB independent entries in lockstep, so each
// literal coefficient (one uniform-register immediate) is shared by TB FMAs and the TB Horner
// chains hide each other's latency.  Kernels pick one band per CTA-uniform work segment (setup
// classifies every interaction by the exact [z_min, z_max] of its point pairs, DESIGN.md
// §Kernels), so the band is a template parameter and inner loops never diverge.  ln u uses a
// 128-entry table of (1/c_i, ln c_i): device callers pass its shared-memory copy
// (load_log_table), host callers kLogTabHost.
#pragma once
#include "common.h"
#include "hankel_coeffs.h"

namespace dafmm {

constexpr double kPi = 3.14159265358979323846;

using dafmm_fit::Pair;

struct KernelConsts {
  double kappa;       // wavenumber
  double inv_kappa;   // 1 / kappa
  double quarter_k2;  // kappa^2 / 4   (u = z^2 / 4 = quarter_k2 * r2)
  double amp_k;       // sqrt(2 / (pi kappa))
  double r2_safe;     // a squared distance inside every band's domain (u = 1), for masked lanes
};

inline KernelConsts make_kernel_consts(double kappa) {
  return {kappa, 1.0 / kappa, 0.25 * kappa * kappa, std::sqrt(2.0 / (kPi * kappa)), 4.0 / (kappa * kappa)};
}

// Band codes of a work segment: 0 generic, 1 near, 2 + b far-type band b.
constexpr int kBandGeneric = 0;
constexpr int kBandNear = 1;
constexpr int kNumBandCodes = 2 + dafmm_fit::NUM_FAR;

// ln u for TB positive normal u.
template <int TB>
DAFMM_HD void log_vec(const double* u, double* out, const Pair* logtab) {
#ifdef __CUDA_ARCH__
  double r[TB], r2[TB], qe[TB], qo[TB], lc[TB];
  int e[TB];
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    const int hi = __double2hiint(u[i]);
    e[i] = (hi >> 20) - 1023;
    const int ix = (hi >> (20 - dafmm_fit::LOG_BITS)) & ((1 << dafmm_fit::LOG_BITS) - 1);
    const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, __double2loint(u[i]));  // [1, 2)
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
  for (int i = 0; i < TB; ++i) out[i] = std::log(u[i]);
#endif
}

// Near band (z <= 8): valid for 0 < r2 with kappa^2 r2 / 4 <= 16.
template <int TB>
DAFMM_HD void h0_near_vec(const double* r2, double* re, double* im, const KernelConsts& k, const Pair* logtab) {
  double u[TB], t[TB], j0[TB], rr[TB], lu[TB];
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    u[i] = k.quarter_k2 * r2[i];
    t[i] = fma(u[i], dafmm_fit::T_SCALE, -1.0);
  }
  dafmm_fit::near_jr<TB>(t, j0, rr);
  log_vec<TB>(u, lu, logtab);
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    re[i] = j0[i];
    im[i] = fma(dafmm_fit::INV_PI * lu[i], j0[i], rr[i]);
  }
}

// y = r2^(-1/4) = r^(-1/2): fp32 MUFU seed (r2 must lie in the normal fp32 range), two Newton
// steps y <- y (5 - r2 y^4) / 4 in fp64.
DAFMM_HD double rsqrt_sqrt(double r2) {
#ifdef __CUDA_ARCH__
  float f = __double2float_rn(r2), g;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(g) : "f"(f));
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(f) : "f"(g));
  double y = (double)f;
  const double mq = -0.25 * r2;
  double y2 = y * y;
  y *= fma(mq, y2 * y2, 1.25);
  y2 = y * y;
  y *= fma(mq, y2 * y2, 1.25);
  return y;
#else
  return 1.0 / std::sqrt(std::sqrt(r2));
#endif
}

// Far-type band B: valid for z = kappa r in [FAR_ZLO[B], FAR_ZHI[B]].
template <int B, int TB>
DAFMM_HD void h0_far_vec(const double* r2, double* re, double* im, const KernelConsts& k) {
  double y[TB], z[TB], x[TB], P[TB], Q[TB], rho[TB], rh2[TB], sp[TB], c[TB];
  int quad[TB];
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    y[i] = rsqrt_sqrt(r2[i]);            // r^(-1/2)
    const double ir = y[i] * y[i];       // 1/r
    z[i] = k.kappa * (r2[i] * ir);       // kappa r
    x[i] = fma(ir * k.inv_kappa, dafmm_fit::FarPQ<B>::A, dafmm_fit::FarPQ<B>::B);
  }
  dafmm_fit::FarPQ<B>::template eval<TB>(x, P, Q);
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    // theta = z - pi/4 = rho + q pi/2, m = q + 1/2, rho = z - m pi/2 (Cody-Waite, 3 parts)
    const double qf = rint(fma(z[i], dafmm_fit::TWO_OVER_PI, -0.5));
    const double m = qf + 0.5;
    double t = fma(-m, dafmm_fit::PIO2_1, z[i]);
    t = fma(-m, dafmm_fit::PIO2_2, t);
    rho[i] = fma(-m, dafmm_fit::PIO2_3, t);
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
    const double amp = k.amp_k * y[i];   // sqrt(2/(pi z))
    const double pr = amp * P[i], pi_ = amp * Q[i];
    re[i] = fma(pr, cr, -pi_ * sr);
    im[i] = fma(pr, sr, pi_ * cr);
  }
}

// Generic: any z > 0 (per-lane band choice; used where a segment straddles the bands).
template <int TB>
DAFMM_HD void h0_generic_vec(const double* r2, double* re, double* im, const KernelConsts& k,
                             const Pair* logtab) {
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    if (k.quarter_k2 * r2[i] <= dafmm_fit::U_MAX) h0_near_vec<1>(r2 + i, re + i, im + i, k, logtab);
    else h0_far_vec<0, 1>(r2 + i, re + i, im + i, k);
  }
}

// Evaluation by band code (compile-time).
template <int CODE, int TB>
DAFMM_HD void h0_band_vec(const double* r2, double* re, double* im, const KernelConsts& k, const Pair* logtab) {
  if constexpr (CODE == kBandGeneric) h0_generic_vec<TB>(r2, re, im, k, logtab);
  else if constexpr (CODE == kBandNear) h0_near_vec<TB>(r2, re, im, k, logtab);
  else h0_far_vec<CODE - 2, TB>(r2, re, im, k);
}

// Scalar host evaluation (setup: ACA entries and operators).
inline cplx h0(double r2, const KernelConsts& k) {
  double re, im;
  h0_generic_vec<1>(&r2, &re, &im, k, dafmm_fit::kLogTabHost);
  return {re, im};
}

// Setup-side band choice for a segment whose point pairs have z in [zmin, zmax]: the
// cheapest band (estimated fp64 operations per entry) that covers the whole range.
inline int choose_band(double zmin, double zmax) {
  int best = kBandGeneric;
  double cost = 1e30;
  if (zmax <= dafmm_fit::Z_NEAR) {
    best = kBandNear;
    cost = 52.0;
  }
  for (int b = 0; b < dafmm_fit::NUM_FAR; ++b) {
    if (zmin >= dafmm_fit::FAR_ZLO[b] && zmax <= dafmm_fit::FAR_ZHI[b]) {
      double c = 44.0 + 2.0 * dafmm_fit::FAR_N[b];
      if (c < cost) {
        cost = c;
        best = 2 + b;
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
#endif

}  // namespace dafmm
