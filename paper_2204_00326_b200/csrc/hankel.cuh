// H0^(1)(z) = J0(z) + i Y0(z) for the product (host setup and device kernels share this code).
//
// The paper only names the kernel G_k(x,y) = (i/4) H0^(1)(k|x-y|).  This
// is the product's own evaluator, independent of the oracle's series /
// Miller / asymptotic bands:
//   near band  z < 8 : J0 = pJ(t), Y0 = (1/pi) ln(u) J0 + pR(t),  u = z^2/4, t = u/8 - 1
//   far band   z >= 8: H0 = sqrt(2/(pi z)) (P + iQ) e^{i(z - pi/4)},  P, Q polynomials in
//                      v = 2 (8/z)^2 - 1 (Hankel's P/Q functions fitted by tools/fit_hankel.py)
// Both take the squared distance r2 = |x - y|^2 so the near band never needs a square root.
#pragma once
#include "common.h"
#include "hankel_coeffs.h"

namespace dafmm {

constexpr double kPi = 3.14159265358979323846;
constexpr double kInvPi = 0.31830988618379067154;
constexpr double kTwoOverPi = 0.63661977236758134308;

struct KernelConsts {
  double kappa;      // wavenumber
  double inv_kappa;  // 1 / kappa
  double quarter_k2; // kappa^2 / 4   (u = z^2 / 4 = quarter_k2 * r2)
  double amp_k;      // sqrt(2 / (pi kappa))
};

inline KernelConsts make_kernel_consts(double kappa) {
  return {kappa, 1.0 / kappa, 0.25 * kappa * kappa, std::sqrt(2.0 / (kPi * kappa))};
}

DAFMM_HD double dafmm_rsqrt(double x) {
#ifdef __CUDA_ARCH__
  return rsqrt(x);
#else
  return 1.0 / std::sqrt(x);
#endif
}

// Near band (z < 8): valid for 0 < r2 with kappa^2 r2 / 4 <= 16.
DAFMM_HD cplx h0_near(double r2, const KernelConsts& k) {
  double u = k.quarter_k2 * r2;
  double t = fma(u, 2.0 / dafmm_fit::U_MAX, -1.0);
  double j0 = dafmm_fit::near_j0(t);
  double rr = dafmm_fit::near_r(t);
  double y0 = fma(kInvPi * log(u), j0, rr);
  return {j0, y0};
}

// Far band (z >= 8).
DAFMM_HD cplx h0_far(double r2, const KernelConsts& k) {
  double ir = dafmm_rsqrt(r2);            // 1/r
  double z = k.kappa * (r2 * ir);         // kappa r
  double iz = ir * k.inv_kappa;           // 1/z
  double sq = (dafmm_fit::Z_FAR * iz);    // 8/z = sqrt(s)
  double v = fma(2.0 * sq, sq, -1.0);     // 2 s - 1
  double P = dafmm_fit::far_p(v);
  double Q = dafmm_fit::far_q(v) * sq;
  double amp = k.amp_k * sqrt(ir);        // sqrt(2/(pi z))
  // theta = z - pi/4 = rho + q pi/2 with m = q + 1/2:  rho = z - m pi/2 (Cody-Waite, 3 parts)
  double qf = rint(fma(z, kTwoOverPi, -0.5));
  double m = qf + 0.5;
  double rho = fma(-m, dafmm_fit::PIO2_1, z);
  rho = fma(-m, dafmm_fit::PIO2_2, rho);
  rho = fma(-m, dafmm_fit::PIO2_3, rho);
  double w = fma(rho * rho, 2.0 / dafmm_fit::SC_R2MAX, -1.0);
  double s = rho * dafmm_fit::sin_over_x(w);
  double c = dafmm_fit::cos_poly(w);
  int quadrant = ((int)qf) & 3;
  double cr, sr;  // cos/sin of theta
  if (quadrant == 0) { cr = c; sr = s; }
  else if (quadrant == 1) { cr = -s; sr = c; }
  else if (quadrant == 2) { cr = -c; sr = -s; }
  else { cr = s; sr = -c; }
  double pr = amp * P, pi_ = amp * Q;
  return {fma(pr, cr, -pi_ * sr), fma(pr, sr, pi_ * cr)};
}

// Band selection by squared distance: z < 8  <=>  u = kappa^2 r2 / 4 < 16.
DAFMM_HD cplx h0(double r2, const KernelConsts& k) {
  if (k.quarter_k2 * r2 < dafmm_fit::U_MAX) return h0_near(r2, k);
  return h0_far(r2, k);
}

}  // namespace dafmm
