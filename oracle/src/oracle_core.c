/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU evaluation of the entries of the discrete
 * Lippmann-Schwinger operator A of arxiv 2204.00326 (PAPER.md, cited "P:<line>").
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  It shares no code, header, table or
 * constant generator with the product (paper_2204_00326_b200/).
 *
 * Contents
 *   h0_oracle(z)       H0^(1)(z) = J0(z) + i Y0(z), three bands:
 *                        z <= 8      ascending series  (A&S 9.1.12 / 9.1.13)
 *                        8 < z < 20  Miller backward recurrence for J_n, normalised by
 *                                    J0 + 2 sum J_2k = 1 (A&S 9.1.46), Y0 from the Neumann
 *                                    series (A&S 9.1.88)
 *                        z >= 20     Hankel asymptotic expansion (A&S 9.2.7), truncated at
 *                                    the smallest term
 *                      The paper only names the function: G_k(x,y) = (i/4) H0^(1)(k|x-y|).
 *   h1_series(z)       H1^(1) by its ascending series (A&S 9.1.10 / 9.1.11), small z only.
 *   self_term_disk     D = int_{|y|<R} G_k(0,y) dy = (i pi R / (2k)) H1(kR) - 1/k^2 with
 *                      R = sqrt(w/pi): the diagonal reading D1 (R1).  The paper's Eq. 13
 *                       integrates G over the cell; for a point rule the cell is the
 *                      equal-area disk.
 *   A_block            entries A_ij of Eq. 12a/13 in point form:
 *                        A_ij = k^2 q_i G(x_i,x_j) w_j          (i != j)
 *                        A_ii = 1 + k^2 q_i D_i
 *   K_block            entries of the discretised volume potential V (Eq. 5) that the
 *                      DAFMM accelerates (reading R9): A = I + k^2 diag(q) K with
 *                        K_ij = G(x_i,x_j) w_j   (i != j),      K_ii = D_i
 *   dense_matvec       y = A x by direct summation over all j (the plain definition), optionally
 *                      on a subset of rows.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define ORACLE_PI 3.14159265358979323846264338327950288
#define ORACLE_EULER_GAMMA 0.57721566490153286060651209008240243

/* ---- Band 1: ascending series, A&S 9.1.12 (J0) and 9.1.13 (Y0) -------------------------
 * J0(z) = sum_k (-u)^k / (k!)^2,  u = z^2/4
 * Y0(z) = (2/pi) [ (ln(z/2) + gamma) J0(z) + sum_{k>=1} (-1)^(k+1) H_k u^k / (k!)^2 ]
 * with H_k the k-th harmonic number. */
static void j0y0_series(double z, double *j0, double *y0) {
  double u = 0.25 * z * z;
  double term = 1.0; /* (-u)^k / (k!)^2 */
  double sum_j = 1.0, sum_y = 0.0, harmonic = 0.0;
  for (int k = 1; k < 400; ++k) {
    term *= -u / ((double)k * (double)k);
    harmonic += 1.0 / k;
    sum_j += term;
    sum_y -= harmonic * term; /* (-1)^(k+1) H_k u^k/(k!)^2 = -H_k * term */
    if ((double)k > u && fabs(term) * (1.0 + harmonic) < 1e-22) break;
  }
  *j0 = sum_j;
  *y0 = (2.0 / ORACLE_PI) * ((log(0.5 * z) + ORACLE_EULER_GAMMA) * sum_j + sum_y);
}

/* ---- Band 2: Miller's backward recurrence + Neumann series --------------------------------
 * J_{n-1}(z) = (2n/z) J_n(z) - J_{n+1}(z), run downward from n = N with J_{N+1}=0, J_N=tiny,
 * normalised by 1 = J0 + 2 sum_{k>=1} J_{2k} (A&S 9.1.46);
 * Y0(z) = (2/pi)(ln(z/2)+gamma) J0(z) - (4/pi) sum_{k>=1} (-1)^k J_{2k}(z)/k (A&S 9.1.88). */
static void j0y0_miller(double z, double *j0, double *y0) {
  int N = 2 * (int)((z + 80.0) / 2.0); /* even start index, well above z */
  double *J = (double *)malloc(sizeof(double) * (size_t)(N + 2));
  J[N + 1] = 0.0;
  J[N] = 1e-200;
  for (int n = N; n >= 1; --n) {
    J[n - 1] = (2.0 * n / z) * J[n] - J[n + 1];
    if (fabs(J[n - 1]) > 1e200) { /* rescale everything computed so far */
      for (int m = n - 1; m <= N + 1; ++m) J[m] *= 1e-200;
    }
  }
  double norm = J[0];
  for (int k = 1; 2 * k <= N; ++k) norm += 2.0 * J[2 * k];
  double neumann = 0.0;
  for (int k = 1; 2 * k <= N; ++k) neumann += ((k % 2) ? -1.0 : 1.0) * (J[2 * k] / norm) / k;
  *j0 = J[0] / norm;
  *y0 = (2.0 / ORACLE_PI) * (log(0.5 * z) + ORACLE_EULER_GAMMA) * (*j0) - (4.0 / ORACLE_PI) * neumann;
  free(J);
}

/* ---- Band 3: Hankel asymptotic expansion, A&S 9.2.7 with nu = 0 -----------------------------
 * H0(z) ~ sqrt(2/(pi z)) e^{i(z - pi/4)} sum_k (-i)^k a_k z^{-k},
 * a_k = prod_{j<=k} (2j-1)^2 / (k! 8^k); truncated before the first increasing term. */
static double complex h0_asymptotic(double z) {
  double complex sum = 1.0, term = 1.0;
  double last = 1.0;
  for (int k = 1; k <= 60; ++k) {
    term *= -I * ((2.0 * k - 1.0) * (2.0 * k - 1.0)) / (8.0 * k * z);
    double mag = cabs(term);
    if (mag > last) break; /* optimal truncation: smallest term reached */
    sum += term;
    last = mag;
    if (mag < 1e-18) break;
  }
  double phase = z - 0.25 * ORACLE_PI;
  return sqrt(2.0 / (ORACLE_PI * z)) * (cos(phase) + I * sin(phase)) * sum;
}

/* H0^(1)(z) = J0(z) + i Y0(z), z > 0. */
double complex h0_oracle(double z) {
  double j0, y0;
  if (z <= 8.0) {
    j0y0_series(z, &j0, &y0);
  } else if (z < 20.0) {
    j0y0_miller(z, &j0, &y0);
  } else {
    return h0_asymptotic(z);
  }
  return j0 + I * y0;
}

/* H1^(1)(z) = J1 + i Y1 by the ascending series (A&S 9.1.10, 9.1.11 with n = 1):
 * J1 = (z/2) sum_k (-u)^k / (k!(k+1)!)
 * Y1 = -2/(pi z) + (2/pi) ln(z/2) J1 - (1/pi)(z/2) sum_k [psi(k+1)+psi(k+2)] (-u)^k/(k!(k+1)!)
 * psi(k+1) = -gamma + H_k.  Used only for the self term, where z = kR is small. */
double complex h1_series(double z) {
  double u = 0.25 * z * z;
  double term = 1.0; /* (-u)^k / (k! (k+1)!) */
  double harmonic_k = 0.0, harmonic_k1 = 1.0; /* H_k, H_{k+1} */
  double sum_j = 1.0;
  double sum_y = (-ORACLE_EULER_GAMMA + harmonic_k) + (-ORACLE_EULER_GAMMA + harmonic_k1);
  for (int k = 1; k < 400; ++k) {
    term *= -u / ((double)k * (double)(k + 1));
    harmonic_k += 1.0 / k;
    harmonic_k1 += 1.0 / (k + 1);
    sum_j += term;
    sum_y += ((-ORACLE_EULER_GAMMA + harmonic_k) + (-ORACLE_EULER_GAMMA + harmonic_k1)) * term;
    if ((double)k > u && fabs(term) * (2.0 + harmonic_k1) < 1e-22) break;
  }
  double j1 = 0.5 * z * sum_j;
  double y1 = -2.0 / (ORACLE_PI * z) + (2.0 / ORACLE_PI) * log(0.5 * z) * j1 - (1.0 / ORACLE_PI) * 0.5 * z * sum_y;
  return j1 + I * y1;
}

/* Self term of reading D1: integral of G_k(0,y) over the disk of area w. */
double complex self_term_disk(double kappa, double w) {
  double R = sqrt(w / ORACLE_PI);
  return (I * ORACLE_PI * R / (2.0 * kappa)) * h1_series(kappa * R) - 1.0 / (kappa * kappa);
}

/* ---- exported C-ABI of the oracle library (called through ctypes by oracle/*.py) -------- */

/* out[k] = H0^(1)(z[k]) as (re, im) pairs. */
void oracle_h0(const double *z, int64_t n, double *out) {
  for (int64_t k = 0; k < n; ++k) {
    double complex h = h0_oracle(z[k]);
    out[2 * k] = creal(h);
    out[2 * k + 1] = cimag(h);
  }
}

void oracle_h1_small(const double *z, int64_t n, double *out) {
  for (int64_t k = 0; k < n; ++k) {
    double complex h = h1_series(z[k]);
    out[2 * k] = creal(h);
    out[2 * k + 1] = cimag(h);
  }
}

/* D_i for every point (mode 0: zero, mode 1: disk reading D1). */
void oracle_self_terms(const double *w, int64_t n, double kappa, int mode, double *out) {
  for (int64_t k = 0; k < n; ++k) {
    double complex d = (mode == 1) ? self_term_disk(kappa, w[k]) : 0.0;
    out[2 * k] = creal(d);
    out[2 * k + 1] = cimag(d);
  }
}

/* Entry A_ij of the discrete operator (point form; diagonal per D1). */
static double complex A_entry(int64_t i, int64_t j, const double *pts, const double *w, const double *q,
                              const double *D, double kappa) {
  if (i == j) return 1.0 + kappa * kappa * q[i] * (D[2 * i] + I * D[2 * i + 1]);
  double dx = pts[2 * i] - pts[2 * j], dy = pts[2 * i + 1] - pts[2 * j + 1];
  double r = sqrt(dx * dx + dy * dy);
  double complex G = 0.25 * I * h0_oracle(kappa * r);
  return kappa * kappa * q[i] * G * w[j];
}

/* Entry K_ij of the discretised volume potential (reading R9). */
static double complex K_entry(int64_t i, int64_t j, const double *pts, const double *w, const double *D,
                              double kappa) {
  if (i == j) return D[2 * i] + I * D[2 * i + 1];
  double dx = pts[2 * i] - pts[2 * j], dy = pts[2 * i + 1] - pts[2 * j + 1];
  double r = sqrt(dx * dx + dy * dy);
  return 0.25 * I * h0_oracle(kappa * r) * w[j];
}

/* out (n_rows x n_cols, row-major, complex) = K[rows, cols]. */
void oracle_K_block(const int64_t *rows, int64_t n_rows, const int64_t *cols, int64_t n_cols, const double *pts,
                    const double *w, const double *D, double kappa, double *out) {
  /* every entry independently (a single ACA row is one long row: threads over all entries) */
#pragma omp parallel for collapse(2) schedule(static) if (n_rows * n_cols > 512)
  for (int64_t a = 0; a < n_rows; ++a) {
    for (int64_t b = 0; b < n_cols; ++b) {
      double complex v = K_entry(rows[a], cols[b], pts, w, D, kappa);
      out[2 * (a * n_cols + b)] = creal(v);
      out[2 * (a * n_cols + b) + 1] = cimag(v);
    }
  }
}

/* out (n_rows x n_cols, row-major, complex) = A[rows, cols]. */
void oracle_A_block(const int64_t *rows, int64_t n_rows, const int64_t *cols, int64_t n_cols, const double *pts,
                    const double *w, const double *q, const double *D, double kappa, double *out) {
#pragma omp parallel for collapse(2) schedule(static) if (n_rows * n_cols > 512)
  for (int64_t a = 0; a < n_rows; ++a) {
    for (int64_t b = 0; b < n_cols; ++b) {
      double complex v = A_entry(rows[a], cols[b], pts, w, q, D, kappa);
      out[2 * (a * n_cols + b)] = creal(v);
      out[2 * (a * n_cols + b) + 1] = cimag(v);
    }
  }
}

/* y[rows[a]] = sum_j A[rows[a], j] x[j]: the dense product by definition (all j, N^2 work). */
void oracle_dense_matvec_rows(const int64_t *rows, int64_t n_rows, const double *pts, const double *w,
                              const double *q, const double *D, double kappa, int64_t n, const double *x,
                              double *y) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t a = 0; a < n_rows; ++a) {
    int64_t i = rows[a];
    double complex acc = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      acc += A_entry(i, j, pts, w, q, D, kappa) * (x[2 * j] + I * x[2 * j + 1]);
    }
    y[2 * a] = creal(acc);
    y[2 * a + 1] = cimag(acc);
  }
}
