// Host setup of the DAFMM plan: quadtree, regimes, cones, neighbour and
// interaction lists, nested cross approximation pivots and the
// translation operators in the form the device passes consume.
//
// Product code: shares nothing with oracle/.  Readings of silent passages are the
// R-numbers of DESIGN.md.  Everything here runs once per handle and is timed separately
// from the matvec (dafmm_stats).
#include <omp.h>

#include <memory>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <tuple>
#include <sys/stat.h>

#include "dafmm.h"
#include "plan.h"
#include "setup_device.h"

namespace dafmm {

namespace {

constexpr double kPhi0 = kPi / 4096.0;  // R5: cone boundaries at odd multiples of pi/4096

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

uint64_t pack_key(int64_t ix, int64_t iy) { return ((uint64_t)ix << 32) | (uint64_t)(uint32_t)iy; }

uint64_t spread_bits(uint64_t v) {
  uint64_t r = 0;
  for (int b = 0; b < 32; ++b) r |= ((v >> b) & 1ull) << (2 * b);
  return r;
}
uint64_t morton(int64_t ix, int64_t iy) { return spread_bits((uint64_t)ix) | (spread_bits((uint64_t)iy) << 1); }

// ---- self term (reading D1): D = (i pi R / (2 kappa)) H1(kappa R) - 1/kappa^2, R = sqrt(w/pi) ----
// H1^(1)(z) for small z from the power series of J1 and Y1 (Bessel's series; z <= 8 here).
zd hankel1_small(double z) {
  const double g = 0.57721566490153286061;
  double h = 0.25 * z * z;
  double c = 1.0;          // (-h)^k / (k! (k+1)!)
  double sj = 0.0, sy = 0.0;
  double psi_k = -g, psi_k1 = 1.0 - g;  // psi(k+1), psi(k+2)
  for (int k = 0; k < 300; ++k) {
    if (k > 0) {
      c *= -h / (double(k) * double(k + 1));
      psi_k += 1.0 / k;
      psi_k1 += 1.0 / (k + 1);
    }
    sj += c;
    sy += (psi_k + psi_k1) * c;
    if (k > h && std::fabs(c) < 1e-24) break;
  }
  double j1 = 0.5 * z * sj;
  double y1 = -2.0 / (kPi * z) + (2.0 / kPi) * std::log(0.5 * z) * j1 - (0.5 * z / kPi) * sy;
  return zd(j1, y1);
}

zd self_term_disk(double kappa, double w) {
  double R = std::sqrt(w / kPi);
  return zd(0.0, kPi * R / (2.0 * kappa)) * hankel1_small(kappa * R) - 1.0 / (kappa * kappa);
}

// Square cell of side h = sqrt(w) (option self_term = 2; Eq. 13 integrates G over the cell,
// P:260): 8 triangles in polar coordinates, the radial integral in closed form
// (z H1(z))' = z H0(z), z H1(z) -> -2i/pi as z -> 0, the smooth angular integral over
// [0, pi/4] by Gauss-Legendre with 40 nodes (Newton on the Legendre recurrence).
zd self_term_square(double kappa, double w) {
  constexpr int kN = 40;
  static double node[kN], weight[kN];
  static bool init = false;
#pragma omp critical(gauss_legendre)
  if (!init) {
    for (int i = 0; i < kN; ++i) {
      double x = std::cos(kPi * (i + 0.75) / (kN + 0.5)), dp = 1.0;
      for (int it = 0; it < 100; ++it) {
        double p0 = 1.0, p1 = x;
        for (int k = 2; k <= kN; ++k) {
          const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
          p0 = p1;
          p1 = p2;
        }
        dp = kN * (x * p1 - p0) / (x * x - 1.0);
        const double dx = p1 / dp;
        x -= dx;
        if (std::fabs(dx) < 1e-16) break;
      }
      node[i] = x;
      weight[i] = 2.0 / ((1.0 - x * x) * dp * dp);
    }
    init = true;
  }
  const double h = std::sqrt(w);
  zd acc(0.0, 0.0);
  for (int i = 0; i < kN; ++i) {
    const double th = (node[i] + 1.0) * (kPi / 8.0);
    const double z = kappa * h / (2.0 * std::cos(th));
    acc += weight[i] * (z * hankel1_small(z) + zd(0.0, 2.0 / kPi));
  }
  return zd(0.0, 0.25) * 8.0 * (kPi / 8.0) * acc / (kappa * kappa);
}

// ---- complex LU with partial pivoting (reading R12: solves, never explicit inverses) ----
struct LU {
  int r = 0;
  std::vector<zd> a;  // row-major, factors in place
  std::vector<int> p;
  bool factor(const std::vector<zd>& m, int n) {
    r = n;
    a = m;
    p.resize(n);
    for (int k = 0; k < n; ++k) {
      int piv = k;
      double best = std::abs(a[(size_t)k * n + k]);
      for (int i = k + 1; i < n; ++i) {
        double v = std::abs(a[(size_t)i * n + k]);
        if (v > best) { best = v; piv = i; }
      }
      if (!(best > 0.0)) return false;
      p[k] = piv;
      if (piv != k)
        for (int j = 0; j < n; ++j) std::swap(a[(size_t)k * n + j], a[(size_t)piv * n + j]);
      zd inv = 1.0 / a[(size_t)k * n + k];
      for (int i = k + 1; i < n; ++i) {
        zd f = a[(size_t)i * n + k] * inv;
        a[(size_t)i * n + k] = f;
        if (f != 0.0)
          for (int j = k + 1; j < n; ++j) a[(size_t)i * n + j] -= f * a[(size_t)k * n + j];
      }
    }
    return true;
  }
  // Solve A x = b in place (b length r).
  void solve(zd* b) const {
    int n = r;
    for (int k = 0; k < n; ++k)
      if (p[k] != k) std::swap(b[k], b[p[k]]);
    for (int i = 0; i < n; ++i) {
      zd s = b[i];
      for (int j = 0; j < i; ++j) s -= a[(size_t)i * n + j] * b[j];
      b[i] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
      zd s = b[i];
      for (int j = i + 1; j < n; ++j) s -= a[(size_t)i * n + j] * b[j];
      b[i] = s / a[(size_t)i * n + i];
    }
  }
};

struct Ctx {
  const Plan& p;
  double k2;
  explicit Ctx(const Plan& plan) : p(plan), k2(plan.kappa * plan.kappa) {}
  // H0^(1)(kappa |x_i - x_j|), i != j (original indices)
  zd H(int32_t i, int32_t j) const {
    double dx = p.pts[2 * (size_t)i] - p.pts[2 * (size_t)j];
    double dy = p.pts[2 * (size_t)i + 1] - p.pts[2 * (size_t)j + 1];
    cplx h = h0(k2 * (dx * dx + dy * dy));
    return zd(h.re, h.im);
  }
  // K_ij = G(x_i, x_j) w_j: the discretised volume potential compressed by the NCA (reading R9)
  zd K(int32_t i, int32_t j) const { return zd(0.0, 0.25) * H(i, j) * p.w[j]; }
};

// ---- partially pivoted ACA on K[rows, cols] (stopping rule of Rjasanow 2002
// cited at P:816; tie-breaking and termination of reading R10) ----
void aca(const Ctx& cx, const std::vector<int32_t>& rows, const std::vector<int32_t>& cols, double eps,
         std::vector<int32_t>& prow, std::vector<int32_t>& pcol, int64_t& entries) {
  prow.clear();
  pcol.clear();
  const int m = (int)rows.size(), n = (int)cols.size();
  if (m == 0 || n == 0) return;
  const int cap = std::min(std::min(m, n), 200);
  std::vector<zd> U, V;  // k x m, k x n
  U.reserve((size_t)cap * m);
  V.reserve((size_t)cap * n);
  std::vector<char> used_r(m, 0), used_c(n, 0);
  std::vector<zd> r(n), u(m);
  double norm2 = 0.0;
  int i = 0, k = 0;
  // R10: a residual row whose largest entry is at rounding level relative to the row itself
  // (<= 1e3 eps x its largest original entry) lies in the span of the earlier terms; pivoting on
  // it would make the cross matrix singular, so it counts as a zero row
  constexpr double kZeroRowRtol = 1e3 * 2.220446049250313e-16;
  while (k < cap) {
    double row_max = 0.0;
    for (int j = 0; j < n; ++j) {
      r[j] = cx.K(rows[i], cols[j]);
      row_max = std::max(row_max, std::abs(r[j]));
    }
    entries += n;
    for (int l = 0; l < k; ++l) {
      zd ul = U[(size_t)l * m + i];
      const zd* vl = &V[(size_t)l * n];
      for (int j = 0; j < n; ++j) r[j] -= ul * vl[j];
    }
    used_r[i] = 1;
    int jm = -1;
    double best = -1.0;
    for (int j = 0; j < n; ++j) {
      if (used_c[j]) continue;
      double a = std::abs(r[j]);
      if (a > best) { best = a; jm = j; }
    }
    if (!(best > kZeroRowRtol * row_max)) {
      int nxt = -1;
      for (int t = 0; t < m; ++t)
        if (!used_r[t]) { nxt = t; break; }
      if (nxt < 0) break;
      i = nxt;
      continue;
    }
    zd inv = 1.0 / r[jm];
    for (int j = 0; j < n; ++j) r[j] *= inv;  // v
    for (int t = 0; t < m; ++t) u[t] = cx.K(rows[t], cols[jm]);
    entries += m;
    for (int l = 0; l < k; ++l) {
      zd vl = V[(size_t)l * n + jm];
      const zd* ul = &U[(size_t)l * m];
      for (int t = 0; t < m; ++t) u[t] -= vl * ul[t];
    }
    double cross = 0.0;
    for (int l = 0; l < k; ++l) {
      zd du = 0.0, dv = 0.0;
      const zd* ul = &U[(size_t)l * m];
      const zd* vl = &V[(size_t)l * n];
      for (int t = 0; t < m; ++t) du += std::conj(ul[t]) * u[t];
      for (int j = 0; j < n; ++j) dv += std::conj(vl[j]) * r[j];
      cross += 2.0 * std::real(du * dv);
    }
    double nu2 = 0.0, nv2 = 0.0;
    for (int t = 0; t < m; ++t) nu2 += std::norm(u[t]);
    for (int j = 0; j < n; ++j) nv2 += std::norm(r[j]);
    norm2 += cross + nu2 * nv2;
    if (k > 0 && std::sqrt(nu2 * nv2) <= eps * std::sqrt(norm2)) break;
    U.insert(U.end(), u.begin(), u.end());
    V.insert(V.end(), r.begin(), r.end());
    prow.push_back(rows[i]);
    pcol.push_back(cols[jm]);
    used_c[jm] = 1;
    ++k;
    bool all = true;
    int im = -1;
    double bu = -1.0;
    for (int t = 0; t < m; ++t) {
      if (used_r[t]) continue;
      all = false;
      double a = std::abs(u[t]);
      if (a > bu) { bu = a; im = t; }
    }
    if (all) break;
    i = im;
  }
}

int cone_of(int n, int64_t dx, int64_t dy, bool& ok) {
  double a = std::atan2((double)dy, (double)dx) - kPhi0;
  if (a < 0.0) a += 2.0 * kPi;
  double t = a * n / (2.0 * kPi);
  double fl = std::floor(t);
  double frac = t - fl;
  ok = std::min(frac, 1.0 - frac) > 1e-9;
  return ((int)fl) % n;
}

void sorted_union(std::vector<int32_t>& v) {
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
}

}  // namespace

// ============================================================================================
int build_plan(Plan& P, const double* points, const double* weights, const double* q, int64_t n, double kappa,
               int leaf_size, double nca_tol, const Options& opt, std::string& err) {
  double t0 = now_s();
  if (!points || !weights || !q) { err = "null input pointer"; return DAFMM_EINVAL; }
  if (n <= 0 || n > (int64_t)1 << 30) { err = "n must be in [1, 2^30]"; return DAFMM_EINVAL; }
  if (!(kappa > 0.0) || !std::isfinite(kappa)) { err = "kappa must be positive and finite"; return DAFMM_EINVAL; }
  if (!(nca_tol > 0.0 && nca_tol < 1.0)) { err = "nca_tol must be in (0, 1)"; return DAFMM_EINVAL; }
  if (leaf_size < 1) { err = "leaf_size must be >= 1"; return DAFMM_EINVAL; }
  if (!(opt.T > 0.0) || opt.self_term < 0 || opt.self_term > 2 || opt.kernel_mode < 0 || opt.kernel_mode > 1 ||
      opt.max_level < 0 || opt.max_level > 24 || opt.w_reading < 0 || opt.w_reading > 1) {
    err = "invalid options";
    return DAFMM_EINVAL;
  }
  if (opt.num_threads > 0) omp_set_num_threads(opt.num_threads);
  P.opt = opt;
  P.n = n;
  P.kappa = kappa;
  P.nca_tol = nca_tol;
  P.pts.assign(points, points + 2 * n);
  P.w.assign(weights, weights + n);
  P.q.assign(q, q + n);
  for (int64_t i = 0; i < n; ++i) {
    if (!std::isfinite(P.pts[2 * i]) || !std::isfinite(P.pts[2 * i + 1]) || !std::isfinite(P.q[i]) ||
        !std::isfinite(P.w[i])) {
      err = "non-finite input at index " + std::to_string(i);
      return DAFMM_EINVAL;
    }
    if (!(P.w[i] > 0.0)) { err = "weights must be > 0"; return DAFMM_EINVAL; }
    if (opt.self_term == 1 && kappa * std::sqrt(P.w[i] / kPi) > 8.0) {
      err = "self-term disk too large (kappa sqrt(w/pi) > 8)";
      return DAFMM_EINVAL;
    }
    if (opt.self_term == 2 && kappa * std::sqrt(0.5 * P.w[i]) > 8.0) {
      err = "self-term square too large (kappa sqrt(w/2) > 8)";
      return DAFMM_EINVAL;
    }
  }
  // ---- root square of the quadrature cells (reading R2) ----
  double lox = INFINITY, hix = -INFINITY, loy = INFINITY, hiy = -INFINITY;
  for (int64_t i = 0; i < n; ++i) {
    double h = 0.5 * std::sqrt(P.w[i]);
    lox = std::min(lox, P.pts[2 * i] - h);
    hix = std::max(hix, P.pts[2 * i] + h);
    loy = std::min(loy, P.pts[2 * i + 1] - h);
    hiy = std::max(hiy, P.pts[2 * i + 1] + h);
  }
  P.W = std::max(hix - lox, hiy - loy);
  double cxr = 0.5 * (lox + hix), cyr = 0.5 * (loy + hiy);
  P.x0 = cxr - 0.5 * P.W;
  P.y0 = cyr - 0.5 * P.W;
  auto width = [&](int l) { return std::ldexp(P.W, -l); };
  // ---- adaptive tree (reading R2): a box is split while it holds more than
  // leaf_size points or is in the high-frequency regime (refinement rule 3), up to
  // max_level.  Points are binned once on the 2^20 lattice; a box at level l is that index
  // >> (20 - l), and tree order (Morton order of the lattice cell, then input index) makes
  // every box a contiguous range. ----
  constexpr int kMaxL = 20;
  if (opt.max_level > kMaxL) { err = "max_level must be <= 20"; return DAFMM_EINVAL; }
  std::vector<int64_t> fx(n), fy(n);
  {
    const double m = std::ldexp(1.0, kMaxL);
    const int64_t mx = ((int64_t)1 << kMaxL) - 1;
    for (int64_t i = 0; i < n; ++i) {
      int64_t a = (int64_t)std::floor(((P.pts[2 * i] - P.x0) / P.W) * m);
      int64_t b = (int64_t)std::floor(((P.pts[2 * i + 1] - P.y0) / P.W) * m);
      fx[i] = std::min<int64_t>(std::max<int64_t>(a, 0), mx);
      fy[i] = std::min<int64_t>(std::max<int64_t>(b, 0), mx);
    }
  }
  std::vector<uint64_t> mcode(n);
  for (int64_t i = 0; i < n; ++i) mcode[i] = morton(fx[i], fy[i]);
  P.perm.resize(n);
  std::iota(P.perm.begin(), P.perm.end(), 0);
  std::sort(P.perm.begin(), P.perm.end(), [&](int32_t a, int32_t b) {
    return mcode[a] != mcode[b] ? mcode[a] < mcode[b] : a < b;
  });
  // duplicate points (G is singular off the diagonal): they share a lattice cell
  {
    int64_t s0 = 0;
    while (s0 < n) {
      int64_t e = s0 + 1;
      while (e < n && mcode[P.perm[e]] == mcode[P.perm[s0]]) ++e;
      if (e - s0 > 1) {
        std::vector<std::pair<double, double>> xy;
        for (int64_t t = s0; t < e; ++t)
          xy.emplace_back(P.pts[2 * (size_t)P.perm[t]], P.pts[2 * (size_t)P.perm[t] + 1]);
        std::sort(xy.begin(), xy.end());
        for (size_t t = 1; t < xy.size(); ++t)
          if (xy[t] == xy[t - 1]) { err = "duplicate points"; return DAFMM_EINVAL; }
      }
      s0 = e;
    }
  }
  auto make_level = [&](int l) {
    Level lv;
    lv.level = l;
    lv.b = width(l);
    lv.kb = kappa * lv.b;
    lv.hfr = lv.kb * lv.kb > opt.T;
    if (lv.hfr) {  // R5 with reading R4: half-angle <= 1/(kappa w), w = b / sqrt(2) (w_reading 1: w = b)
      double x = opt.w_reading == 1 ? kPi * lv.kb : kPi * lv.kb / std::sqrt(2.0);
      int nc = 1;
      while (nc < x) nc *= 2;
      lv.ncones = nc;
    }
    return lv;
  };
  P.levels.clear();
  P.levels.push_back(make_level(0));
  P.levels[0].index[pack_key(0, 0)] = 0;
  P.levels[0].boxes.push_back({0, 0, 0, (int32_t)n, false});
  for (int l = 0;; ++l) {
    Level& lv = P.levels[l];
    Level next = make_level(l + 1);
    const int sh = kMaxL - (l + 1);
    for (Box& B : lv.boxes) {
      const int cnt = B.end - B.begin;
      const bool split = (cnt > leaf_size || lv.hfr) && l < opt.max_level;
      if (!split) {
        if (cnt > leaf_size) {
          err = "leaf_size not reachable within max_level";
          return DAFMM_EINVAL;
        }
        if (lv.hfr) {  // refinement rule 3: every leaf must be LFR (no directional leaf bases)
          err = "a high-frequency box cannot be split within max_level (refinement rule 3 needs LFR leaves)";
          return DAFMM_EINVAL;
        }
        B.leaf = true;
        continue;
      }
      int32_t t = B.begin;
      while (t < B.end) {  // children: contiguous runs of the level-(l+1) cell
        const int32_t o = P.perm[t];
        const int64_t cx = fx[o] >> sh, cy = fy[o] >> sh;
        int32_t e = t + 1;
        while (e < B.end && (fx[P.perm[e]] >> sh) == cx && (fy[P.perm[e]] >> sh) == cy) ++e;
        next.index[pack_key(cx, cy)] = (int)next.boxes.size();
        next.boxes.push_back({cx, cy, t, e, false});
        t = e;
      }
    }
    if (next.boxes.empty()) break;
    P.levels.push_back(std::move(next));
  }
  const int L = (int)P.levels.size() - 1;
  P.L = L;
  int leaf_levels = 0;
  for (const Level& lv : P.levels) {
    bool any = false;
    for (const Box& B : lv.boxes) any = any || B.leaf;
    leaf_levels += any ? 1 : 0;
  }
  P.multi_level_leaves = leaf_levels > 1;
  // level restriction (boxes sharing a boundary are at most one level apart) -- a
  // property of the input tree, reported (dafmm_stats.level_restricted), not required: the
  // near field folds the U / W / X lists in either way (R18)
  {
    std::vector<std::vector<int>> deep(L + 1);  // deepest leaf level in each box's subtree
    for (int l = L; l >= 0; --l) {
      const Level& lv = P.levels[l];
      deep[l].assign(lv.boxes.size(), l);
      if (l < L) {
        const Level& ch = P.levels[l + 1];
        for (size_t b = 0; b < lv.boxes.size(); ++b) {
          if (lv.boxes[b].leaf) continue;
          for (int c = 0; c < 4; ++c) {
            auto it = ch.index.find(pack_key(2 * lv.boxes[b].ix + (c & 1), 2 * lv.boxes[b].iy + (c >> 1)));
            if (it != ch.index.end()) deep[l][b] = std::max(deep[l][b], deep[l + 1][it->second]);
          }
        }
      }
    }
    P.level_restricted = true;
    for (int l = 0; l <= L && P.level_restricted; ++l) {
      const Level& lv = P.levels[l];
      for (const Box& B : lv.boxes) {
        if (!B.leaf) continue;
        for (int dx = -1; dx <= 1; ++dx)
          for (int dy = -1; dy <= 1; ++dy) {
            if (!dx && !dy) continue;
            auto it = lv.index.find(pack_key(B.ix + dx, B.iy + dy));
            if (B.ix + dx >= 0 && B.iy + dy >= 0 && it != lv.index.end() && deep[l][it->second] > l + 1)
              P.level_restricted = false;
          }
      }
    }
  }
  P.D.assign(n, zd(0.0, 0.0));
  if (opt.self_term == 1)
    for (int64_t i = 0; i < n; ++i) P.D[i] = self_term_disk(kappa, P.w[i]);
  if (opt.self_term == 2) {
    // equal weights share one value (the uniform configs): evaluate each distinct w once
    double wl = -1.0;
    zd dl(0.0, 0.0);
    for (int64_t i = 0; i < n; ++i) {
      if (P.w[i] != wl) {
        wl = P.w[i];
        dl = self_term_square(kappa, wl);
      }
      P.D[i] = dl;
    }
  }
  double t1 = now_s();
  P.t_tree = t1 - t0;

  // ---- lists ----
  for (int l = 0; l <= L; ++l) {
    Level& lv = P.levels[l];
    int nb = (int)lv.boxes.size();
    lv.N.assign(nb, {});
    int64_t reach = lv.hfr ? (int64_t)std::ceil(opt.w_reading == 1 ? lv.kb : lv.kb / 2.0) + 1 : 1;
    const double kb2 = lv.kb * lv.kb;
#pragma omp parallel for schedule(dynamic, 64)
    for (int b = 0; b < nb; ++b) {
      const Box& B = lv.boxes[b];
      for (int64_t dx = -reach; dx <= reach; ++dx)
        for (int64_t dy = -reach; dy <= reach; ++dy) {
          auto it = lv.index.find(pack_key(B.ix + dx, B.iy + dy));
          if (B.ix + dx < 0 || B.iy + dy < 0 || it == lv.index.end()) continue;
          int64_t d2 = dx * dx + dy * dy;
          // P:286 / P:302 (R4: centre distance < kappa w^2, w = b / sqrt(2); w_reading 1: w = b)
          bool nbr = lv.hfr ? (opt.w_reading == 1 ? (double)d2 < kb2 : 4.0 * (double)d2 < kb2) : (d2 < 4);
          if (nbr) lv.N[b].push_back(it->second);
        }
      std::sort(lv.N[b].begin(), lv.N[b].end());
    }
  }
  bool cone_ok = true;
  for (int l = 1; l <= L; ++l) {
    Level& lv = P.levels[l];
    const Level& pv = P.levels[l - 1];
    int nb = (int)lv.boxes.size();
    lv.IL.assign(nb, {});
    lv.ILdir.assign(nb, {});
#pragma omp parallel for schedule(dynamic, 64)
    for (int b = 0; b < nb; ++b) {
      const Box& B = lv.boxes[b];
      int pb = pv.index.at(pack_key(B.ix >> 1, B.iy >> 1));
      std::vector<int> il;
      for (int pn : pv.N[pb]) {
        const Box& PB = pv.boxes[pn];
        for (int c = 0; c < 4; ++c) {
          auto it = lv.index.find(pack_key(2 * PB.ix + (c & 1), 2 * PB.iy + (c >> 1)));
          if (it == lv.index.end()) continue;
          if (!std::binary_search(lv.N[b].begin(), lv.N[b].end(), it->second)) il.push_back(it->second);
        }
      }
      std::sort(il.begin(), il.end());
      lv.IL[b] = il;
      if (lv.hfr) {
        for (int a : il) {
          bool ok1, ok2;
          int k = cone_of(lv.ncones, lv.boxes[a].ix - B.ix, lv.boxes[a].iy - B.iy, ok1);
          int kp = cone_of(lv.ncones, B.ix - lv.boxes[a].ix, B.iy - lv.boxes[a].iy, ok2);
          if (!ok1 || !ok2 || kp != (k + lv.ncones / 2) % lv.ncones) {
#pragma omp atomic write
            cone_ok = false;
          }
          lv.ILdir[b].push_back({k, a, kp});
        }
        std::sort(lv.ILdir[b].begin(), lv.ILdir[b].end());
      }
    }
  }
  if (!cone_ok) { err = "box centre on a cone boundary"; return DAFMM_ESETUP; }
  // ---- near field of every leaf (coarse levels first): the source leaves C whose ancestor
  // at level min(l, l_C) neighbours B's (R6; the adaptive U, W and X lists folded
  // into the direct near field): leaves at a level m <= l neighbouring B's ancestor at level m
  // (B itself first: the only entry with i == j pairs), then the whole range of every non-leaf
  // neighbour of B at level l (all its leaves) ----
  P.leaves.clear();
  P.near.clear();
  for (int l = 0; l <= L; ++l) {
    const Level& lv = P.levels[l];
    for (size_t b = 0; b < lv.boxes.size(); ++b) {
      const Box& B = lv.boxes[b];
      if (!B.leaf) continue;
      std::vector<std::pair<int, int>> src = {{l, (int)b}};
      for (int m = l; m >= 0; --m) {
        const Level& mv = P.levels[m];
        const int bm = mv.index.at(pack_key(B.ix >> (l - m), B.iy >> (l - m)));
        for (int a : mv.N[bm])
          if (mv.boxes[a].leaf && !(m == l && a == (int)b)) src.push_back({m, a});
      }
      for (int a : lv.N[b])
        if (!lv.boxes[a].leaf) src.push_back({l, a});
      P.leaves.push_back({l, (int)b});
      P.near.push_back(std::move(src));
    }
  }
  // ---- active nodes, top-down ----
  for (int l = 0; l <= L; ++l) {
    Level& lv = P.levels[l];
    lv.node_of.assign(lv.boxes.size() * (size_t)lv.ncones, -1);
    if (l == 0) continue;
    const Level& pv = P.levels[l - 1];
    std::vector<char> parent_any(pv.boxes.size(), 0);
    for (auto& nd : pv.nodes) parent_any[nd.first] = 1;
    for (int b = 0; b < (int)lv.boxes.size(); ++b) {
      const Box& B = lv.boxes[b];
      int pb = pv.index.at(pack_key(B.ix >> 1, B.iy >> 1));
      if (lv.hfr) {
        std::vector<char> has(lv.ncones, 0);
        for (auto& e : lv.ILdir[b]) has[e[0]] = 1;
        for (int k = 0; k < lv.ncones; ++k) {
          bool need = has[k];
          if (l > 1 && pv.hfr)
            need = need || pv.node_id(pb, 2 * k) >= 0 || pv.node_id(pb, 2 * k + 1) >= 0;
          if (need) {
            lv.node_of[(size_t)b * lv.ncones + k] = (int)lv.nodes.size();
            lv.nodes.push_back({b, k});
          }
        }
      } else {
        bool need = !lv.IL[b].empty() || (l > 1 && parent_any[pb]);
        if (need) {
          lv.node_of[b] = (int)lv.nodes.size();
          lv.nodes.push_back({b, -1});
        }
      }
    }
  }
  double t2 = now_s();
  P.t_lists = t2 - t1;

  // ---- NCA pivots, bottom-up ----
  Ctx cx(P);
  P.piv.assign(L + 1, {});
  // F2: the ACAs run on the device unless the plan is host-only or opt.setup_device = 0
  std::unique_ptr<DeviceAca> dev_aca;
  if (opt.setup_device && !opt.host_only) {
    dev_aca.reset(new DeviceAca());
    int rc = dev_aca->init(P.pts.data(), P.w.data(), n, kappa, err);
    if (rc != DAFMM_OK) return rc;
  }
  int64_t total_entries = 0;
  for (int l = L; l >= 1; --l) {
    Level& lv = P.levels[l];
    P.piv[l].assign(lv.nodes.size(), NodePivots());
    const Level& pv = P.levels[l - 1];
    // child node ids of (box, cone) at level l+1 (C(B) / C(B, k))
    auto children = [&](const Level& at, int lvl, int box, int cone, std::vector<int>& out) {
      out.clear();
      const Level& ch = P.levels[lvl + 1];
      const Box& B = at.boxes[box];
      for (int c = 0; c < 4; ++c) {
        auto it = ch.index.find(pack_key(2 * B.ix + (c & 1), 2 * B.iy + (c >> 1)));
        if (it == ch.index.end()) continue;
        int nd = ch.node_id(it->second, ch.hfr ? cone / 2 : 0);
        if (nd >= 0) out.push_back(nd);
      }
    };
    // reading R17: nested-basis errors compound over the LFR levels of an adaptive tree, so
    // the ACA runs at nca_tol / 2 when leaves lie on several levels
    const double eps = P.multi_level_leaves ? 0.5 * nca_tol : nca_tol;
    auto is_leaf_node = [&](int nd) { return !lv.hfr && lv.boxes[lv.nodes[nd].first].leaf; };
    // leaf nodes first: a non-leaf node's search sets use the pivots of the leaves in its
    // interaction list (adaptive trees); two parallel sweeps
    int64_t level_entries = 0;
    // search sets t~^{B,i}, s~^{B,i}, t~^{B,o}, s~^{B,o} of node nd
    auto build_sets = [&](int nd, bool leafnode, std::vector<int32_t>& ti, std::vector<int32_t>& si,
                          std::vector<int32_t>& to, std::vector<int32_t>& so) {
      int b = lv.nodes[nd].first, k = lv.nodes[nd].second;
      // far list: IL(B) / IL(B,k); R7 substitute for an active HFR node with empty IL(B,k)
      std::vector<std::pair<int, int>> far;
      if (!lv.hfr) {
        for (int a : lv.IL[b]) far.push_back({a, -1});
      } else {
        for (auto& e : lv.ILdir[b])
          if (e[0] == k) far.push_back({e[1], e[2]});
        // R7: an active node with an empty IL(B,k) searches the children (matching child cones) of
        // its parent's IL in the two parent cones nesting in k; R7b (option hfr_parent_search):
        // every node with an HFR parent adds them to its own IL(B,k)
        if (far.empty() || (P.opt.hfr_parent_search && l > 1 && pv.hfr)) {
          const Box& B = lv.boxes[b];
          int pb = pv.index.at(pack_key(B.ix >> 1, B.iy >> 1));
          for (auto& e : pv.ILdir[pb]) {
            if (e[0] != 2 * k && e[0] != 2 * k + 1) continue;
            const Box& A = pv.boxes[e[1]];
            for (int c = 0; c < 4; ++c) {
              auto it = lv.index.find(pack_key(2 * A.ix + (c & 1), 2 * A.iy + (c >> 1)));
              if (it != lv.index.end()) far.push_back({it->second, e[2] / 2});
            }
          }
          std::sort(far.begin(), far.end());
          far.erase(std::unique(far.begin(), far.end()), far.end());
        }
      }
      if (leafnode) {
        const Box& B = lv.boxes[b];
        for (int32_t t = B.begin; t < B.end; ++t) ti.push_back(P.perm[t]);
        so = ti;
        auto add_box = [&](const Box& A) {
          for (int32_t t = A.begin; t < A.end; ++t) si.push_back(P.perm[t]);
        };
        for (auto& f : far) add_box(lv.boxes[f.first]);
        // reading R16: a leaf whose LFR parent has a leaf neighbour also searches IL(parent)
        if (l >= 2 && !pv.hfr) {
          int pb = pv.index.at(pack_key(B.ix >> 1, B.iy >> 1));
          bool leaf_nb = false;
          for (int a : pv.N[pb]) leaf_nb = leaf_nb || pv.boxes[a].leaf;
          if (leaf_nb)
            for (int a : pv.IL[pb]) add_box(pv.boxes[a]);
        }
        sorted_union(ti);
        sorted_union(so);
        sorted_union(si);
        to = si;
      } else {
        std::vector<int> kids;
        children(lv, l, b, k, kids);
        for (int c : kids) {
          const NodePivots& pc = P.piv[l + 1][c];
          ti.insert(ti.end(), pc.ti.begin(), pc.ti.end());
          so.insert(so.end(), pc.so.begin(), pc.so.end());
        }
        for (auto& f : far) {
          if (!lv.hfr && lv.boxes[f.first].leaf) {
            // a leaf in the interaction list has no children: its own pivots at this level
            const NodePivots& pa = P.piv[l][lv.node_id(f.first, 0)];
            si.insert(si.end(), pa.so.begin(), pa.so.end());
            to.insert(to.end(), pa.ti.begin(), pa.ti.end());
            continue;
          }
          children(lv, l, f.first, f.second, kids);
          for (int c : kids) {
            const NodePivots& pc = P.piv[l + 1][c];
            si.insert(si.end(), pc.so.begin(), pc.so.end());
            to.insert(to.end(), pc.ti.begin(), pc.ti.end());
          }
        }
        // reading R16 for non-leaf nodes: the points of IL(parent) when the LFR parent has a
        // leaf neighbour (the directions its own interaction list does not reach)
        if (!lv.hfr && l >= 2 && !pv.hfr) {
          const Box& B = lv.boxes[b];
          int pb = pv.index.at(pack_key(B.ix >> 1, B.iy >> 1));
          bool leaf_nb = false;
          for (int a : pv.N[pb]) leaf_nb = leaf_nb || pv.boxes[a].leaf;
          if (leaf_nb)
            for (int a : pv.IL[pb])
              for (int32_t t = pv.boxes[a].begin; t < pv.boxes[a].end; ++t) {
                si.push_back(P.perm[t]);
                to.push_back(P.perm[t]);
              }
        }
        sorted_union(ti);
        sorted_union(so);
        sorted_union(si);
        sorted_union(to);
      }
    };
    for (int sweep = 0; sweep < 2; ++sweep) {
      std::vector<int> sweep_nodes;
      for (int nd = 0; nd < (int)lv.nodes.size(); ++nd)
        if (is_leaf_node(nd) == (sweep == 0)) sweep_nodes.push_back(nd);
      if (sweep_nodes.empty()) continue;
      if (!dev_aca) {
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : level_entries)
        for (int t = 0; t < (int)sweep_nodes.size(); ++t) {
          const int nd = sweep_nodes[t];
          std::vector<int32_t> ti, si, to, so;
          build_sets(nd, sweep == 0, ti, si, to, so);
          NodePivots& np = P.piv[l][nd];
          int64_t ent = 0;
          aca(cx, ti, si, eps, np.ti, np.si, ent);
          if (P.opt.symmetric_pivots) {
            // reading R19: G is symmetric, and the outgoing search sets equal the incoming ones
            // with rows and columns swapped, so the incoming skeleton (t^{B,i}, s^{B,i}) also serves
            // as the outgoing one (s^{B,o} = t^{B,i}, t^{B,o} = s^{B,i}): one ACA per node
            np.so = np.ti;
            np.to = np.si;
          } else {
            aca(cx, to, so, eps, np.to, np.so, ent);
          }
          level_entries += ent;
        }
        continue;
      }
      // device ACA (F2): the search sets of every node of the sweep, packed into one index
      // array; one ACA problem per (node, direction), all run by one launch
      const int ns = (int)sweep_nodes.size();
      const double ts0 = now_s();
      std::vector<std::array<std::vector<int32_t>, 4>> sets(ns);
#pragma omp parallel for schedule(dynamic, 4)
      for (int t = 0; t < ns; ++t) {
        auto& S = sets[t];
        build_sets(sweep_nodes[t], sweep == 0, S[0], S[1], S[2], S[3]);
      }
      // leaf nodes: to = si, so = ti (stored once)
      const bool leafsweep = sweep == 0;
      std::vector<int64_t> off(4 * (size_t)ns + 1, 0);
      for (int t = 0; t < ns; ++t)
        for (int c = 0; c < 4; ++c) {
          const bool dup = leafsweep && c >= 2;
          off[4 * t + c + 1] = off[4 * t + c] + (dup ? 0 : (int64_t)sets[t][c].size());
        }
      std::vector<int32_t> idx(off.back());
#pragma omp parallel for schedule(dynamic, 16)
      for (int t = 0; t < ns; ++t)
        for (int c = 0; c < 4; ++c)
          if (!(leafsweep && c >= 2)) std::copy(sets[t][c].begin(), sets[t][c].end(), idx.begin() + off[4 * t + c]);
      auto set_off = [&](int t, int c) { return leafsweep && c >= 2 ? off[4 * t + (c == 2 ? 1 : 0)] : off[4 * t + c]; };
      auto set_len = [&](int t, int c) {
        return (int32_t)(leafsweep && c >= 2 ? sets[t][c == 2 ? 1 : 0].size() : sets[t][c].size());
      };
      const int dirs = P.opt.symmetric_pivots ? 1 : 2;
      std::vector<AcaProblem> probs((size_t)dirs * ns);
      for (int t = 0; t < ns; ++t) {
        probs[(size_t)dirs * t] = {set_off(t, 0), set_off(t, 1), set_len(t, 0), set_len(t, 1), 0, 0, 0, 0, 0};
        if (dirs == 2) probs[(size_t)dirs * t + 1] = {set_off(t, 2), set_off(t, 3), set_len(t, 2), set_len(t, 3), 0, 0, 0, 0, 0};
      }
      std::vector<int32_t> prow, pcol, rank;
      const double td = now_s();
      int rc = dev_aca->run(idx, probs, eps, prow, pcol, rank, level_entries, err);
      P.t_nca_device += now_s() - td;
      if (std::getenv("DAFMM_SETUP_TRACE"))
        std::fprintf(stderr, "nca level %d sweep %d: %d nodes, %zu set indices, sets %.3f s, device %.3f s\n", l,
                     sweep, ns, idx.size(), td - ts0, now_s() - td);
      if (rc != DAFMM_OK) return rc;
#pragma omp parallel for schedule(dynamic, 16)
      for (int t = 0; t < ns; ++t) {
        NodePivots& np = P.piv[l][sweep_nodes[t]];
        auto take = [&](const AcaProblem& pr, int r, std::vector<int32_t>& out_r, std::vector<int32_t>& out_c) {
          out_r.resize(r);
          out_c.resize(r);
          for (int q = 0; q < r; ++q) {
            out_r[q] = idx[pr.row_off + prow[pr.out_off + q]];
            out_c[q] = idx[pr.col_off + pcol[pr.out_off + q]];
          }
        };
        take(probs[(size_t)dirs * t], rank[(size_t)dirs * t], np.ti, np.si);
        if (dirs == 2) {
          take(probs[(size_t)dirs * t + 1], rank[(size_t)dirs * t + 1], np.to, np.so);
        } else {  // reading R19 (see the host path)
          np.so = np.ti;
          np.to = np.si;
        }
      }
    }
    total_entries += level_entries;
  }
  P.aca_entries = total_entries;
  double t3 = now_s();
  P.t_nca = t3 - t2;
  return DAFMM_OK;
}

// ============================================================================================
// Packing: node offsets, pivot coordinates, operator blocks (P:427-562 in the G-only form of
// DESIGN.md §Operators), and the per-pass work lists.
int pack_plan(const Plan& P, Packed& pk, std::string& err, size_t device_free) {
  const bool trace = std::getenv("DAFMM_SETUP_TRACE") != nullptr;
  double tr0 = now_s();
  auto mark = [&](const char* what) {
    if (trace) {
      const double t = now_s();
      std::fprintf(stderr, "pack: %-28s %.3f s\n", what, t - tr0);
      tr0 = t;
    }
  };
  double t0 = now_s();
  const int L = P.L;
  const int64_t n = P.n;
  Ctx cx(P);
  pk.perm = P.perm;

  pk.pts_t.resize(2 * n);
  pk.w_t.resize(n);
  pk.qk2_t.resize(n);
  pk.D_t.resize(n);
  for (int64_t t = 0; t < n; ++t) {
    int32_t o = P.perm[t];
    pk.pts_t[2 * t] = P.kappa * P.pts[2 * (size_t)o];  // kappa-scaled (the kernels evaluate H0 of z^2)
    pk.pts_t[2 * t + 1] = P.kappa * P.pts[2 * (size_t)o + 1];
    pk.w_t[t] = P.w[o];
    pk.qk2_t[t] = P.kappa * P.kappa * P.q[o];
    pk.D_t[t] = {P.D[o].real(), P.D[o].imag()};
  }
  // ---- node offsets ----
  std::vector<std::vector<int64_t>> moff(L + 1), loff(L + 1);
  int64_t nm = 0, nl = 0;
  for (int l = 1; l <= L; ++l) {
    size_t nn = P.levels[l].nodes.size();
    moff[l].resize(nn);
    loff[l].resize(nn);
    for (size_t nd = 0; nd < nn; ++nd) {
      moff[l][nd] = nm;
      loff[l][nd] = nl;
      nm += (int64_t)P.piv[l][nd].so.size();
      nl += (int64_t)P.piv[l][nd].ti.size();
    }
  }
  pk.n_mult = nm;
  pk.n_loc = nl;
  pk.so_xy.resize(2 * nm);
  pk.ti_xy.resize(2 * nl);
  for (int l = 1; l <= L; ++l)
    for (size_t nd = 0; nd < P.levels[l].nodes.size(); ++nd) {
      const NodePivots& np = P.piv[l][nd];
      for (size_t k = 0; k < np.so.size(); ++k) {
        pk.so_xy[2 * (moff[l][nd] + k)] = P.kappa * P.pts[2 * (size_t)np.so[k]];
        pk.so_xy[2 * (moff[l][nd] + k) + 1] = P.kappa * P.pts[2 * (size_t)np.so[k] + 1];
      }
      for (size_t k = 0; k < np.ti.size(); ++k) {
        pk.ti_xy[2 * (loff[l][nd] + k)] = P.kappa * P.pts[2 * (size_t)np.ti[k]];
        pk.ti_xy[2 * (loff[l][nd] + k) + 1] = P.kappa * P.pts[2 * (size_t)np.ti[k] + 1];
      }
    }
  // ---- operator block descriptors; blocks are filled in parallel afterwards ----
  // Translation items (P2M, M2M, L2L) store one block per item.  Column-major (default): entry
  // (row, col) at col * rows + row, the terms' blocks one after another, read one column per step
  // by translate_cm_kernel.  Row-major (DAFMM_OPS_ROWMAJOR): the terms' blocks side by side (row
  // stride = the item's total column count).  U (L2P) is column-major (one point per thread in combine).
  struct Job {
    int kind;  // 0: V (P2M), 1: T (M2M), 2: C (L2L), 3: U (L2P)
    int level, node, child;  // node at `level`, child node at level + 1
    int64_t off;             // block start
    int64_t stride;          // row stride (row-major item block); 0: column-major
    int col_start;           // first column of this term inside the item block
    int rows;                // the item's rows (column-major: column stride)
  };
  std::vector<Job> jobs;
  int64_t ops_len = 0;
  // column-major items (default): the translate kernel gives every output row a lane and reads
  // one coalesced column per step; DAFMM_OPS_ROWMAJOR=1 keeps the row-major items of the
  // warp-per-row kernels (A/B only)
  pk.ops_colmajor = std::getenv("DAFMM_OPS_ROWMAJOR") ? 0 : 1;
  auto add_job = [&](int kind, int l, int nd, int ch, int64_t len) {
    jobs.push_back({kind, l, nd, ch, ops_len, 0, 0, 0});
    ops_len += len;
    return jobs.back().off;
  };
  // one translation item: rows x (sum of term columns); terms = (child/parent node, src offset, cols)
  struct Term {
    int node, child;
    int64_t src_off;
    int cols;
  };
  auto add_item = [&](Packed::Batch& bt, int kind, int l, int64_t dst_off, int rows, const std::vector<Term>& terms) {
    int C = 0;
    for (const Term& t : terms) C += t.cols;
    const int64_t off = ops_len;
    ops_len += (int64_t)rows * C;
    bt.dst_off.push_back(dst_off);
    bt.dst_rows.push_back(rows);
    bt.item_mat_off.push_back(off);
    bt.item_cols.push_back(C);
    bt.term_ptr.push_back((int32_t)bt.src_off.size());
    int cs = 0;
    for (const Term& t : terms) {
      jobs.push_back({kind, l, t.node, t.child, off, pk.ops_colmajor ? 0 : C, cs, rows});
      bt.src_off.push_back(t.src_off);
      bt.src_cols.push_back(t.cols);
      cs += t.cols;
    }
  };
  auto child_nodes = [&](int l, int nd, std::vector<int>& out) {
    out.clear();
    const Level& lv = P.levels[l];
    const Level& ch = P.levels[l + 1];
    const Box& B = lv.boxes[lv.nodes[nd].first];
    int cone = lv.nodes[nd].second;
    for (int c = 0; c < 4; ++c) {
      auto it = ch.index.find(pack_key(2 * B.ix + (c & 1), 2 * B.iy + (c >> 1)));
      if (it == ch.index.end()) continue;
      int cn = ch.node_id(it->second, ch.hfr ? cone / 2 : 0);
      if (cn >= 0) out.push_back(cn);
    }
  };
  // P2M at every leaf node (the leaves of an adaptive tree sit on several levels)
  for (int l = 1; l <= L; ++l) {
    const Level& lv = P.levels[l];
    if (lv.hfr) continue;
    for (size_t nd = 0; nd < lv.nodes.size(); ++nd) {
      const Box& B = lv.boxes[lv.nodes[nd].first];
      int ro = (int)P.piv[l][nd].so.size();
      if (!B.leaf || ro == 0) continue;
      add_item(pk.p2m, 0, l, moff[l][nd], ro, {Term{(int)nd, -1, (int64_t)B.begin, B.end - B.begin}});
    }
  }
  pk.p2m.term_ptr.push_back((int32_t)pk.p2m.src_off.size());
  // M2M, fine to coarse
  std::vector<int> kids;
  pk.m2m.clear();
  for (int l = L - 1; l >= 1; --l) {
    Packed::Batch bt;
    const Level& lv = P.levels[l];
    for (size_t nd = 0; nd < lv.nodes.size(); ++nd) {
      int ro = (int)P.piv[l][nd].so.size();
      if (ro == 0 || (!lv.hfr && lv.boxes[lv.nodes[nd].first].leaf)) continue;
      child_nodes(l, (int)nd, kids);
      std::vector<Term> terms;
      for (int c : kids) {
        int rc = (int)P.piv[l + 1][c].so.size();
        if (rc > 0) terms.push_back({(int)nd, c, moff[l + 1][c], rc});
      }
      if (!terms.empty()) add_item(bt, 1, l, moff[l][nd], ro, terms);
    }
    bt.term_ptr.push_back((int32_t)bt.src_off.size());
    pk.m2m.push_back(std::move(bt));
  }
  // L2L, coarse to fine: items are the child nodes, terms the parent nodes listing them
  pk.l2l.clear();
  for (int l = 1; l <= L - 1; ++l) {
    const Level& lv = P.levels[l];
    const Level& ch = P.levels[l + 1];
    std::vector<std::vector<int>> incoming(ch.nodes.size());  // child -> parent nodes
    for (size_t nd = 0; nd < lv.nodes.size(); ++nd) {
      if (P.piv[l][nd].ti.empty()) continue;
      child_nodes(l, (int)nd, kids);
      for (int c : kids) incoming[c].push_back((int)nd);
    }
    Packed::Batch bt;
    for (size_t c = 0; c < ch.nodes.size(); ++c) {
      int rc = (int)P.piv[l + 1][c].ti.size();
      if (rc == 0 || incoming[c].empty()) continue;
      std::vector<Term> terms;
      for (int pn : incoming[c]) terms.push_back({pn, (int)c, loff[l][pn], (int)P.piv[l][pn].ti.size()});
      add_item(bt, 2, l, loff[l + 1][c], rc, terms);
    }
    bt.term_ptr.push_back((int32_t)bt.src_off.size());
    pk.l2l.push_back(std::move(bt));
  }
  mark("offsets, translation items");
  // M2L targets (all levels, one launch).  Each target's source nodes are
  // classified by the exact z-range of their pivot-point pairs and grouped into band-uniform
  // segments.
  struct M2LTarget {
    int level, node;
    std::vector<int> src;  // source node ids at `level`
  };
  std::vector<M2LTarget> tg;
  for (int l = 1; l <= L; ++l) {
    const Level& lv = P.levels[l];
    for (size_t nd = 0; nd < lv.nodes.size(); ++nd) {
      int ri = (int)P.piv[l][nd].ti.size();
      if (ri == 0) continue;
      int b = lv.nodes[nd].first, k = lv.nodes[nd].second;
      M2LTarget t{l, (int)nd, {}};
      auto add_src = [&](int sn) {
        if (!P.piv[l][sn].so.empty()) t.src.push_back(sn);
      };
      if (lv.hfr) {
        for (auto& e : lv.ILdir[b])
          if (e[0] == k) add_src(lv.node_id(e[1], e[2]));
      } else {
        for (int a : lv.IL[b]) add_src(lv.node_id(a, 0));
      }
      if (!t.src.empty()) tg.push_back(std::move(t));
    }
  }
  // symmetric stored M2L (R22): keep only the pairs the target owns (source id > target id at
  // the level; the interaction lists are symmetric, so every unordered pair is kept once)
  {
    int maxr = 0;
    int64_t half = 0;
    for (auto& t : tg) {
      const int ri = (int)P.piv[t.level][t.node].ti.size();
      maxr = std::max(maxr, ri);
      for (int sn : t.src)
        if (sn > t.node) half += (int64_t)ri * (int64_t)P.piv[t.level][sn].so.size();
    }
    const bool fits = device_free == 0 || (size_t)half * 16 <= device_free / 2;
    if (P.opt.m2l_store == 2) {
      if (!P.opt.symmetric_pivots) {
        err = "m2l_store=2 (blocks per node pair) needs symmetric_pivots=1 (one skeleton per node)";
        return DAFMM_EINVAL;
      }
      if (maxr > 128) {
        err = "m2l_store=2: a node has " + std::to_string(maxr) + " pivots (at most 128 supported)";
        return DAFMM_EINVAL;
      }
      if (device_free && (size_t)half * 16 > device_free) {
        err = "m2l_store=2: the M2L pair blocks need " + std::to_string(half * 16) + " bytes";
        return DAFMM_ENOMEM;
      }
    }
    pk.m2l_sym = (P.opt.m2l_store == 2 || (P.opt.m2l_store == -1 && P.opt.symmetric_pivots && maxr <= 128 && fits))
                     ? 1 : 0;
    if (pk.m2l_sym) {
      // incoming slots of every node: (owner target, position of the node's block in its stream)
      for (auto& t : tg) {
        std::vector<int> kept;
        for (int sn : t.src)
          if (sn > t.node) kept.push_back(sn);
        t.src.swap(kept);
      }
      std::vector<M2LTarget> keep;
      for (auto& t : tg)
        if (!t.src.empty()) keep.push_back(std::move(t));
      tg.swap(keep);
    }
  }
  mark("M2L target lists");
  std::vector<std::vector<int>> codes(tg.size());
#pragma omp parallel for schedule(dynamic, 16)
  for (size_t i = 0; i < tg.size(); ++i) {
    const NodePivots& pt = P.piv[tg[i].level][tg[i].node];
    codes[i].resize(tg[i].src.size());
    for (size_t e = 0; e < tg[i].src.size(); ++e) {
      const NodePivots& ps = P.piv[tg[i].level][tg[i].src[e]];
      double lo = INFINITY, hi = 0.0;
      for (int32_t a : pt.ti)
        for (int32_t c : ps.so) {
          double dx = P.pts[2 * (size_t)a] - P.pts[2 * (size_t)c];
          double dy = P.pts[2 * (size_t)a + 1] - P.pts[2 * (size_t)c + 1];
          double r2 = dx * dx + dy * dy;
          lo = std::min(lo, r2);
          hi = std::max(hi, r2);
        }
      codes[i][e] = choose_band(P.kappa * std::sqrt(lo), P.kappa * std::sqrt(hi), false);
    }
  }
  mark("M2L band classification");
  // targets in order of decreasing work (the persistent M2L kernel takes them in this order)
  std::vector<int64_t> tcost(tg.size(), 0);
  for (size_t i = 0; i < tg.size(); ++i) {
    int64_t so = 0;
    for (int sn : tg[i].src) so += (int64_t)P.piv[tg[i].level][sn].so.size();
    tcost[i] = so * (int64_t)P.piv[tg[i].level][tg[i].node].ti.size();
  }
  std::vector<size_t> torder(tg.size());
  std::iota(torder.begin(), torder.end(), 0);
  // the deepest level's targets first (their M2L needs only the leaves' multipoles and runs
  // beside M2M), each part in order of decreasing work
  std::stable_sort(torder.begin(), torder.end(), [&](size_t a, size_t b) {
    const bool la = tg[a].level == L, lb = tg[b].level == L;
    if (la != lb) return la;
    return tcost[a] > tcost[b];
  });
  pk.m2l_leaf_targets = 0;
  for (auto& t : tg) pk.m2l_leaf_targets += t.level == L ? 1 : 0;
  pk.m2l_src_ptr.push_back(0);
  pk.m2l_item_ptr.push_back(0);
  pk.m2l_stream_ptr.push_back(0);
  // R22: per level, (receiving node, slot of its first pivot in the owner's stream)
  std::vector<std::vector<std::pair<int, int64_t>>> in_lists((size_t)L + 1);
  int64_t stream_len = 0;
  for (size_t i : torder) {
    const int l = tg[i].level;
    const int ri = (int)P.piv[l][tg[i].node].ti.size();
    std::vector<int> order(tg[i].src.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return codes[i][a] < codes[i][b]; });
    const int64_t stream0 = stream_len;
    int prev = -1;
    int32_t cum = 0;  // offset in the target's source-pivot stream
    for (int e : order) {
      int sn = tg[i].src[e];
      int ro = (int)P.piv[l][sn].so.size();
      int code = codes[i][e];
      if (code != prev) {
        if (prev >= 0) pk.m2l_item_end.push_back(cum);
        pk.m2l_item_code.push_back(code);
        pk.m2l_item_begin.push_back(cum);
        prev = code;
      }
      pk.m2l_src_off.push_back(moff[l][sn]);
      pk.m2l_src_cnt.push_back(ro);
      if (pk.m2l_sym) in_lists[(size_t)l].push_back({sn, stream0 + cum});
      stream_len += ro;  // (the run's slots are written in parallel after the loop)
      cum += ro;
      const int64_t uses = pk.m2l_sym ? 2 : 1;  // a pair block serves both directions
      pk.m2l_entries += uses * (int64_t)ri * ro;
      pk.m2l_stored_entries += (int64_t)ri * ro;
      pk.m2l_band_entries[code] += uses * (int64_t)ri * ro;
      pk.m2l_pairs += uses;
    }
    pk.m2l_item_end.push_back(cum);
    pk.m2l_item_ptr.push_back((int32_t)pk.m2l_item_code.size());
    pk.m2l_loc_off.push_back(loff[l][tg[i].node]);
    pk.m2l_self_moff.push_back(moff[l][tg[i].node]);
    pk.m2l_rows.push_back(ri);
    pk.m2l_src_ptr.push_back((int32_t)pk.m2l_src_off.size());
    pk.m2l_stream_ptr.push_back(stream_len);
  }
  {  // the source streams: every run is the consecutive multipole slots of its source node
    pk.m2l_stream_idx.resize((size_t)stream_len);
    const size_t ntg = pk.m2l_rows.size();
#pragma omp parallel for schedule(dynamic, 64)
    for (size_t t = 0; t < ntg; ++t) {
      int64_t pos = pk.m2l_stream_ptr[t];
      for (int32_t e = pk.m2l_src_ptr[t]; e < pk.m2l_src_ptr[t + 1]; ++e)
        for (int32_t k = 0; k < pk.m2l_src_cnt[e]; ++k) pk.m2l_stream_idx[(size_t)pos++] = (int32_t)(pk.m2l_src_off[e] + k);
    }
  }
  if (pk.m2l_sym) {  // R22: the slot lists of every receiving node, level by level, by node id
    pk.m2l_in_ptr.assign(1, 0);
    for (int l = 1; l <= L; ++l) {
      auto& v = in_lists[(size_t)l];
      std::stable_sort(v.begin(), v.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      for (size_t a = 0; a < v.size();) {
        size_t b = a;
        while (b < v.size() && v[b].first == v[a].first) pk.m2l_in_off.push_back(v[b++].second);
        pk.m2l_in_lo.push_back(loff[l][v[a].first]);
        pk.m2l_in_rows.push_back((int32_t)P.piv[l][v[a].first].ti.size());
        pk.m2l_in_ptr.push_back((int32_t)pk.m2l_in_off.size());
        a = b;
      }
    }
  }
  mark("M2L streams and slot lists");
  // leaves (every level, coarse first): near field and L2P.  The near field of a leaf B at
  // level l is every source leaf C whose ancestor at level min(l, l_C) neighbours B's (P:750-755,
  // R6; the adaptive U, W and X lists folded into the direct near field):
  //   - leaves at a level m <= l neighbouring B's ancestor at level m (B itself first: the only
  //     entry with i == j pairs);
  //   - the whole range of every non-leaf neighbour of B at level l (all its leaves).
  auto bbox = [&](const Box& B, double* bb) {
    bb[0] = bb[1] = INFINITY;
    bb[2] = bb[3] = -INFINITY;
    for (int32_t t = B.begin; t < B.end; ++t) {
      int32_t o = P.perm[t];
      bb[0] = std::min(bb[0], P.pts[2 * (size_t)o]);
      bb[1] = std::min(bb[1], P.pts[2 * (size_t)o + 1]);
      bb[2] = std::max(bb[2], P.pts[2 * (size_t)o]);
      bb[3] = std::max(bb[3], P.pts[2 * (size_t)o + 1]);
    }
  };
  pk.near_ptr.push_back(0);
  pk.max_leaf = 0;
  // symmetric near field when every leaf has 32 or 64 points: the pairs between
  // two different leaves are evaluated once, by the leaf that comes first in tree order
  pk.p2p_sym = 1;
  for (int l = 0; l <= L; ++l)
    for (const Box& B : P.levels[l].boxes)
      if (B.leaf && B.end - B.begin != 64 && B.end - B.begin != 32) pk.p2p_sym = 0;
  struct SlotRange {
    int32_t r0, r1;
    int64_t slot;
  };
  std::vector<SlotRange> slot_ranges;
  pk.slot_total = 0;
  for (int l = 0; l <= L; ++l) {
    const Level& lv = P.levels[l];
    for (size_t b = 0; b < lv.boxes.size(); ++b) {
      const Box& B = lv.boxes[b];
      if (!B.leaf) continue;
      pk.leaf_begin.push_back(B.begin);
      pk.leaf_end.push_back(B.end);
      pk.max_leaf = std::max(pk.max_leaf, B.end - B.begin);
      const size_t li = pk.leaf_begin.size() - 1;  // leaves are packed in P.leaves order
      std::vector<const Box*> src;
      for (const auto& e : P.near[li]) src.push_back(&P.levels[e.first].boxes[e.second]);
      double pb[4], qb[4], zmax = 0.0;
      bbox(B, pb);
      int64_t pairs = 0;
      pk.leaf_slot_base.push_back(pk.slot_total);
      for (const Box* A : src) {
        pairs += (int64_t)(B.end - B.begin) * (A->end - A->begin);
        if (pk.p2p_sym && A != &B) {
          if (A->end <= B.begin) continue;  // evaluated by the earlier leaves' CTAs (slots)
          slot_ranges.push_back({A->begin, A->end, pk.slot_total});
          pk.slot_total += A->end - A->begin;
        }
        pk.near_begin.push_back(A->begin);
        pk.near_end.push_back(A->end);
        bbox(*A, qb);
        double dx = std::max(pb[2] - qb[0], qb[2] - pb[0]);
        double dy = std::max(pb[3] - qb[1], qb[3] - pb[1]);
        zmax = std::max(zmax, P.kappa * std::sqrt(dx * dx + dy * dy));
      }
      pairs -= (B.end - B.begin);
      pk.p2p_pairs += pairs;
      int band = zmax <= 7.0 ? kBandNear7 : zmax <= 8.0 ? kBandNear8 : zmax <= 12.0 ? kBandNear12 : kBandGeneric;
      pk.leaf_band.push_back(band);
      pk.p2p_band_entries[band] += pairs;
      pk.near_ptr.push_back((int32_t)pk.near_begin.size());
      int nd = lv.hfr ? -1 : lv.node_of[b];
      int ri = nd >= 0 ? (int)P.piv[l][nd].ti.size() : 0;
      if (ri > 0) {
        pk.leaf_loc_off.push_back(loff[l][nd]);
        pk.leaf_rank.push_back(ri);
        pk.leaf_U_off.push_back(add_job(3, l, nd, (int)b, (int64_t)(B.end - B.begin) * ri));
      } else {
        pk.leaf_loc_off.push_back(-1);
        pk.leaf_rank.push_back(0);
        pk.leaf_U_off.push_back(0);
      }
    }
  }
  // slots -> leaves: every slot range covers whole leaves (near ranges are boxes)
  pk.in_ptr.assign(1, 0);
  pk.in_off.clear();
  if (pk.p2p_sym) {
    const int nl = (int)pk.leaf_begin.size();
    std::vector<int> by_begin(nl);
    std::iota(by_begin.begin(), by_begin.end(), 0);
    std::sort(by_begin.begin(), by_begin.end(), [&](int a, int b) { return pk.leaf_begin[a] < pk.leaf_begin[b]; });
    std::vector<std::vector<int64_t>> in(nl);
    for (const SlotRange& sr : slot_ranges) {
      auto it = std::lower_bound(by_begin.begin(), by_begin.end(), sr.r0,
                                 [&](int li, int32_t v) { return pk.leaf_begin[li] < v; });
      for (; it != by_begin.end() && pk.leaf_begin[*it] < sr.r1; ++it)
        in[*it].push_back(sr.slot + (pk.leaf_begin[*it] - sr.r0));
    }
    for (int li = 0; li < nl; ++li) {
      for (int64_t o : in[li]) pk.in_off.push_back(o);
      pk.in_ptr.push_back((int32_t)pk.in_off.size());
    }
  }
  pk.ops_len = ops_len;
  mark("near lists, L2P");
  // ---- operator blocks on the device (F2): one group per (node, V~ or U~) sharing its cross
  // matrix; every job lists the caller indices of its columns (V~) or rows (U~) ----
  bool dev_ops = P.opt.setup_device && !P.opt.host_only;
  for (size_t jb = 0; dev_ops && jb < jobs.size(); ++jb) {
    const NodePivots& np = P.piv[jobs[jb].level][jobs[jb].node];
    if ((int)std::max(np.so.size(), np.ti.size()) > 64) dev_ops = false;  // kDeviceOpsMaxRank
  }
  if (dev_ops) {
    std::vector<size_t> order(jobs.size());
    std::iota(order.begin(), order.end(), 0);
    auto gkey = [&](const Job& J) { return std::make_tuple(J.level, J.node, J.kind >= 2 ? 1 : 0); };
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return gkey(jobs[a]) < gkey(jobs[b]); });
    auto push = [&](const std::vector<int32_t>& v) {
      const int64_t o = (int64_t)pk.opd_piv.size();
      pk.opd_piv.insert(pk.opd_piv.end(), v.begin(), v.end());
      return o;
    };
    for (size_t q = 0; q < order.size();) {
      const Job& J0 = jobs[order[q]];
      const int type = J0.kind >= 2 ? 1 : 0;
      const NodePivots& np = P.piv[J0.level][J0.node];
      const std::vector<int32_t>& A = type == 0 ? np.to : np.ti;
      const std::vector<int32_t>& B = type == 0 ? np.so : np.si;
      std::array<int32_t, 6> g = {(int32_t)push(A), (int32_t)push(B), (int32_t)A.size(), type,
                                  (int32_t)pk.opd_jobs.size(), 0};
      size_t e = q;
      for (; e < order.size() && gkey(jobs[order[e]]) == gkey(J0); ++e) {
        const Job& J = jobs[order[e]];
        std::vector<int32_t> src;
        int rows = J.rows;
        if (J.kind == 0 || J.kind == 3) {  // the leaf's points
          const Level& jl = P.levels[J.level];
          const Box& Bx = J.kind == 0 ? jl.boxes[jl.nodes[J.node].first] : jl.boxes[J.child];
          for (int32_t t = Bx.begin; t < Bx.end; ++t) src.push_back(P.perm[t]);
          if (J.kind == 3) rows = Bx.end - Bx.begin;
        } else if (J.kind == 1) {
          src = P.piv[J.level + 1][J.child].so;
        } else {
          src = P.piv[J.level + 1][J.child].ti;
        }
        const int64_t so = push(src);
        pk.opd_jobs.push_back({J.off, rows, J.col_start, (int32_t)J.stride, 0, so, (int32_t)src.size(), 0});
      }
      g[5] = (int32_t)pk.opd_jobs.size();
      if (g[2] > 0) pk.opd_groups.push_back(g);
      q = e;
    }
    pk.ops_on_device = 1;
    return DAFMM_OK;
  }
  mark("device operator jobs");
  // ---- operator blocks (column-major), in parallel ----
  try {
    pk.ops.assign((size_t)ops_len, cplx{0.0, 0.0});
  } catch (...) {
    err = "host allocation of operator blocks failed";
    return DAFMM_ENOMEM;
  }
  int fail = 0;
#pragma omp parallel for schedule(dynamic, 4)
  for (size_t jb = 0; jb < jobs.size(); ++jb) {
    const Job& J = jobs[jb];
    const NodePivots& np = P.piv[J.level][J.node];
    cplx* out = pk.ops.data() + J.off;
    if (J.kind == 0 || J.kind == 1) {
      // V~ = H(to, so)^{-1} H(to, s) : rows = so, cols = s (leaf points or child's so)
      int r = (int)np.so.size();
      std::vector<int32_t> cols;
      if (J.kind == 0) {
        const Level& jl = P.levels[J.level];
        const Box& B = jl.boxes[jl.nodes[J.node].first];
        for (int32_t t = B.begin; t < B.end; ++t) cols.push_back(P.perm[t]);
      } else {
        cols = P.piv[J.level + 1][J.child].so;
      }
      std::vector<zd> M((size_t)r * r);
      for (int a = 0; a < r; ++a)
        for (int c = 0; c < r; ++c) M[(size_t)a * r + c] = cx.H(np.to[a], np.so[c]);
      LU lu;
      if (!lu.factor(M, r)) {
#pragma omp atomic write
        fail = 1;
        continue;
      }
      std::vector<zd> rhs(r);
      for (size_t c = 0; c < cols.size(); ++c) {
        for (int a = 0; a < r; ++a) rhs[a] = cx.H(np.to[a], cols[c]);
        lu.solve(rhs.data());
        for (int a = 0; a < r; ++a) {
          const size_t at = J.stride > 0 ? (size_t)a * J.stride + J.col_start + c
                                         : (size_t)(J.col_start + c) * J.rows + a;
          out[at] = {rhs[a].real(), rhs[a].imag()};
        }
      }
    } else {
      // U~ = H(t, si) H(ti, si)^{-1}: rows = t (leaf points or child's ti), cols = ti.
      // X M = B  <=>  M^T X^T = B^T : factor M^T, solve one row of X per right-hand side.
      int r = (int)np.ti.size();
      std::vector<int32_t> rows;
      if (J.kind == 3) {
        const Box& B = P.levels[J.level].boxes[J.child];
        for (int32_t t = B.begin; t < B.end; ++t) rows.push_back(P.perm[t]);
      } else {
        rows = P.piv[J.level + 1][J.child].ti;
      }
      std::vector<zd> MT((size_t)r * r);
      for (int a = 0; a < r; ++a)
        for (int c = 0; c < r; ++c) MT[(size_t)c * r + a] = cx.H(np.ti[a], np.si[c]);
      LU lu;
      if (!lu.factor(MT, r)) {
#pragma omp atomic write
        fail = 1;
        continue;
      }
      std::vector<zd> rhs(r);
      int nr = (int)rows.size();
      for (int a = 0; a < nr; ++a) {
        for (int c = 0; c < r; ++c) rhs[c] = cx.H(rows[a], np.si[c]);
        lu.solve(rhs.data());
        for (int c = 0; c < r; ++c) {
          const size_t at = J.kind == 3      ? (size_t)c * nr + a
                            : J.stride > 0 ? (size_t)a * J.stride + J.col_start + c
                                           : (size_t)(J.col_start + c) * J.rows + a;
          out[at] = {rhs[c].real(), rhs[c].imag()};
        }
      }
    }
  }
  if (fail) {
    err = "singular NCA cross matrix";
    return DAFMM_ESETUP;
  }
  (void)t0;
  return DAFMM_OK;
}

// ============================================================================================
// Plan export (.npy files) for the oracle.
namespace {
template <typename T>
bool write_npy(const std::string& path, const char* descr, const std::vector<T>& data, std::vector<int64_t> shape) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) return false;
  std::string sh = "(";
  for (size_t i = 0; i < shape.size(); ++i) sh += std::to_string(shape[i]) + (shape.size() == 1 ? "," : (i + 1 < shape.size() ? ", " : ""));
  sh += ")";
  std::string hdr = std::string("{'descr': '") + descr + "', 'fortran_order': False, 'shape': " + sh + ", }";
  size_t total = 10 + hdr.size() + 1;
  size_t pad = (64 - total % 64) % 64;
  hdr += std::string(pad, ' ') + "\n";
  unsigned char magic[8] = {0x93, 'N', 'U', 'M', 'P', 'Y', 1, 0};
  uint16_t hl = (uint16_t)hdr.size();
  std::fwrite(magic, 1, 8, f);
  std::fwrite(&hl, 2, 1, f);
  std::fwrite(hdr.data(), 1, hdr.size(), f);
  if (!data.empty()) std::fwrite(data.data(), sizeof(T), data.size(), f);
  std::fclose(f);
  return true;
}
}  // namespace

int export_plan(const Plan& P, const std::string& dir, std::string& err) {
  for (size_t i = 1; i <= dir.size(); ++i)  // mkdir -p
    if (i == dir.size() || dir[i] == '/') mkdir(dir.substr(0, i).c_str(), 0755);
  bool ok = true;
  std::vector<double> meta = {(double)P.n, (double)P.L, P.W, P.x0, P.y0, P.kappa, P.opt.T, P.nca_tol,
                              (double)P.opt.hfr_parent_search, (double)P.opt.w_reading};
  ok &= write_npy(dir + "/meta.npy", "<f8", meta, {(int64_t)meta.size()});
  std::vector<int64_t> perm(P.perm.begin(), P.perm.end());
  ok &= write_npy(dir + "/perm.npy", "<i8", perm, {(int64_t)perm.size()});
  {  // self terms D_i (caller order), complex128
    std::vector<double> d(2 * (size_t)P.n);
    for (int64_t i = 0; i < P.n; ++i) {
      d[2 * i] = P.D[i].real();
      d[2 * i + 1] = P.D[i].imag();
    }
    ok &= write_npy(dir + "/self.npy", "<c16", d, {(int64_t)P.n});
  }
  // leaves (level, box) and their near-field source boxes (level, box)
  {
    std::vector<int64_t> leaves, ptr = {0}, src;
    for (size_t i = 0; i < P.leaves.size(); ++i) {
      leaves.push_back(P.leaves[i].first);
      leaves.push_back(P.leaves[i].second);
      for (auto& e : P.near[i]) {
        src.push_back(e.first);
        src.push_back(e.second);
      }
      ptr.push_back((int64_t)src.size() / 2);
    }
    ok &= write_npy(dir + "/leaves.npy", "<i8", leaves, {(int64_t)P.leaves.size(), 2});
    ok &= write_npy(dir + "/near_ptr.npy", "<i8", ptr, {(int64_t)ptr.size()});
    ok &= write_npy(dir + "/near_src.npy", "<i8", src, {(int64_t)src.size() / 2, 2});
  }
  for (int l = 0; l <= P.L; ++l) {
    const Level& lv = P.levels[l];
    std::string pre = dir + "/l" + std::to_string(l) + "_";
    std::vector<int64_t> boxes, leaf;
    for (auto& b : lv.boxes) { boxes.push_back(b.ix); boxes.push_back(b.iy); leaf.push_back(b.leaf ? 1 : 0); }
    ok &= write_npy(pre + "boxes.npy", "<i8", boxes, {(int64_t)lv.boxes.size(), 2});
    ok &= write_npy(pre + "leaf.npy", "<i8", leaf, {(int64_t)lv.boxes.size()});
    std::vector<int64_t> info = {lv.hfr ? 1 : 0, lv.ncones};
    ok &= write_npy(pre + "info.npy", "<i8", info, {2});
    auto csr = [&](const std::vector<std::vector<int>>& lists, const std::string& name) {
      std::vector<int64_t> ptr = {0}, idx;
      for (auto& v : lists) {
        for (int a : v) idx.push_back(a);
        ptr.push_back((int64_t)idx.size());
      }
      ok &= write_npy(pre + name + "_ptr.npy", "<i8", ptr, {(int64_t)ptr.size()});
      ok &= write_npy(pre + name + "_idx.npy", "<i8", idx, {(int64_t)idx.size()});
    };
    csr(lv.N, "N");
    if (l >= 1) {
      csr(lv.IL, "IL");
      std::vector<int64_t> dir4;
      for (size_t b = 0; b < lv.ILdir.size(); ++b)
        for (auto& e : lv.ILdir[b]) { dir4.push_back((int64_t)b); dir4.push_back(e[0]); dir4.push_back(e[1]); dir4.push_back(e[2]); }
      ok &= write_npy(pre + "ILdir.npy", "<i8", dir4, {(int64_t)dir4.size() / 4, 4});
      std::vector<int64_t> nodes;
      for (auto& nd : lv.nodes) { nodes.push_back(nd.first); nodes.push_back(nd.second); }
      ok &= write_npy(pre + "nodes.npy", "<i8", nodes, {(int64_t)lv.nodes.size(), 2});
      const char* names[4] = {"ti", "si", "to", "so"};
      for (int s = 0; s < 4; ++s) {
        std::vector<int64_t> ptr = {0}, idx;
        for (auto& np : P.piv[l]) {
          const std::vector<int32_t>& v = s == 0 ? np.ti : s == 1 ? np.si : s == 2 ? np.to : np.so;
          for (int32_t a : v) idx.push_back(a);
          ptr.push_back((int64_t)idx.size());
        }
        ok &= write_npy(pre + names[s] + "_ptr.npy", "<i8", ptr, {(int64_t)ptr.size()});
        ok &= write_npy(pre + names[s] + "_idx.npy", "<i8", idx, {(int64_t)idx.size()});
      }
    }
  }
  if (!ok) { err = "could not write plan files to " + dir; return DAFMM_EINVAL; }
  return DAFMM_OK;
}

}  // namespace dafmm
