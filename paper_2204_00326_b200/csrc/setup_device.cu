// Device-side NCA setup: the partially pivoted ACAs of the nested cross
// approximation (stopping rule of [Rjasanow 2002] cited at P:816; reading R10) for
// every node of one tree level at once, one CTA per ACA problem.
//
// The host builds the search sets exactly as before (setup.cpp: they depend on the
// children's pivots, so the levels run bottom-up); this file only replaces the inner loop, the
// ACA itself, which evaluated ~3.4e9 kernel entries on the host at config 4.  Every ACA
// problem is an m x n block K[rows, cols], K_ij = G(x_i, x_j) w_j (reading R9); the constant
// i/4 of G is dropped (every test of the ACA is invariant under a uniform scale of the block).
//
// Mapping: persistent CTAs of 256 threads take problems from a ticket counter (the host
// orders them by decreasing m + n).  Each CTA owns a global-memory scratch slot holding the
// residual terms V (k x n rows) and U (k x m columns) of its current problem plus the used
// flags; they are written once and re-read every step, so they stay in L2.  A step: evaluate
// the residual row i (H0 on the fly, minus the earlier terms) and its first argmax over unused
// columns (block reduction, ties to the lower position), the residual column jm, then the
// 2k + 2 dot products of the incremental Frobenius norm (one warp per term), and the next row.
// All reductions run in a fixed order, so the pivots are deterministic for a given launch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <string>
#include <vector>

#include "dense.cuh"
#include "setup_device.h"

namespace dafmm {

namespace {

constexpr int kAcaThreads = 256;
constexpr int kAcaWarps = kAcaThreads / 32;
constexpr int kAcaMaxRank = 200;  // R10 rank cap
// R10: a residual row at or below this multiple of its largest original entry is a zero row
constexpr double kZeroRowRtol = 1e3 * 2.220446049250313e-16;

bool ck(cudaError_t e, std::string& err, const char* what) {
  if (e == cudaSuccess) return true;
  err = std::string(what) + ": " + cudaGetErrorString(e);
  return false;
}

__device__ __forceinline__ double cabs2(double2 a) { return fma(a.x, a.x, a.y * a.y); }

// K'(i, j) = H0(kappa |x_i - x_j|) w_j with kappa-scaled coordinates
__device__ __forceinline__ double2 kentry(double2 xi, double2 xj, double wj, const PolyTable& T) {
  const double dx = xi.x - xj.x, dy = xi.y - xj.y;
  const double d2 = fma(dx, dx, dy * dy);
  double hr, hi;
  h0_generic_vec<1>(&d2, &hr, &hi, T);
  return make_double2(hr * wj, hi * wj);
}

// Block-wide (value, position) maximum: larger value wins, ties go to the lower position;
// positions < 0 mean "none".  Also reduces a plain maximum `aux`.  All threads get the result.
struct ArgMax {
  double v;
  int p;
};
__device__ __forceinline__ ArgMax better(ArgMax a, ArgMax b) {
  if (b.p < 0) return a;
  if (a.p < 0) return b;
  if (b.v > a.v || (b.v == a.v && b.p < a.p)) return b;
  return a;
}
__device__ ArgMax block_argmax(ArgMax a, double& aux, ArgMax* s_am, double* s_aux) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax b{__shfl_xor_sync(0xffffffffu, a.v, o), __shfl_xor_sync(0xffffffffu, a.p, o)};
    a = better(a, b);
    aux = fmax(aux, __shfl_xor_sync(0xffffffffu, aux, o));
  }
  __syncthreads();  // the previous use of s_am / s_aux is finished
  if (lane == 0) {
    s_am[wid] = a;
    s_aux[wid] = aux;
  }
  __syncthreads();
  ArgMax r = s_am[0];
  double x = s_aux[0];
  for (int w = 1; w < kAcaWarps; ++w) {
    r = better(r, s_am[w]);
    x = fmax(x, s_aux[w]);
  }
  aux = x;
  return r;
}

__global__ void __launch_bounds__(kAcaThreads) aca_kernel(const AcaProblem* __restrict__ probs, int nprob,
                                                          int* __restrict__ ticket, const int32_t* __restrict__ idx,
                                                          const double2* __restrict__ pts,
                                                          const double* __restrict__ w,
                                                          const double* __restrict__ qrow, double k4, double eps,
                                                          double2* __restrict__ scratch, int64_t stride,
                                                          int32_t* __restrict__ piv_row, int32_t* __restrict__ piv_col,
                                                          int32_t* __restrict__ rank_out,
                                                          unsigned long long* __restrict__ entries) {
  __shared__ PolyTable T;
  __shared__ double2 s_coef[kAcaMaxRank];
  __shared__ double2 s_du[kAcaMaxRank + 1], s_dv[kAcaMaxRank + 1];
  __shared__ ArgMax s_am[kAcaWarps];
  __shared__ double s_aux[kAcaWarps];
  __shared__ int s_prob, s_flag;
  __shared__ double s_norm2;
  load_poly_table(T);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double2* const V = scratch + (int64_t)blockIdx.x * stride;
  unsigned long long ent = 0;
  for (;;) {
    if (tid == 0) s_prob = atomicAdd(ticket, 1);
    __syncthreads();
    const int p = s_prob;
    if (p >= nprob) break;
    const AcaProblem P = probs[p];
    const int m = P.m, n = P.n;
    const int mode = P.mode;
    const int cap = min(min(m, n), P.cap > 0 ? min(P.cap, kAcaMaxRank) : kAcaMaxRank);
    const int32_t* R = idx + P.row_off;
    const int32_t* C = idx + P.col_off;
    double2* const U = V + (int64_t)cap * n;
    unsigned char* const used_r = reinterpret_cast<unsigned char*>(U + (int64_t)cap * m);
    unsigned char* const used_c = used_r + m;
    for (int t = tid; t < m + n; t += kAcaThreads) used_r[t] = 0;
    if (tid == 0) s_norm2 = 0.0;
    __syncthreads();
    int i = mode == 1 ? P.first_row : 0, k = 0;
    while (k < cap) {
      // ---- residual row i: V[k][j] = K(i, j) - sum_l U[l][i] V[l][j] ----
      for (int l = tid; l < k; l += kAcaThreads) s_coef[l] = U[(int64_t)l * m + i];
      __syncthreads();
      const double2 xi = pts[R[i]];
      const double qi = mode == 1 ? qrow[R[i]] : 1.0;
      double row_max = 0.0;
      ArgMax best{-1.0, -1};
      double2* const Vk = V + (int64_t)k * n;
      for (int j = tid; j < n; j += kAcaThreads) {
        const int cj = C[j];
        double2 val = kentry(xi, pts[cj], qi * w[cj], T);
        row_max = fmax(row_max, cabs2(val));
        for (int l = 0; l < k; ++l) {
          const double2 ul = s_coef[l], vl = V[(int64_t)l * n + j];
          val.x -= ul.x * vl.x - ul.y * vl.y;
          val.y -= ul.x * vl.y + ul.y * vl.x;
        }
        Vk[j] = val;
        if (!used_c[j]) best = better(best, ArgMax{cabs2(val), j});
      }
      if (tid == 0) ent += n;
      best = block_argmax(best, row_max, s_am, s_aux);  // squared magnitudes
      if (tid == 0) used_r[i] = 1;
      const int jm = best.p;
      if (!(jm >= 0 && sqrt(best.v) > kZeroRowRtol * sqrt(row_max))) {
        if (mode == 1) break;  // HR2: the block is exhausted at this rank
        // zero residual row: the next unused row (smallest position), if any
        __syncthreads();
        ArgMax nx{-1.0, -1};
        for (int t = tid; t < m; t += kAcaThreads)
          if (!used_r[t]) { nx = better(nx, ArgMax{(double)-t, t}); }
        double dummy = 0.0;
        nx = block_argmax(nx, dummy, s_am, s_aux);
        if (nx.p < 0) break;
        i = nx.p;
        continue;
      }
      // ---- v = r / r[jm]; residual column jm: U[k][t] = K(t, jm) - sum_l V[l][jm] U[l][t] ----
      const double2 piv = Vk[jm];
      const double pd = cabs2(piv);
      const double2 inv = make_double2(piv.x / pd, -piv.y / pd);
      __syncthreads();  // every thread has read the pivot before it is normalised
      for (int j = tid; j < n; j += kAcaThreads) {
        const double2 r = Vk[j];
        Vk[j] = make_double2(r.x * inv.x - r.y * inv.y, r.x * inv.y + r.y * inv.x);
      }
      for (int l = tid; l < k; l += kAcaThreads) s_coef[l] = V[(int64_t)l * n + jm];
      __syncthreads();
      const int cjm = C[jm];
      const double2 xj = pts[cjm];
      const double wj = w[cjm];
      double2* const Uk = U + (int64_t)k * m;
      double col_max = 0.0;
      for (int t = tid; t < m; t += kAcaThreads) {
        double2 val = kentry(pts[R[t]], xj, (mode == 1 ? qrow[R[t]] : 1.0) * wj, T);
        col_max = fmax(col_max, cabs2(val));
        for (int l = 0; l < k; ++l) {
          const double2 vl = s_coef[l], ul = U[(int64_t)l * m + t];
          val.x -= vl.x * ul.x - vl.y * ul.y;
          val.y -= vl.x * ul.y + vl.y * ul.x;
        }
        Uk[t] = val;
      }
      if (tid == 0) ent += m;
      __syncthreads();
      if (mode == 1) {  // HR2: fixed rank, no tolerance test
        if (tid == 0) {
          piv_row[P.out_off + k] = i;
          piv_col[P.out_off + k] = jm;
          used_c[jm] = 1;
        }
        ++k;
        ArgMax nx{-1.0, -1};
        for (int t = tid; t < m; t += kAcaThreads)
          if (!used_r[t]) nx = better(nx, ArgMax{cabs2(Uk[t]), t});
        nx = block_argmax(nx, col_max, s_am, s_aux);
        if (nx.p < 0 || !(sqrt(nx.v) > kZeroRowRtol * sqrt(col_max))) break;
        i = nx.p;
        continue;
      }
      // ---- incremental ||S_k||_F^2: du_l = <U_l, u>, dv_l = <V_l, v> (one warp per term l),
      // and |u|^2, |v|^2 (term l = k) ----
      for (int l = wid; l <= k; l += kAcaWarps) {
        const double2* Ul = U + (int64_t)l * m;
        const double2* Vl = V + (int64_t)l * n;
        double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
        for (int t = lane; t < m; t += 32) {
          const double2 a = Ul[t], b = Uk[t];
          ar += a.x * b.x + a.y * b.y;  // conj(a) b
          ai += a.x * b.y - a.y * b.x;
        }
        for (int j = lane; j < n; j += 32) {
          const double2 a = Vl[j], b = Vk[j];
          br += a.x * b.x + a.y * b.y;
          bi += a.x * b.y - a.y * b.x;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          ar += __shfl_xor_sync(0xffffffffu, ar, o);
          ai += __shfl_xor_sync(0xffffffffu, ai, o);
          br += __shfl_xor_sync(0xffffffffu, br, o);
          bi += __shfl_xor_sync(0xffffffffu, bi, o);
        }
        if (lane == 0) {
          s_du[l] = make_double2(ar, ai);
          s_dv[l] = make_double2(br, bi);
        }
      }
      __syncthreads();
      if (tid == 0) {
        double cross = 0.0;
        for (int l = 0; l < k; ++l) {
          const double2 a = s_du[l], b = s_dv[l];
          cross += 2.0 * (a.x * b.x - a.y * b.y);  // 2 Re(du dv)
        }
        const double nu2 = s_du[k].x, nv2 = s_dv[k].x;
        const double norm2 = s_norm2 + cross + nu2 * nv2;
        s_norm2 = norm2;
        const bool stop = k > 0 && sqrt(nu2 * nv2) <= eps * sqrt(norm2);
        s_flag = stop ? 1 : 0;
        if (!stop) {
          piv_row[P.out_off + k] = i;
          piv_col[P.out_off + k] = jm;
          used_c[jm] = 1;
        }
      }
      __syncthreads();
      if (s_flag) break;
      ++k;
      // ---- next row: argmax |u| over unused rows ----
      ArgMax nx{-1.0, -1};
      for (int t = tid; t < m; t += kAcaThreads)
        if (!used_r[t]) nx = better(nx, ArgMax{cabs2(Uk[t]), t});
      double dummy = 0.0;
      nx = block_argmax(nx, dummy, s_am, s_aux);
      if (nx.p < 0) break;  // every row used
      i = nx.p;
    }
    if (tid == 0) rank_out[p] = k;
    if (mode == 1 && P.u_out) {
      // the ACA factors of A's block (its entries are (i kappa^2 / 4) q_i H0 w_j: the ACA ran on
      // q_i H0 w_j, so u_l takes the constant i k4, k4 = kappa^2 / 4), balanced: u_l / s_l and
      // v_l s_l with s_l = sqrt(|u_l| / |v_l|)
      __syncthreads();
      for (int l = wid; l < k; l += kAcaWarps) {
        double su = 0.0, sv = 0.0;
        for (int t = lane; t < m; t += 32) su += cabs2(U[(int64_t)l * m + t]);
        for (int j = lane; j < n; j += 32) sv += cabs2(V[(int64_t)l * n + j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          su += __shfl_xor_sync(0xffffffffu, su, o);
          sv += __shfl_xor_sync(0xffffffffu, sv, o);
        }
        if (lane == 0) s_coef[l].x = (su > 0.0 && sv > 0.0) ? sqrt(sqrt(su) / sqrt(sv)) : 1.0;
      }
      __syncthreads();
      const int ldo = P.ldo;
      for (int64_t e = tid; e < (int64_t)m * ldo; e += kAcaThreads) {
        const int t = (int)(e / ldo), l = (int)(e % ldo);
        double2 v = make_double2(0.0, 0.0);
        if (l < k) {
          const double2 u = U[(int64_t)l * m + t];
          const double c = k4 / s_coef[l].x;
          v = make_double2(-u.y * c, u.x * c);
        }
        P.u_out[(P.row_off + t) * ldo + l] = v;
      }
      for (int64_t e = tid; e < (int64_t)n * ldo; e += kAcaThreads) {
        const int j = (int)(e / ldo), l = (int)(e % ldo);
        double2 v = make_double2(0.0, 0.0);
        if (l < k) {
          const double2 w = V[(int64_t)l * n + j];
          v = make_double2(w.x * s_coef[l].x, w.y * s_coef[l].x);
        }
        P.v_out[(P.col_off + j) * ldo + l] = v;
      }
    }
    __syncthreads();
  }
  if (tid == 0) atomicAdd(entries, ent);
}


// ---- translation operators (one CTA per group; the cross matrix LU shared by its jobs) ----
__device__ __forceinline__ double2 hentry(double2 a, double2 b, const PolyTable& T) {
  const double dx = a.x - b.x, dy = a.y - b.y;
  const double d2 = fma(dx, dx, dy * dy);
  double hr, hi;
  h0_generic_vec<1>(&d2, &hr, &hi, T);
  return make_double2(hr, hi);
}

__global__ void __launch_bounds__(128) ops_form_kernel(const OpGroup* __restrict__ groups,
                                                       const OpJob* __restrict__ jobs,
                                                       const int32_t* __restrict__ piv,
                                                       const double2* __restrict__ pts, double2* __restrict__ ops,
                                                       int* status) {
  __shared__ PolyTable T;
  extern __shared__ double2 M[];  // r x r, column-major
  __shared__ int s_perm[kDeviceOpsMaxRank];
  __shared__ int s_piv;
  load_poly_table(T);
  const OpGroup G = groups[blockIdx.x];
  const int r = G.r;
  const int32_t* A = piv + G.a_off;
  const int32_t* B = piv + G.b_off;
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) M[e] = hentry(pts[A[e % r]], pts[B[e / r]], T);
  __syncthreads();
  block_lu(M, r, s_perm, &s_piv, status);  // P M = L U
  for (int jb = G.job_begin; jb < G.job_end; ++jb) {
    const OpJob J = jobs[jb];
    const int32_t* src = piv + J.src_off;
    for (int j = threadIdx.x; j < J.src_len; j += blockDim.x) {
      const double2 xs = pts[src[j]];
      double2 x[kDeviceOpsMaxRank];
      if (G.type == 0) {  // M x = H(A, src_j)
        for (int i = 0; i < r; ++i) x[i] = hentry(pts[A[s_perm[i]]], xs, T);
        for (int i = 1; i < r; ++i)
          for (int k = 0; k < i; ++k) cfms2(x[i], M[k * r + i], x[k]);
        for (int i = r - 1; i >= 0; --i) {
          for (int k = i + 1; k < r; ++k) cfms2(x[i], M[k * r + i], x[k]);
          x[i] = cdiv2(x[i], M[i * r + i]);
        }
        for (int i = 0; i < r; ++i) {
          const int64_t at = J.stride > 0 ? (int64_t)i * J.stride + J.col_start + j : (int64_t)(J.col_start + j) * J.rows + i;
          ops[J.off + at] = x[i];
        }
      } else {  // x M = H(src_j, B): w U = a, y L = w, x_{perm[i]} = y_i
        for (int c = 0; c < r; ++c) x[c] = hentry(xs, pts[B[c]], T);
        for (int c = 0; c < r; ++c) {
          double2 s2 = x[c];
          for (int i = 0; i < c; ++i) cfms2(s2, x[i], M[c * r + i]);
          x[c] = cdiv2(s2, M[c * r + c]);
        }
        for (int c = r - 2; c >= 0; --c) {
          double2 s2 = x[c];
          for (int i = c + 1; i < r; ++i) cfms2(s2, x[i], M[c * r + i]);
          x[c] = s2;
        }
        for (int i = 0; i < r; ++i) {
          const int c = J.col_start + s_perm[i];
          const int64_t at = J.stride > 0 ? (int64_t)j * J.stride + c : (int64_t)c * J.rows + j;
          ops[J.off + at] = x[i];
        }
      }
    }
  }
}

template <typename T>
bool dev_upload(T** dst, const T* src, size_t count, cudaStream_t s, std::string& err) {
  if (!ck(cudaMalloc((void**)dst, std::max<size_t>(count, 1) * sizeof(T)), err, "cudaMalloc (ACA)")) return false;
  return count == 0 || ck(cudaMemcpyAsync(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice, s), err,
                          "cudaMemcpy (ACA)");
}

}  // namespace

DeviceAca::~DeviceAca() {
  if (pts_) cudaFree(pts_);
  if (w_) cudaFree(w_);
  if (q_) cudaFree(q_);
  if (stream_) cudaStreamDestroy(stream_);
}

int DeviceAca::init(const double* pts, const double* w, int64_t n, double kappa, std::string& err, const double* q) {
  kappa_ = kappa;
  if (!ck(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), err, "cudaStreamCreate (ACA)"))
    return DAFMM_ECUDA;
  std::vector<double2> xy(n);
  for (int64_t i = 0; i < n; ++i) xy[i] = make_double2(kappa * pts[2 * i], kappa * pts[2 * i + 1]);
  if (!dev_upload(&pts_, xy.data(), (size_t)n, stream_, err) || !dev_upload(&w_, w, (size_t)n, stream_, err) ||
      (q && !dev_upload(&q_, q, (size_t)n, stream_, err)) ||
      !ck(cudaStreamSynchronize(stream_), err, "upload (ACA)"))
    return DAFMM_ECUDA;
  return DAFMM_OK;
}

int DeviceAca::run(const std::vector<int32_t>& idx, std::vector<AcaProblem>& probs, double eps,
                   std::vector<int32_t>& piv_row, std::vector<int32_t>& piv_col, std::vector<int32_t>& rank,
                   int64_t& entries, std::string& err) {
  const int np = (int)probs.size();
  rank.assign(np, 0);
  if (np == 0) return DAFMM_OK;
  // output slots and the scratch stride (V: cap x n, U: cap x m, flags m + n bytes)
  int64_t out = 0, stride = 0;
  for (AcaProblem& p : probs) {
    const int cap = std::min(std::min(p.m, p.n), p.cap > 0 ? std::min(p.cap, kAcaMaxRank) : kAcaMaxRank);
    p.out_off = out;
    out += cap;
    const int64_t s = (int64_t)cap * (p.m + p.n) + ((int64_t)p.m + p.n + 15) / 16 + 1;
    stride = std::max(stride, s);
  }
  piv_row.assign(std::max<int64_t>(out, 1), -1);
  piv_col.assign(std::max<int64_t>(out, 1), -1);
  // problems by decreasing size (the larger ones start first); results are per problem
  std::vector<int> order(np);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return probs[a].m + probs[a].n > probs[b].m + probs[b].n; });
  std::vector<AcaProblem> sorted(np);
  for (int t = 0; t < np; ++t) sorted[t] = probs[order[t]];
  // grid: up to 4 CTAs per SM, within a scratch budget of a quarter of the free memory
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  size_t free_b = 0, total_b = 0;
  if (!ck(cudaMemGetInfo(&free_b, &total_b), err, "cudaMemGetInfo (ACA)")) return DAFMM_ECUDA;
  const size_t slot = (size_t)stride * sizeof(double2);
  int64_t grid = std::min<int64_t>(np, 4LL * sms);
  grid = std::min<int64_t>(grid, std::max<int64_t>(1, (int64_t)(free_b / 4 / slot)));
  if ((size_t)grid * slot > free_b) {
    err = "device ACA: scratch for one problem does not fit in device memory";
    return DAFMM_ENOMEM;
  }
  int32_t *d_idx = nullptr, *d_pr = nullptr, *d_pc = nullptr, *d_rank = nullptr;
  int* d_ticket = nullptr;
  AcaProblem* d_probs = nullptr;
  double2* d_scratch = nullptr;
  unsigned long long* d_ent = nullptr;
  bool ok = dev_upload(&d_idx, idx.data(), idx.size(), stream_, err) &&
            dev_upload(&d_probs, sorted.data(), sorted.size(), stream_, err) &&
            ck(cudaMalloc((void**)&d_pr, out * sizeof(int32_t) + 4), err, "cudaMalloc (ACA)") &&
            ck(cudaMalloc((void**)&d_pc, out * sizeof(int32_t) + 4), err, "cudaMalloc (ACA)") &&
            ck(cudaMalloc((void**)&d_rank, np * sizeof(int32_t)), err, "cudaMalloc (ACA)") &&
            ck(cudaMalloc((void**)&d_ticket, sizeof(int)), err, "cudaMalloc (ACA)") &&
            ck(cudaMalloc((void**)&d_ent, sizeof(unsigned long long)), err, "cudaMalloc (ACA)") &&
            ck(cudaMalloc((void**)&d_scratch, (size_t)grid * slot), err, "cudaMalloc (ACA scratch)") &&
            ck(cudaMemsetAsync(d_ticket, 0, sizeof(int), stream_), err, "memset") &&
            ck(cudaMemsetAsync(d_ent, 0, sizeof(unsigned long long), stream_), err, "memset");
  std::vector<int32_t> rk(np), pr(out), pc(out);
  unsigned long long ent = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  const bool trace = std::getenv("DAFMM_SETUP_TRACE") != nullptr;
  if (trace) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, stream_);
  }
  if (ok) {
    aca_kernel<<<(int)grid, kAcaThreads, 0, stream_>>>(d_probs, np, d_ticket, d_idx, pts_, w_, q_, 0.25 * kappa_ * kappa_, eps, d_scratch, stride,
                                                       d_pr, d_pc, d_rank, d_ent);
    if (trace) cudaEventRecord(e1, stream_);
    ok = ck(cudaGetLastError(), err, "aca_kernel") &&
         ck(cudaMemcpyAsync(rk.data(), d_rank, np * sizeof(int32_t), cudaMemcpyDeviceToHost, stream_), err, "D2H") &&
         (out == 0 || (ck(cudaMemcpyAsync(pr.data(), d_pr, out * sizeof(int32_t), cudaMemcpyDeviceToHost, stream_),
                          err, "D2H") &&
                       ck(cudaMemcpyAsync(pc.data(), d_pc, out * sizeof(int32_t), cudaMemcpyDeviceToHost, stream_),
                          err, "D2H"))) &&
         ck(cudaMemcpyAsync(&ent, d_ent, sizeof(ent), cudaMemcpyDeviceToHost, stream_), err, "D2H") &&
         ck(cudaStreamSynchronize(stream_), err, "aca_kernel");
  }
  if (trace && ok) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    int64_t mx = 0;
    for (const AcaProblem& q : probs) mx = std::max<int64_t>(mx, (int64_t)q.m + q.n);
    std::fprintf(stderr, "  aca: %d problems, grid %lld, slot %.1f MB, largest m+n %lld, kernel %.3f ms\n", np,
                 (long long)grid, slot / 1e6, (long long)mx, ms);
  }
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  for (void* q : {(void*)d_idx, (void*)d_pr, (void*)d_pc, (void*)d_rank, (void*)d_ticket, (void*)d_probs,
                  (void*)d_scratch, (void*)d_ent})
    if (q) cudaFree(q);
  if (!ok) return DAFMM_ECUDA;
  // back to the caller's problem order (out_off of the sorted copy = that of the original)
  for (int t = 0; t < np; ++t) rank[order[t]] = rk[t];
  for (int64_t t = 0; t < out; ++t) {
    piv_row[t] = pr[t];
    piv_col[t] = pc[t];
  }
  entries += (int64_t)ent;
  return DAFMM_OK;
}

int form_ops_device(const double* pts, int64_t n, double kappa, const std::vector<int32_t>& piv,
                    const std::vector<OpGroup>& groups, const std::vector<OpJob>& jobs, double2* ops,
                    std::string& err) {
  if (groups.empty()) return DAFMM_OK;
  cudaStream_t s = nullptr;
  if (!ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), err, "cudaStreamCreate (ops)")) return DAFMM_ECUDA;
  std::vector<double2> xy(n);
  for (int64_t i = 0; i < n; ++i) xy[i] = make_double2(kappa * pts[2 * i], kappa * pts[2 * i + 1]);
  double2* d_pts = nullptr;
  int32_t* d_piv = nullptr;
  OpGroup* d_groups = nullptr;
  OpJob* d_jobs = nullptr;
  int* d_status = nullptr;
  int st = 0;
  bool ok = dev_upload(&d_pts, xy.data(), (size_t)n, s, err) && dev_upload(&d_piv, piv.data(), piv.size(), s, err) &&
            dev_upload(&d_groups, groups.data(), groups.size(), s, err) &&
            dev_upload(&d_jobs, jobs.data(), jobs.size(), s, err) &&
            ck(cudaMalloc((void**)&d_status, sizeof(int)), err, "cudaMalloc (ops)") &&
            ck(cudaMemsetAsync(d_status, 0, sizeof(int), s), err, "memset (ops)");
  int rmax = 1;
  for (const OpGroup& g : groups) rmax = std::max(rmax, (int)g.r);
  const size_t smem = sizeof(double2) * rmax * rmax;
  ok = ok && ck(cudaFuncSetAttribute(ops_form_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), err,
                "ops_form_kernel shared memory");
  if (ok) {
    ops_form_kernel<<<(int)groups.size(), 128, smem, s>>>(d_groups, d_jobs, d_piv, d_pts, ops, d_status);
    ok = ck(cudaGetLastError(), err, "ops_form_kernel") &&
         ck(cudaMemcpyAsync(&st, d_status, sizeof(int), cudaMemcpyDeviceToHost, s), err, "D2H (ops)") &&
         ck(cudaStreamSynchronize(s), err, "ops_form_kernel");
  }
  for (void* q : {(void*)d_pts, (void*)d_piv, (void*)d_groups, (void*)d_jobs, (void*)d_status})
    if (q) cudaFree(q);
  cudaStreamDestroy(s);
  if (!ok) return DAFMM_ECUDA;
  if (st) {
    err = "singular NCA cross matrix";
    return DAFMM_ESETUP;
  }
  return DAFMM_OK;
}

}  // namespace dafmm
