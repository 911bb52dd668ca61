// HODLR preconditioner (Eq. hybrid) on the device.
//
// Ã approximates A = I + kappa^2 diag(q) K in the DAFMM tree order (HR1: binary tree of
// midpoint splits over the tree positions, leaves of at most n0 points).  Every off-diagonal
// sibling block A[gamma, sib(gamma)] is its rank-k ACA approximant U_gamma V_gamma^H = sum_l u_l
// v_l^T from the fixed-rank ACA (HR2; device ACA of setup_device.cu, mode 1, which writes the
// balanced factors straight into the planes below) -- in exact arithmetic the cross
// approximation A[gamma, J] A[I, J]^{-1} A[I, sib(gamma)] of its pivots, but without the
// inverse of the cross matrix, whose condition number reaches 1e15 once a fixed-rank ACA runs
// past the block's numerical rank.  Factorisation (HR3, the
// recursive Sherman-Morrison-Woodbury form of the HODLR direct solver the paper cites):
//
//   Ã_nu = diag(Ã_alpha, Ã_beta) (I + W Z^H),  W = diag(W_alpha, W_beta),  W_gamma = Ã_gamma^{-1} U_gamma,
//   Z^H = [[0, V_alpha^H], [V_beta^H, 0]],  S_nu = I + Z^H W = [[I, G_beta], [G_alpha, I]],
//   G_gamma = V_sib(gamma)^H W_gamma = sum_{t in gamma} Vcat[t]^T W[t],
//
// so Ã^{-1} b = leaf LU solves, then for every depth from the deepest split up to the root,
// b <- b - W S_nu^{-1} Z^H b.  The W of every depth are produced together, bottom-up: the leaf
// solves and then each depth's (I + W Z^H)^{-1} are applied to the U columns of all coarser
// depths (one N x (depths r) row-major matrix, Ucat).
//
// Layout: one plane per depth, N x r row-major: per point t (tree position), r complex values of
// Ucat (its row of W) and of Vcat (A[I_sib, t], its column of the sibling block's V^H),
// zero-padded beyond the block's rank.  Padding is exact: a zero column of Vcat / Ucat adds
// identity rows and columns to S.  Column c of the factorisation's right-hand sides (the U of
// all depths) is value c % r of plane c / r.
// Kernels per depth: segdot (Y_gamma = sum_t Vcat[t]^T X[t] over parts of each child),
// node (S factor / solve per split node), update (X[t] -= W[t] C_nu(t)).  The same kernels run the
// factorisation (X = Ucat, column chunks) and the apply (X = one vector).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <numeric>
#include <string>
#include <sys/stat.h>
#include <vector>

#include "dense.cuh"
#include "hodlr.h"
#include "setup_device.h"

namespace dafmm {

namespace {

constexpr int kMaxLeaf = 64;   // n0 <= 64 (two rows per lane in the warp solves)
constexpr int kMaxRank = 32;   // r <= 32 (S is at most 64 x 64)
constexpr int kChunk = 64;     // factorisation: right-hand-side columns per round

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

bool ck(cudaError_t e, std::string& err, const char* what) {
  if (e == cudaSuccess) return true;
  err = std::string(what) + ": " + cudaGetErrorString(e);
  return false;
}

// A_ts of the Lippmann-Schwinger matrix in tree positions: 1 + kappa^2 q_t D_t on the
// diagonal, kappa^2 q_t (i/4) H0(kappa |x_t - x_s|) w_s off it (reading D1).
struct AEntries {
  const double2* pts;  // kappa-scaled
  const double* w;
  const double* qk2;
  const double2* D;
  __device__ __forceinline__ double2 operator()(int64_t t, int64_t s, const PolyTable& T) const {
    const double q = qk2[t];
    if (t == s) {
      const double2 d = D[t];
      return make_double2(1.0 + q * d.x, q * d.y);
    }
    const double2 a = pts[t], b = pts[s];
    const double dx = a.x - b.x, dy = a.y - b.y;
    const double d2 = fma(dx, dx, dy * dy);
    double hr, hi;
    h0_generic_vec<1>(&d2, &hr, &hi, T);
    const double sc = 0.25 * q * w[s];
    return make_double2(-sc * hi, sc * hr);
  }
};

// Element (t, c) of a set of column planes: p + (c / pc) plane + t rs + c % pc.  The U planes
// (pc = rs = r, plane = N r) or one vector (pc = rs = 1).
struct XA {
  double2* p;
  int64_t plane;
  int pc, rs;
  __device__ __forceinline__ double2& at(int64_t t, int c) const {
    return p[(int64_t)(c / pc) * plane + t * rs + c % pc];
  }
};

// Inverse of the n x n matrix whose LU (P M = L U, column-major, in shared memory) is M, one
// column per thread: column c solves L U x = P e_c; written column-major to out.  (The leaf blocks
// and the Woodbury factors are applied as dense inverses: a GEMV per apply instead of a latency
// chain of 2n dependent substitution steps.)
__device__ void lu_inverse(const double2* M, const int* perm, int n, double2* __restrict__ out) {
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    double2 x[kMaxLeaf];
    for (int i = 0; i < n; ++i) x[i] = make_double2(perm[i] == c ? 1.0 : 0.0, 0.0);
    for (int i = 1; i < n; ++i)
      for (int j = 0; j < i; ++j) cfms2(x[i], M[j * n + i], x[j]);
    for (int i = n - 1; i >= 0; --i) {
      for (int j = i + 1; j < n; ++j) cfms2(x[i], M[j * n + i], x[j]);
      x[i] = cdiv2(x[i], M[i * n + i]);
    }
    for (int i = 0; i < n; ++i) out[(int64_t)c * n + i] = x[i];
  }
}

// ---- leaves: dense A[leaf, leaf], its LU and inverse ----
__global__ void hodlr_leaf_lu_kernel(const int64_t* __restrict__ la, const int32_t* __restrict__ ln,
                                     const int64_t* __restrict__ lu_off, AEntries A, double2* __restrict__ lu,
                                     int32_t* __restrict__ prow, int* status) {
  extern __shared__ double2 M[];
  __shared__ PolyTable T;
  __shared__ int s_perm[kMaxLeaf];
  __shared__ int s_piv;
  load_poly_table(T);
  const int leaf = blockIdx.x;
  const int64_t a = la[leaf];
  const int n = ln[leaf];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) M[e] = A(a + e % n, a + e / n, T);
  __syncthreads();
  block_lu(M, n, s_perm, &s_piv, status);
  lu_inverse(M, s_perm, n, lu + lu_off[leaf]);  // the leaf's A^{-1}, column-major
  (void)prow;
}

// X[leaf rows, 0 .. nc) <- A_leaf^{-1} X (factorisation: many columns, one per thread)
__global__ void hodlr_leaf_solve_multi_kernel(const int64_t* __restrict__ la, const int32_t* __restrict__ ln,
                                              const int64_t* __restrict__ lu_off, const double2* __restrict__ inv,
                                              XA X, int nc) {
  extern __shared__ double2 M[];
  const int leaf = blockIdx.x;
  const int64_t a = la[leaf];
  const int n = ln[leaf];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) M[e] = inv[lu_off[leaf] + e];
  __syncthreads();
  for (int c = threadIdx.x; c < nc; c += blockDim.x) {
    double2 v[kMaxLeaf];
    for (int i = 0; i < n; ++i) v[i] = X.at(a + i, c);
    for (int i = 0; i < n; ++i) {
      double2 acc = make_double2(0.0, 0.0);
      for (int j = 0; j < n; ++j) cfma2(acc, M[j * n + i], v[j]);
      X.at(a + i, c) = acc;
    }
  }
}

// apply: x[leaf] <- A_leaf^{-1} x[leaf], one warp per leaf: lanes own rows lane, lane + 32; the
// inverse's columns are read coalesced and independent of each other (loads pipeline)
__global__ void __launch_bounds__(128) hodlr_leaf_solve_vec_kernel(int nleaves, const int64_t* __restrict__ la,
                                                                   const int32_t* __restrict__ ln,
                                                                   const int64_t* __restrict__ lu_off,
                                                                   const double2* __restrict__ inv,
                                                                   double2* __restrict__ x) {
  const int leaf = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (leaf >= nleaves) return;
  const int lane = threadIdx.x & 31;
  const int64_t a = la[leaf];
  const int n = ln[leaf];
  const double2* M = inv + lu_off[leaf];
  double2 v0 = make_double2(0.0, 0.0), v1 = v0;
  if (lane < n) v0 = x[a + lane];
  if (lane + 32 < n) v1 = x[a + lane + 32];
  double2 y0 = make_double2(0.0, 0.0), y1 = y0;
#pragma unroll 4
  for (int j = 0; j < n; ++j) {
    const double2 src = j < 32 ? v0 : v1;
    const double2 xj = make_double2(__shfl_sync(0xffffffffu, src.x, j & 31), __shfl_sync(0xffffffffu, src.y, j & 31));
    if (lane < n) cfma2(y0, M[j * n + lane], xj);
    if (lane + 32 < n) cfma2(y1, M[j * n + lane + 32], xj);
  }
  if (lane < n) x[a + lane] = y0;
  if (lane + 32 < n) x[a + lane + 32] = y1;
}

// ---- per depth: Y partials over parts (part = child id, t0, t1) ----
// partial[(p r + i) nc + c] = sum_{t in part p} Vp[t r + i] X(t, xc0 + c)   (factorisation)
__global__ void hodlr_segdot_kernel(const int32_t* __restrict__ parts, const double2* __restrict__ Vp, int r, XA X,
                                    int xc0, int nc, double2* __restrict__ partial) {
  const int p = blockIdx.x;
  const int tc = max(1, (int)blockDim.x / r);
  const int i = threadIdx.x / tc, c = blockIdx.y * tc + threadIdx.x % tc;
  if (i >= r || c >= nc) return;
  const int64_t t0 = parts[3 * p + 1], t1 = parts[3 * p + 2];
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t t = t0; t < t1; ++t) cfma2(acc, Vp[t * r + i], X.at(t, xc0 + c));
  partial[((int64_t)p * r + i) * nc + c] = acc;
}

// apply (one vector): partial[p r + i] = sum_{t in part p} Vp[t r + i] x[t]; the CTA's threads
// are (row slot, i) with rp = r rounded up to a power of two lanes per row, so each row's r
// values are one contiguous read; the slots are summed in a fixed order.
__global__ void __launch_bounds__(256) hodlr_segdot_vec_kernel(const int32_t* __restrict__ parts,
                                                               const double2* __restrict__ Vp, int r, int rp,
                                                               const double2* __restrict__ x,
                                                               double2* __restrict__ partial) {
  __shared__ double2 red[256];
  const int p = blockIdx.x;
  const int slot = threadIdx.x / rp, i = threadIdx.x % rp, nslot = blockDim.x / rp;
  const int64_t t0 = parts[3 * p + 1], t1 = parts[3 * p + 2];
  double2 acc = make_double2(0.0, 0.0);
  if (i < r)
    for (int64_t t = t0 + slot; t < t1; t += nslot) cfma2(acc, Vp[t * r + i], x[t]);
  red[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < r) {
    double2 sm = make_double2(0.0, 0.0);
    for (int q = 0; q < nslot; ++q) {
      sm.x += red[q * rp + threadIdx.x].x;
      sm.y += red[q * rp + threadIdx.x].y;
    }
    partial[(int64_t)p * r + threadIdx.x] = sm;
  }
}

// apply: x[t] -= sum_i Up[t r + i] C[nu][half r + i] over the rows of part p (child 2 nu + half);
// rp lanes per row, reduced by xor shuffles within the lane group.
__global__ void __launch_bounds__(256) hodlr_update_vec_kernel(const int32_t* __restrict__ parts,
                                                               const double2* __restrict__ Up, int r, int rp,
                                                               const double2* __restrict__ C,
                                                               double2* __restrict__ x) {
  const int p = blockIdx.x;
  const int child = parts[3 * p];
  const int slot = threadIdx.x / rp, i = threadIdx.x % rp, nslot = blockDim.x / rp;
  const int64_t t0 = parts[3 * p + 1], t1 = parts[3 * p + 2];
  const double2 cc = i < r ? C[(int64_t)(child >> 1) * 2 * r + (child & 1) * r + i] : make_double2(0.0, 0.0);
  for (int64_t base = t0; base < t1; base += nslot) {  // uniform trip count: every lane shuffles
    const int64_t t = base + slot;
    double2 v = make_double2(0.0, 0.0);
    if (t < t1 && i < r) cfma2(v, Up[t * r + i], cc);
    for (int o = rp >> 1; o > 0; o >>= 1) {
      v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
      v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    if (t < t1 && i == 0) {
      x[t].x -= v.x;
      x[t].y -= v.y;
    }
  }
}

// Y_gamma[i][c]: the sum of the child's parts, in part order
__device__ __forceinline__ double2 child_sum(const double2* __restrict__ partial, const int32_t* __restrict__ pptr,
                                             int child, int r, int nc, int i, int c) {
  double2 s = make_double2(0.0, 0.0);
#pragma unroll 4
  for (int p = pptr[child]; p < pptr[child + 1]; ++p) {
    const double2 v = partial[((int64_t)p * r + i) * nc + c];
    s.x += v.x;
    s.y += v.y;
  }
  return s;
}

// ---- per split node nu (children 2 nu = alpha, 2 nu + 1 = beta) ----
// factor (gcol >= 0): S = [[I, G_beta], [G_alpha, I]] from partial columns gcol .. gcol + r, LU to
// S_lu / S_prow.  Then (ncs > 0) C[nu][i][c] = (S^{-1} [Y_beta; Y_alpha])_i for columns c < ncs.
__global__ void hodlr_node_kernel(const int32_t* __restrict__ pptr, const double2* __restrict__ partial, int r,
                                  int nc, int gcol, int ncs, double2* __restrict__ S_lu, double2* __restrict__ S_inv,
                                  int32_t* __restrict__ S_prow, double2* __restrict__ C, int* status) {
  extern __shared__ double2 S[];  // (2r)^2, column-major (factor and multi-column solves)
  __shared__ int s_perm[2 * kMaxRank];
  __shared__ int s_piv;
  const int nu = blockIdx.x, R2 = 2 * r;
  const int ca = 2 * nu, cb = 2 * nu + 1;
  double2* lu = S_lu + (int64_t)nu * R2 * R2;
  if (gcol < 0 && ncs == 1) {  // apply: one warp, C = S^{-1} [Y_beta; Y_alpha] as a GEMV
    const int lane = threadIdx.x;
    if (lane >= 32) return;
    const double2* Si = S_inv + (int64_t)nu * R2 * R2;
    auto rhs = [&](int q) {  // the child's parts summed in part order
      return q < r ? child_sum(partial, pptr, cb, r, nc, q, 0) : child_sum(partial, pptr, ca, r, nc, q - r, 0);
    };
    const double2 b0 = lane < R2 ? rhs(lane) : make_double2(0.0, 0.0);
    const double2 b1 = lane + 32 < R2 ? rhs(lane + 32) : make_double2(0.0, 0.0);
    double2 y0 = make_double2(0.0, 0.0), y1 = y0;
#pragma unroll 4
    for (int q = 0; q < R2; ++q) {
      const double2 src = q < 32 ? b0 : b1;
      const double2 bq = make_double2(__shfl_sync(0xffffffffu, src.x, q & 31), __shfl_sync(0xffffffffu, src.y, q & 31));
      if (lane < R2) cfma2(y0, Si[q * R2 + lane], bq);
      if (lane + 32 < R2) cfma2(y1, Si[q * R2 + lane + 32], bq);
    }
    if (lane < R2) C[(int64_t)nu * R2 + lane] = y0;
    if (lane + 32 < R2) C[(int64_t)nu * R2 + lane + 32] = y1;
    return;
  }
  if (gcol >= 0) {
    for (int e = threadIdx.x; e < R2 * R2; e += blockDim.x) {
      const int i = e % R2, j = e / R2;
      double2 v = make_double2(i == j ? 1.0 : 0.0, 0.0);
      if (i < r && j >= r) v = child_sum(partial, pptr, cb, r, nc, i, gcol + j - r);       // G_beta
      else if (i >= r && j < r) v = child_sum(partial, pptr, ca, r, nc, i - r, gcol + j);  // G_alpha
      S[e] = v;
    }
    __syncthreads();
    block_lu(S, R2, s_perm, &s_piv, status);
    for (int e = threadIdx.x; e < R2 * R2; e += blockDim.x) lu[e] = S[e];
    lu_inverse(S, s_perm, R2, S_inv + (int64_t)nu * R2 * R2);  // for the apply
    for (int i = threadIdx.x; i < R2; i += blockDim.x) S_prow[(int64_t)nu * R2 + i] = s_perm[i];
  } else {
    for (int e = threadIdx.x; e < R2 * R2; e += blockDim.x) S[e] = lu[e];
    for (int i = threadIdx.x; i < R2; i += blockDim.x) s_perm[i] = S_prow[(int64_t)nu * R2 + i];
  }
  __syncthreads();
  if (ncs <= 0) return;
  for (int c = threadIdx.x; c < ncs; c += blockDim.x) {
    double2 v[2 * kMaxRank];
    for (int i = 0; i < R2; ++i) {
      const int q = s_perm[i];
      v[i] = q < r ? child_sum(partial, pptr, cb, r, nc, q, c) : child_sum(partial, pptr, ca, r, nc, q - r, c);
    }
    for (int i = 1; i < R2; ++i)
      for (int j = 0; j < i; ++j) cfms2(v[i], S[j * R2 + i], v[j]);
    for (int i = R2 - 1; i >= 0; --i) {
      for (int j = i + 1; j < R2; ++j) cfms2(v[i], S[j * R2 + i], v[j]);
      v[i] = cdiv2(v[i], S[i * R2 + i]);
    }
    for (int i = 0; i < R2; ++i) C[((int64_t)nu * R2 + i) * ncs + c] = v[i];
  }
}

// X(t, xc0 + c) -= sum_i Up[t r + i] C[nu][half(t) r + i][c] for t in split node nu (factorisation)
__global__ void hodlr_update_kernel(int nnodes, const int64_t* __restrict__ amb, const double2* __restrict__ Up,
                                    int r, const double2* __restrict__ C, int ncs, XA X, int xc0, int64_t n) {
  const int64_t total = n * ncs;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / ncs;
    const int c = (int)(e % ncs);
    int lo = 0, hi = nnodes - 1;  // last split node with a <= t
    if (nnodes == 0 || t < amb[0]) continue;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (amb[3 * mid] <= t) lo = mid;
      else hi = mid - 1;
    }
    if (t >= amb[3 * lo + 2]) continue;
    const int half = t >= amb[3 * lo + 1] ? 1 : 0;
    const double2* cc = C + ((int64_t)lo * 2 * r + half * r) * ncs + c;
    const double2* u = Up + t * r;
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < r; ++i) cfma2(acc, u[i], cc[(int64_t)i * ncs]);
    double2& x = X.at(t, xc0 + c);
    x.x -= acc.x;
    x.y -= acc.y;
  }
}

__global__ void hodlr_gather_kernel(int64_t n, const int32_t* __restrict__ perm, const double2* __restrict__ in,
                                    double2* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = in[perm[t]];
}
__global__ void hodlr_scatter_kernel(int64_t n, const int32_t* __restrict__ perm, const double2* __restrict__ in,
                                     double2* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    out[perm[t]] = in[t];
}

template <typename T>
bool halloc(HodlrPlan& h, T** p, size_t count, std::string& err) {
  *p = nullptr;
  if (!ck(cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T)), err, "cudaMalloc (HODLR)")) return false;
  h.allocations.push_back(*p);
  h.device_bytes += std::max<size_t>(count, 1) * sizeof(T);
  return true;
}
template <typename T>
bool hupload(HodlrPlan& h, T** p, const std::vector<T>& v, std::string& err) {
  if (!halloc(h, p, v.size(), err)) return false;
  return v.empty() || ck(cudaMemcpy(*p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), err, "H2D (HODLR)");
}

int grid_for(int64_t work, int threads) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((work + threads - 1) / threads, 148 * 16));
}

// one round of the per-depth kernels on columns [xc0, xc0 + nc) of the U planes (factorisation:
// segdot, node factor / solve, update)
int factor_round(HodlrPlan& h, int d, int xc0, int nc, bool gcols, cudaStream_t s, std::string& err) {
  const int r = h.r, nn = (int)h.split_a[d].size();
  if (nn == 0) return DAFMM_OK;
  const int64_t plane = h.n * (int64_t)r;
  const XA X{h.Ucat, plane, r, r};
  const double2* Vp = h.Vcat + d * plane;
  const double2* Up = h.Ucat + d * plane;
  const int tc = std::max(1, 256 / r);
  const int threads = ((std::min(nc, tc) * r + 31) / 32) * 32;
  dim3 grid(h.nparts[d], (nc + tc - 1) / tc);
  hodlr_segdot_kernel<<<grid, threads, 0, s>>>(h.part_d[d], Vp, r, X, xc0, nc, h.partial);
  const size_t smem = (size_t)4 * r * r * sizeof(double2);
  if (gcols) {  // the G columns (depth d's own U): S_nu = I + Z^H W, factored
    hodlr_node_kernel<<<nn, 128, smem, s>>>(h.part_ptr_d[d], h.partial, r, nc, 0, 0, h.S_lu[d], h.S_inv[d],
                                            h.S_prow[d], h.C, h.status);
  } else {
    hodlr_node_kernel<<<nn, 128, smem, s>>>(h.part_ptr_d[d], h.partial, r, nc, -1, nc, h.S_lu[d], h.S_inv[d],
                                            h.S_prow[d], h.C, h.status);
    hodlr_update_kernel<<<grid_for(h.n * nc, 256), 256, 0, s>>>(nn, h.split_d[d], Up, r, h.C, nc, X, xc0, h.n);
  }
  return ck(cudaGetLastError(), err, "hodlr factor round") ? DAFMM_OK : DAFMM_ECUDA;
}

// one depth of the apply on the tree-order vector h.xt: b <- b - W S^{-1} Z^H b
int apply_round(HodlrPlan& h, int d, cudaStream_t s, std::string& err) {
  const int r = h.r, nn = (int)h.split_a[d].size();
  if (nn == 0) return DAFMM_OK;
  int rp = 1;
  while (rp < r) rp <<= 1;
  const int64_t plane = h.n * (int64_t)r;
  hodlr_segdot_vec_kernel<<<h.nparts[d], 256, 0, s>>>(h.part_d[d], h.Vcat + d * plane, r, rp, h.xt, h.partial);
  hodlr_node_kernel<<<nn, 32, 0, s>>>(h.part_ptr_d[d], h.partial, r, 1, -1, 1, h.S_lu[d], h.S_inv[d], h.S_prow[d],
                                      h.C, h.status);
  hodlr_update_vec_kernel<<<h.nparts[d], 256, 0, s>>>(h.part_d[d], h.Ucat + d * plane, r, rp, h.C, h.xt);
  return ck(cudaGetLastError(), err, "hodlr apply round") ? DAFMM_OK : DAFMM_ECUDA;
}

bool write_npy_i64(const std::string& path, const std::vector<int64_t>& v, std::vector<int64_t> shape) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) return false;
  std::string sh = "(";
  for (size_t i = 0; i < shape.size(); ++i) sh += std::to_string(shape[i]) + (shape.size() == 1 ? "," : (i + 1 < shape.size() ? ", " : ""));
  sh += ")";
  std::string hdr = "{'descr': '<i8', 'fortran_order': False, 'shape': " + sh + ", }";
  while ((10 + hdr.size() + 1) % 64) hdr += ' ';
  hdr += '\n';
  const unsigned char magic[8] = {0x93, 'N', 'U', 'M', 'P', 'Y', 1, 0};
  const uint16_t hl = (uint16_t)hdr.size();
  bool ok = std::fwrite(magic, 1, 8, f) == 8 && std::fwrite(&hl, 2, 1, f) == 1 &&
            std::fwrite(hdr.data(), 1, hdr.size(), f) == hdr.size() &&
            (v.empty() || std::fwrite(v.data(), sizeof(int64_t), v.size(), f) == v.size());
  return std::fclose(f) == 0 && ok;
}

}  // namespace

void hodlr_free(HodlrPlan& h) {
  for (void* p : h.allocations) cudaFree(p);
  h.allocations.clear();
  h.device_bytes = 0;
}

int hodlr_create(const Plan& P, const DevPlan& d, int rank, int leaf_size, int64_t max_block, HodlrPlan& h,
                 std::string& err) {
  if (P.opt.kernel_mode != 0) { err = "the HODLR preconditioner needs kernel_mode 0 (Lippmann-Schwinger)"; return DAFMM_EINVAL; }
  if (rank < 1 || rank > kMaxRank) { err = "HODLR rank must be in [1, 32]"; return DAFMM_EINVAL; }
  if (leaf_size < 1 || leaf_size > kMaxLeaf) { err = "HODLR leaf size must be in [1, 64]"; return DAFMM_EINVAL; }
  if (max_block < 0) { err = "HODLR max_block must be >= 0"; return DAFMM_EINVAL; }
  h.max_block = max_block;
  const int64_t n = P.n;
  h.n = n;
  h.r = rank;
  h.n0 = leaf_size;
  h.perm = d.perm;
  cudaStream_t s = d.stream;
  // ---- HR1: binary tree of midpoint splits over the tree positions ----
  {
    std::vector<std::pair<int64_t, int64_t>> level = {{0, n}};
    while (!level.empty()) {
      std::vector<std::pair<int64_t, int64_t>> next;
      std::vector<int64_t> sa, sm, sb;
      for (auto& nd : level) {
        if (nd.second - nd.first > leaf_size) {
          const int64_t m = (nd.first + nd.second) / 2;
          sa.push_back(nd.first);
          sm.push_back(m);
          sb.push_back(nd.second);
          next.push_back({nd.first, m});
          next.push_back({m, nd.second});
        } else {
          h.leaf_a.push_back(nd.first);
          h.leaf_n.push_back(nd.second - nd.first);
        }
      }
      if (!sa.empty()) {
        h.split_a.push_back(std::move(sa));
        h.split_m.push_back(std::move(sm));
        h.split_b.push_back(std::move(sb));
      }
      level.swap(next);
    }
  }
  h.depths = (int)h.split_a.size();
  h.ld = std::max(1, h.depths * rank);
  // leaves in tree order
  {
    std::vector<int> o(h.leaf_a.size());
    std::iota(o.begin(), o.end(), 0);
    std::sort(o.begin(), o.end(), [&](int a, int b) { return h.leaf_a[a] < h.leaf_a[b]; });
    std::vector<int64_t> a2, n2;
    for (int i : o) {
      a2.push_back(h.leaf_a[i]);
      n2.push_back(h.leaf_n[i]);
    }
    h.leaf_a.swap(a2);
    h.leaf_n.swap(n2);
  }
  const int nleaves = (int)h.leaf_a.size();
  AEntries A{d.pts_t, d.w_t, d.qk2_t, d.D_t};
  // ---- device buffers ----
  if (!halloc(h, &h.Ucat, (size_t)n * h.ld, err) || !halloc(h, &h.Vcat, (size_t)n * h.ld, err) ||
      !halloc(h, &h.xt, (size_t)n, err) || !halloc(h, &h.status, 1, err))
    return DAFMM_ECUDA;
  if (!ck(cudaMemsetAsync(h.status, 0, sizeof(int), s), err, "memset") ||
      !ck(cudaMemsetAsync(h.Ucat, 0, sizeof(double2) * (size_t)n * h.ld, s), err, "memset") ||
      !ck(cudaMemsetAsync(h.Vcat, 0, sizeof(double2) * (size_t)n * h.ld, s), err, "memset") ||
      !ck(cudaFuncSetAttribute(hodlr_node_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(4 * kMaxRank * kMaxRank * sizeof(double2))),
          err, "smem attr") ||
      // the ACA runs on its own stream and writes into the zeroed planes
      !ck(cudaStreamSynchronize(s), err, "memset (HODLR)"))
    return DAFMM_ECUDA;
  // ---- HR2: pivots of every sibling block by the device ACA (mode 1), depth by depth ----
  double t0 = now_s();
  {
    DeviceAca aca;
    int rc = aca.init(P.pts.data(), P.w.data(), n, P.kappa, err, P.q.data());
    if (rc != DAFMM_OK) return rc;
    std::vector<int32_t> idx(P.perm.begin(), P.perm.end());
    h.blk_ptr.resize(h.depths);
    h.blk_I.resize(h.depths);
    h.blk_J.resize(h.depths);
    int64_t rank_sum = 0, nblk = 0;
    for (int dd = 0; dd < h.depths; ++dd) {
      const size_t nn = h.split_a[dd].size();
      std::vector<AcaProblem> probs;
      std::vector<int> prob_of(2 * nn, -1);
      for (size_t i = 0; i < nn; ++i) {
        const int64_t a = h.split_a[dd][i], m = h.split_m[dd][i], b = h.split_b[dd][i];
        for (int side = 0; side < 2; ++side) {
          const int64_t ra = side ? m : a, rb = side ? b : m, c0 = side ? a : m, c1 = side ? m : b;
          // first row: the first row with the largest |q| (a row with q = 0 is zero in A's
          // off-diagonal blocks); no such row: rank 0
          int64_t best = -1;
          double bq = 0.0;
          for (int64_t t = ra; t < rb; ++t) {
            const double aq = std::fabs(P.q[P.perm[t]]);
            if (aq > bq) { bq = aq; best = t; }
          }
          // HR5 (option): blocks of more than max_block rows are dropped (rank 0)
          if (best < 0 || (max_block > 0 && rb - ra > max_block)) continue;
          AcaProblem pr{};
          pr.row_off = ra;
          pr.col_off = c0;
          pr.m = (int32_t)(rb - ra);
          pr.n = (int32_t)(c1 - c0);
          pr.first_row = (int32_t)(best - ra);
          pr.cap = rank;
          pr.mode = 1;
          // HR2: the block's ACA factors go straight into the depth's planes: U_gamma rows at the
          // rows' tree positions, V columns at the sibling's
          pr.u_out = h.Ucat + (int64_t)dd * n * rank;
          pr.v_out = h.Vcat + (int64_t)dd * n * rank;
          pr.ldo = rank;
          prob_of[2 * i + side] = (int)probs.size();
          probs.push_back(pr);
        }
      }
      std::vector<int32_t> prow, pcol, rk;
      rc = aca.run(idx, probs, 0.0, prow, pcol, rk, h.aca_entries, err);
      if (rc != DAFMM_OK) return rc;
      auto& ptr = h.blk_ptr[dd];
      ptr.assign(1, 0);
      for (size_t g = 0; g < 2 * nn; ++g) {
        const int pi = prob_of[g];
        const int k = pi < 0 ? 0 : rk[pi];
        for (int q = 0; q < k; ++q) {
          h.blk_I[dd].push_back((int32_t)(probs[pi].row_off + prow[probs[pi].out_off + q]));
          h.blk_J[dd].push_back((int32_t)(probs[pi].col_off + pcol[probs[pi].out_off + q]));
        }
        ptr.push_back((int32_t)h.blk_I[dd].size());
        rank_sum += k;
        ++nblk;
        h.max_rank = std::max(h.max_rank, k);
      }
    }
    h.mean_rank = nblk ? (double)rank_sum / nblk : 0.0;
  }
  double t1 = now_s();
  h.t_aca = t1 - t0;
  // parts per depth: children cut into runs of at most `pl` rows
  const int64_t pl = std::max<int64_t>(256, n / 1024);
  int64_t max_parts = 1;
  h.part_d.resize(h.depths);
  h.part_ptr_d.resize(h.depths);
  h.part_ptr.resize(h.depths);
  h.nparts.resize(h.depths);
  h.split_d.resize(h.depths);
  h.S_lu.resize(h.depths);
  h.S_inv.resize(h.depths);
  h.S_prow.resize(h.depths);
  int64_t max_nodes = 1;
  for (int dd = 0; dd < h.depths; ++dd) {
    const size_t nn = h.split_a[dd].size();
    std::vector<int32_t> parts;
    auto& pp = h.part_ptr[dd];
    pp.assign(1, 0);
    std::vector<int64_t> amb;
    for (size_t i = 0; i < nn; ++i) {
      const int64_t a = h.split_a[dd][i], m = h.split_m[dd][i], b = h.split_b[dd][i];
      amb.insert(amb.end(), {a, m, b});
      for (int side = 0; side < 2; ++side) {
        const int64_t ca = side ? m : a, cb = side ? b : m;
        for (int64_t t = ca; t < cb; t += pl) {
          parts.push_back((int32_t)(2 * i + side));
          parts.push_back((int32_t)t);
          parts.push_back((int32_t)std::min(cb, t + pl));
        }
        pp.push_back((int32_t)(parts.size() / 3));
      }
    }
    h.nparts[dd] = (int)(parts.size() / 3);
    max_parts = std::max<int64_t>(max_parts, h.nparts[dd]);
    max_nodes = std::max<int64_t>(max_nodes, (int64_t)nn);
    if (!hupload(h, &h.part_d[dd], parts, err) || !hupload(h, &h.part_ptr_d[dd], pp, err) ||
        !hupload(h, &h.split_d[dd], amb, err) || !halloc(h, &h.S_lu[dd], nn * 4 * rank * rank, err) ||
        !halloc(h, &h.S_inv[dd], nn * 4 * rank * rank, err) ||
        !halloc(h, &h.S_prow[dd], nn * 2 * rank, err))
      return DAFMM_ECUDA;
  }
  const int maxcols = std::max(rank, kChunk);
  h.partial_len = max_parts * rank * maxcols;
  h.C_len = max_nodes * 2 * rank * maxcols;
  if (!halloc(h, &h.partial, (size_t)h.partial_len, err) || !halloc(h, &h.C, (size_t)h.C_len, err)) return DAFMM_ECUDA;
  // ---- leaves: LU of A[leaf, leaf] ----
  std::vector<int64_t> lu_off(nleaves);
  int64_t lu_len = 0;
  std::vector<int32_t> ln32(nleaves);
  for (int i = 0; i < nleaves; ++i) {
    lu_off[i] = lu_len;
    lu_len += h.leaf_n[i] * h.leaf_n[i];
    ln32[i] = (int32_t)h.leaf_n[i];
  }
  if (!hupload(h, &h.leaf_a_d, h.leaf_a, err) || !hupload(h, &h.leaf_n_d, ln32, err) ||
      !hupload(h, &h.leaf_lu_off, lu_off, err) || !halloc(h, &h.leaf_lu, (size_t)lu_len, err) ||
      !halloc(h, &h.leaf_prow, (size_t)nleaves * kMaxLeaf, err))
    return DAFMM_ECUDA;
  const size_t leaf_smem = (size_t)leaf_size * leaf_size * sizeof(double2);
  if (!ck(cudaFuncSetAttribute(hodlr_leaf_lu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)leaf_smem), err,
          "smem attr") ||
      !ck(cudaFuncSetAttribute(hodlr_leaf_solve_multi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)leaf_smem),
          err, "smem attr"))
    return DAFMM_ECUDA;
  hodlr_leaf_lu_kernel<<<nleaves, 256, leaf_smem, s>>>(h.leaf_a_d, h.leaf_n_d, h.leaf_lu_off, A, h.leaf_lu,
                                                      h.leaf_prow, h.status);
  double t2 = now_s();
  h.t_basis = t2 - t1;
  // ---- HR3: factorisation.  W = leaf solves of every depth's U, then depth by depth
  // (deepest split first): factor S from block d (the G columns), apply (I + W Z^H)^{-1} of the
  // depth to the U columns of the coarser depths, chunk by chunk ----
  hodlr_leaf_solve_multi_kernel<<<nleaves, 64, leaf_smem, s>>>(h.leaf_a_d, h.leaf_n_d, h.leaf_lu_off, h.leaf_lu,
                                                              XA{h.Ucat, n * (int64_t)rank, rank, rank}, h.ld);
  if (!ck(cudaGetLastError(), err, "hodlr leaf solve")) return DAFMM_ECUDA;
  for (int dd = h.depths - 1; dd >= 0; --dd) {
    int rc = factor_round(h, dd, dd * rank, rank, true, s, err);
    if (rc != DAFMM_OK) return rc;
    for (int c0 = 0; c0 < dd * rank; c0 += kChunk) {
      rc = factor_round(h, dd, c0, std::min(kChunk, dd * rank - c0), false, s, err);
      if (rc != DAFMM_OK) return rc;
    }
  }
  int st = 0;
  if (!ck(cudaMemcpyAsync(&st, h.status, sizeof(int), cudaMemcpyDeviceToHost, s), err, "D2H") ||
      !ck(cudaStreamSynchronize(s), err, "hodlr factorisation"))
    return DAFMM_ECUDA;
  if (st) { err = "HODLR: singular leaf block, cross matrix or S factor"; return DAFMM_ESETUP; }
  h.t_factor = now_s() - t2;
  return DAFMM_OK;
}

int hodlr_apply(HodlrPlan& h, const double2* in, double2* out, cudaStream_t s, std::string& err) {
  const int64_t n = h.n;
  const int g = grid_for(n, 256);
  hodlr_gather_kernel<<<g, 256, 0, s>>>(n, h.perm, in, h.xt);
  const int nleaves = (int)h.leaf_a.size();
  hodlr_leaf_solve_vec_kernel<<<(nleaves + 3) / 4, 128, 0, s>>>(nleaves, h.leaf_a_d, h.leaf_n_d, h.leaf_lu_off,
                                                                h.leaf_lu, h.xt);
  for (int dd = h.depths - 1; dd >= 0; --dd) {
    int rc = apply_round(h, dd, s, err);
    if (rc != DAFMM_OK) return rc;
  }
  hodlr_scatter_kernel<<<g, 256, 0, s>>>(n, h.perm, h.xt, out);
  return ck(cudaGetLastError(), err, "hodlr apply") ? DAFMM_OK : DAFMM_ECUDA;
}

int hodlr_export(const HodlrPlan& h, const Plan& P, const std::string& dir, std::string& err) {
  mkdir(dir.c_str(), 0755);
  std::vector<int64_t> blocks, ptr = {0}, I, J, perm(P.perm.begin(), P.perm.end());
  for (int dd = 0; dd < h.depths; ++dd)
    for (size_t i = 0; i < h.split_a[dd].size(); ++i) {
      const int64_t a = h.split_a[dd][i], m = h.split_m[dd][i], b = h.split_b[dd][i];
      for (int side = 0; side < 2; ++side) {
        const size_t g = 2 * i + side;
        if (side == 0) blocks.insert(blocks.end(), {dd + 1, a, m, m, b});
        else blocks.insert(blocks.end(), {dd + 1, m, b, a, m});
        for (int q = h.blk_ptr[dd][g]; q < h.blk_ptr[dd][g + 1]; ++q) {
          I.push_back(h.blk_I[dd][q]);
          J.push_back(h.blk_J[dd][q]);
        }
        ptr.push_back((int64_t)I.size());
      }
    }
  const std::vector<int64_t> meta = {h.r, h.n0, h.n, h.max_block};
  bool ok = write_npy_i64(dir + "/hodlr_blocks.npy", blocks, {(int64_t)blocks.size() / 5, 5}) &&
            write_npy_i64(dir + "/hodlr_piv_ptr.npy", ptr, {(int64_t)ptr.size()}) &&
            write_npy_i64(dir + "/hodlr_I.npy", I, {(int64_t)I.size()}) &&
            write_npy_i64(dir + "/hodlr_J.npy", J, {(int64_t)J.size()}) &&
            write_npy_i64(dir + "/hodlr_perm.npy", perm, {(int64_t)perm.size()}) &&
            write_npy_i64(dir + "/hodlr_meta.npy", meta, {(int64_t)meta.size()});
  if (!ok) { err = "could not write HODLR export to " + dir; return DAFMM_EINVAL; }
  return DAFMM_OK;
}

}  // namespace dafmm
