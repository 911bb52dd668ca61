// sm_100a kernels of the DAFMM matvec and the GMRES vector work.
//
// Passes per matvec:
//   gather      x (caller order) -> x_t, v_t = w o x_t (tree order)                 HBM
//   p2m / m2m   batched column-major GEMVs over stored operator blocks            HBM
//   m2l         all levels in one launch: target pivots x staged source pivots,
//               H0^(1) evaluated on the fly (never stored)                       fp64 ALU
//   l2l         batched GEMVs, coarse to fine                                      HBM
//   near        per leaf: P2P over N(leaf) with H0 on the fly + self term, fused
//               with L2P and the combine y = x + kappa^2 q phi, scattered back       fp64 ALU
// Every kernel works in H0 units; the (i/4) of G is applied once per target in `near`.
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "dafmm.h"
#include "device.h"

namespace dafmm {

namespace {

constexpr int kNearThreads = 256;
constexpr int kM2LThreads = 128;
constexpr int kStage = 512;  // staged source pivots / points per chunk (32 B each)
constexpr int kTB = 4;       // kernel entries evaluated in lockstep per thread (shared coefficients)

__device__ __forceinline__ double2 ld2(const double2* p) { return __ldg(p); }

// ---- gather: x_t[t] = x[perm[t]], v_t[t] = w_t[t] x_t[t] ----
__global__ void gather_kernel(int64_t n, const int32_t* __restrict__ perm, const double* __restrict__ w_t,
                              const double2* __restrict__ x, double2* __restrict__ x_t, double2* __restrict__ v_t) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    double2 xv = ld2(x + perm[t]);
    double w = w_t[t];
    x_t[t] = xv;
    v_t[t] = make_double2(w * xv.x, w * xv.y);
  }
}

// ---- batched translation: dst[dst_off + r] (+)= sum_terms Mat (rows x cols, col-major) src ----
// One warp per item; lanes own rows (coalesced column reads of the operator block).
__global__ void translate_kernel(int items, const int64_t* __restrict__ dst_off, const int32_t* __restrict__ dst_rows,
                                 const int32_t* __restrict__ term_ptr, const int64_t* __restrict__ mat_off,
                                 const int64_t* __restrict__ src_off, const int32_t* __restrict__ src_cols,
                                 const double2* __restrict__ ops, const double2* __restrict__ src,
                                 double2* __restrict__ dst, int accumulate) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (warp >= items) return;
  int rows = dst_rows[warp];
  int tb = term_ptr[warp], te = term_ptr[warp + 1];
  int64_t doff = dst_off[warp];
  for (int r0 = 0; r0 < rows; r0 += 32) {
    int r = r0 + lane;
    double ar = 0.0, ai = 0.0;
    for (int t = tb; t < te; ++t) {
      const double2* M = ops + mat_off[t];
      const double2* s = src + src_off[t];
      int cols = src_cols[t];
      if (r < rows) {
#pragma unroll 4
        for (int c = 0; c < cols; ++c) {
          double2 m = ld2(M + (int64_t)c * rows + r);
          double2 v = ld2(s + c);
          ar = fma(m.x, v.x, fma(-m.y, v.y, ar));
          ai = fma(m.x, v.y, fma(m.y, v.x, ai));
        }
      }
    }
    if (r < rows) {
      double2 o = make_double2(ar, ai);
      if (accumulate) {
        double2 p = dst[doff + r];
        o.x += p.x;
        o.y += p.y;
      }
      dst[doff + r] = o;
    }
  }
}

// Stage (x, y, value) of `take` consecutive sources into shared memory.
__device__ __forceinline__ void stage_sources(double4* sbuf, int fill, const double2* xy, const double2* val,
                                              int64_t off, int take) {
  for (int q = threadIdx.x; q < take; q += blockDim.x) {
    double2 p = ld2(xy + off + q);
    double2 v = ld2(val + off + q);
    sbuf[fill + q] = make_double4(p.x, p.y, v.x, v.y);
  }
}

// Source lists as CSR entries e -> (first source, count).
struct M2LSources {
  const int64_t* off;
  const int32_t* cnt;
  __device__ __forceinline__ int64_t first(int e) const { return off[e]; }
  __device__ __forceinline__ int count(int e) const { return cnt[e]; }
};
struct NearSources {
  const int32_t* begin;
  const int32_t* end;
  __device__ __forceinline__ int64_t first(int e) const { return begin[e]; }
  __device__ __forceinline__ int count(int e) const { return end[e] - begin[e]; }
};

// acc += sum over the source entries [e, pe) of H0_band(kappa |xt - s_j|) v_j.  Sources are
// staged through shared memory in chunks of kStage; thread (t, slice) takes every nsl-th
// staged source.  CTA-uniform (contains barriers): every thread calls it with the same
// arguments apart from xt / active / slice.  GUARD: the segment may contain the pair i == j
// (the own leaf of the near field), whose entry is excluded (its value is the self term D_i).
template <int CODE, bool GUARD, class Src>
__device__ __forceinline__ void accumulate(double4* sbuf, const Src& src, int e, int pe, const double2* __restrict__ xy,
                                           const double2* __restrict__ val, double2 xt, bool active, int slice,
                                           int nsl, double& ar, double& ai, const KernelConsts& kc,
                                           const Pair* logtab) {
  int kin = 0;
  while (e < pe) {
    int fill = 0;
    while (e < pe && fill < kStage) {
      int cnt = src.count(e);
      int take = min(cnt - kin, kStage - fill);
      stage_sources(sbuf, fill, xy, val, src.first(e) + kin, take);
      fill += take;
      kin += take;
      if (kin == cnt) {
        ++e;
        kin = 0;
      }
    }
    __syncthreads();
    if (active) {
      // kTB staged sources per step (j, j + nsl, ...), evaluated in lockstep; lanes past the
      // fill (and the i == j pair under GUARD) get a safe distance and a zero weight
      for (int j = slice; j < fill; j += kTB * nsl) {
        double r2[kTB], vr[kTB], vi[kTB], hr[kTB], hi[kTB];
#pragma unroll
        for (int b = 0; b < kTB; ++b) {
          const int jb = j + b * nsl;
          const bool ok = jb < fill;
          const double4 sv = sbuf[ok ? jb : j];
          const double dx = xt.x - sv.x, dy = xt.y - sv.y;
          const double d2 = fma(dx, dx, dy * dy);
          const bool use = ok && (!GUARD || d2 > 0.0);
          r2[b] = use ? d2 : kc.r2_safe;
          vr[b] = use ? sv.z : 0.0;
          vi[b] = use ? sv.w : 0.0;
        }
        h0_band_vec<CODE, kTB>(r2, hr, hi, kc, logtab);
#pragma unroll
        for (int b = 0; b < kTB; ++b) {
          ar = fma(hr[b], vr[b], fma(-hi[b], vi[b], ar));
          ai = fma(hr[b], vi[b], fma(hi[b], vr[b], ai));
        }
      }
    }
    __syncthreads();
  }
}

// Dispatch a CTA-uniform band code to its instantiation.
template <bool GUARD, class Src>
__device__ __forceinline__ void accumulate_code(int code, double4* sbuf, const Src& src, int e, int pe,
                                                const double2* __restrict__ xy, const double2* __restrict__ val,
                                                double2 xt, bool active, int slice, int nsl, double& ar, double& ai,
                                                const KernelConsts& kc, const Pair* logtab) {
#define DAFMM_BAND_CASE(C) \
  case C: accumulate<C, GUARD>(sbuf, src, e, pe, xy, val, xt, active, slice, nsl, ar, ai, kc, logtab); break;
  switch (code) {
    DAFMM_BAND_CASE(1)
    DAFMM_BAND_CASE(2)
    DAFMM_BAND_CASE(3)
    DAFMM_BAND_CASE(4)
    DAFMM_BAND_CASE(5)
    DAFMM_BAND_CASE(6)
    DAFMM_BAND_CASE(7)
    DAFMM_BAND_CASE(8)
    DAFMM_BAND_CASE(9)
    default: accumulate<kBandGeneric, GUARD>(sbuf, src, e, pe, xy, val, xt, active, slice, nsl, ar, ai, kc, logtab);
  }
#undef DAFMM_BAND_CASE
}
static_assert(kNumBandCodes == 10, "accumulate_code lists the band codes 1..9 explicitly");

// ---- M2L: u[t] = sum_{src nodes} sum_k H0(kappa |t - s_k|) m_k --------------------
// One CTA per target node; its source nodes come in band-uniform segments (items).
__global__ void __launch_bounds__(kM2LThreads) m2l_kernel(
    const int64_t* __restrict__ loc_off, const int32_t* __restrict__ rows, const int32_t* __restrict__ item_ptr,
    const int32_t* __restrict__ item_code, const int32_t* __restrict__ item_begin,
    const int32_t* __restrict__ item_end, const int64_t* __restrict__ src_off, const int32_t* __restrict__ src_cnt,
    const double2* __restrict__ ti_xy, const double2* __restrict__ so_xy, const double2* __restrict__ mult,
    double2* __restrict__ loc, KernelConsts kc) {
  __shared__ double4 sbuf[kStage];
  __shared__ double2 red[kM2LThreads];
  __shared__ Pair logtab[1 << dafmm_fit::LOG_BITS];
  load_log_table(logtab);
  const int tgt = blockIdx.x;
  const int r = rows[tgt];
  const int64_t lo = loc_off[tgt];
  const int is = item_ptr[tgt], ie = item_ptr[tgt + 1];
  const M2LSources src{src_off, src_cnt};
  for (int t0 = 0; t0 < r; t0 += kM2LThreads) {
    const int rc = min(kM2LThreads, r - t0);
    const int nsl = kM2LThreads / rc;
    const int t = threadIdx.x % rc;
    const int slice = threadIdx.x / rc;
    const bool active = slice < nsl;
    double2 xt = ld2(ti_xy + lo + t0 + t);
    double ar = 0.0, ai = 0.0;
    for (int it = is; it < ie; ++it)
      accumulate_code<false>(item_code[it], sbuf, src, item_begin[it], item_end[it], so_xy, mult, xt, active, slice,
                             nsl, ar, ai, kc, logtab);
    red[threadIdx.x] = make_double2(ar, ai);
    __syncthreads();
    if (threadIdx.x < rc) {
      double sr = 0.0, si = 0.0;
      for (int s = 0; s < nsl; ++s) {
        double2 v = red[threadIdx.x + s * rc];
        sr += v.x;
        si += v.y;
      }
      loc[lo + t0 + threadIdx.x] = make_double2(sr, si);
    }
    __syncthreads();
  }
}

// ---- near field + L2P + combine ------------------------------------------------
// phi_t = (i/4) [ sum_{j in N(leaf), j != t} H0 v_j + (U u)_t ] + D_t x_t
// y[perm[t]] = x_t + kappa^2 q_t phi_t   (kernel_mode 0)   or   phi_t   (kernel_mode 1)
// The leaf's own block is the first near entry (the only one with i == j pairs).
__global__ void __launch_bounds__(kNearThreads) near_kernel(
    const int32_t* __restrict__ leaf_begin, const int32_t* __restrict__ leaf_end, const int32_t* __restrict__ near_ptr,
    const int32_t* __restrict__ near_begin, const int32_t* __restrict__ near_end, const int32_t* __restrict__ leaf_band,
    const int64_t* __restrict__ leaf_loc_off, const int32_t* __restrict__ leaf_rank,
    const int64_t* __restrict__ leaf_U_off, const double2* __restrict__ ops, const double2* __restrict__ loc,
    const double2* __restrict__ pts_t, const double2* __restrict__ v_t, const double2* __restrict__ x_t,
    const double* __restrict__ qk2_t, const double2* __restrict__ D_t, const int32_t* __restrict__ perm,
    double2* __restrict__ y, KernelConsts kc, int kernel_mode, unsigned mask) {
  __shared__ double4 sbuf[kStage];
  __shared__ double2 red[kNearThreads];
  __shared__ Pair logtab[1 << dafmm_fit::LOG_BITS];
  load_log_table(logtab);
  const int leaf = blockIdx.x;
  const int tb = leaf_begin[leaf], m = leaf_end[leaf] - tb;
  const int ps = near_ptr[leaf], pe = near_ptr[leaf + 1];
  const bool do_near = mask & 1u, do_far = (mask & 2u) && leaf_loc_off[leaf] >= 0;
  const int band = leaf_band[leaf];
  const NearSources src{near_begin, near_end};
  for (int t0 = 0; t0 < m; t0 += kNearThreads) {
    const int rc = min(kNearThreads, m - t0);
    const int nsl = kNearThreads / rc;
    const int t = threadIdx.x % rc;
    const int slice = threadIdx.x / rc;
    const bool active = slice < nsl;
    double2 xt = ld2(pts_t + tb + t0 + t);
    double ar = 0.0, ai = 0.0;
    if (do_near && pe > ps) {
      if (band == kBandNear) {
        accumulate<kBandNear, true>(sbuf, src, ps, ps + 1, pts_t, v_t, xt, active, slice, nsl, ar, ai, kc, logtab);
        accumulate<kBandNear, false>(sbuf, src, ps + 1, pe, pts_t, v_t, xt, active, slice, nsl, ar, ai, kc, logtab);
      } else {
        accumulate<kBandGeneric, true>(sbuf, src, ps, ps + 1, pts_t, v_t, xt, active, slice, nsl, ar, ai, kc, logtab);
        accumulate<kBandGeneric, false>(sbuf, src, ps + 1, pe, pts_t, v_t, xt, active, slice, nsl, ar, ai, kc, logtab);
      }
    }
    red[threadIdx.x] = make_double2(ar, ai);
    __syncthreads();
    if (threadIdx.x < rc) {
      const int tt = t0 + threadIdx.x;
      double sr = 0.0, si = 0.0;
      for (int s = 0; s < nsl; ++s) {
        double2 v = red[threadIdx.x + s * rc];
        sr += v.x;
        si += v.y;
      }
      if (do_far) {  // L2P: (U u)_t, U column-major m x r
        const int rk = leaf_rank[leaf];
        const double2* U = ops + leaf_U_off[leaf];
        const double2* u = loc + leaf_loc_off[leaf];
        for (int c = 0; c < rk; ++c) {
          double2 a = ld2(U + (int64_t)c * m + tt);
          double2 b = ld2(u + c);
          sr = fma(a.x, b.x, fma(-a.y, b.y, sr));
          si = fma(a.x, b.y, fma(a.y, b.x, si));
        }
      }
      // phi = (i/4) (sr + i si) + D x
      double2 xv = x_t[tb + tt];
      double pr = -0.25 * si, pi = 0.25 * sr;
      if (do_near) {
        double2 d = D_t[tb + tt];
        pr = fma(d.x, xv.x, fma(-d.y, xv.y, pr));
        pi = fma(d.x, xv.y, fma(d.y, xv.x, pi));
      }
      double2 out;
      if (kernel_mode == 0) {
        double s = qk2_t[tb + tt];
        out = make_double2(s * pr, s * pi);
        if (do_near) {
          out.x += xv.x;
          out.y += xv.y;
        }
      } else {
        out = make_double2(pr, pi);
      }
      y[perm[tb + tt]] = out;
    }
    __syncthreads();
  }
}

// ---- GMRES vector kernels ----
constexpr int kVecThreads = 256;

__device__ __forceinline__ double2 block_sum2(double2 v, double2* sh) {
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, o);
    v.y += __shfl_down_sync(0xffffffffu, v.y, o);
  }
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double2 r = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      r.x += sh[i].x;
      r.y += sh[i].y;
    }
  }
  __syncthreads();
  return r;
}

// part[b * stride + i] = sum over the block's slice of conj(V_i) w, i < k
__global__ void multidot_kernel(int64_t n, int k, const double2* __restrict__ V, const double2* __restrict__ w,
                                double2* __restrict__ part, int stride) {
  __shared__ double2 sh[32];
  for (int i = 0; i < k; ++i) {
    const double2* v = V + (int64_t)i * n;
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
      double2 a = ld2(v + e), b = ld2(w + e);
      acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));
      acc.y = fma(a.x, b.y, fma(-a.y, b.x, acc.y));
    }
    double2 s = block_sum2(acc, sh);
    if (threadIdx.x == 0) part[(int64_t)blockIdx.x * stride + i] = s;
  }
}

// out[i] = sum_b part[b * stride + i]  (deterministic order)
__global__ void reduce_parts_kernel(int nblocks, int k, const double2* __restrict__ part, int stride,
                                    double2* __restrict__ out) {
  int i = threadIdx.x;
  if (i >= k) return;
  double sr = 0.0, si = 0.0;
  for (int b = 0; b < nblocks; ++b) {
    double2 v = part[(int64_t)b * stride + i];
    sr += v.x;
    si += v.y;
  }
  out[i] = make_double2(sr, si);
}

// w += sign * sum_{i<k} h_i V_i
__global__ void combine_kernel(int64_t n, int k, const double2* __restrict__ V, const double2* __restrict__ h,
                               double sign, double2* __restrict__ w) {
  __shared__ double2 hs[256];
  for (int i = threadIdx.x; i < k; i += blockDim.x) hs[i] = h[i];
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = w[e];
    for (int i = 0; i < k; ++i) {
      double2 v = ld2(V + (int64_t)i * n + e);
      double2 c = make_double2(sign * hs[i].x, sign * hs[i].y);
      acc.x = fma(c.x, v.x, fma(-c.y, v.y, acc.x));
      acc.y = fma(c.x, v.y, fma(c.y, v.x, acc.y));
    }
    w[e] = acc;
  }
}

// out = a * x + b * y   (a, b real)
__global__ void axpby_kernel(int64_t n, double a, const double2* __restrict__ x, double b, const double2* __restrict__ yv,
                             double2* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double2 p = ld2(x + e), q = ld2(yv + e);
    out[e] = make_double2(a * p.x + b * q.x, a * p.y + b * q.y);
  }
}

// part[b] = sum |w|^2 over the block's slice (in .x)
__global__ void norm2_kernel(int64_t n, const double2* __restrict__ w, double2* __restrict__ part) {
  __shared__ double2 sh[32];
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double2 a = ld2(w + e);
    acc.x = fma(a.x, a.x, fma(a.y, a.y, acc.x));
  }
  double2 s = block_sum2(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

int grid_for(int64_t n, int threads, int cap) {
  int64_t g = (n + threads - 1) / threads;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

bool ck(cudaError_t e, std::string& err, const char* what) {
  if (e == cudaSuccess) return true;
  err = std::string(what) + ": " + cudaGetErrorString(e);
  return false;
}

template <typename T>
bool upload(DevPlan& d, T** dst, const std::vector<T>& src, std::string& err) {
  *dst = nullptr;
  if (src.empty()) return true;
  size_t bytes = src.size() * sizeof(T);
  if (!ck(cudaMalloc((void**)dst, bytes), err, "cudaMalloc")) return false;
  d.allocations.push_back(*dst);
  d.device_bytes += bytes;
  return ck(cudaMemcpy(*dst, src.data(), bytes, cudaMemcpyHostToDevice), err, "cudaMemcpy H2D");
}

template <typename T>
bool alloc(DevPlan& d, T** dst, size_t count, std::string& err) {
  *dst = nullptr;
  if (count == 0) count = 1;
  if (!ck(cudaMalloc((void**)dst, count * sizeof(T)), err, "cudaMalloc")) return false;
  d.allocations.push_back(*dst);
  d.device_bytes += count * sizeof(T);
  return true;
}

bool upload_batch(DevPlan& d, DevBatch& b, const Packed::Batch& h, std::string& err) {
  b.items = (int)h.dst_off.size();
  return upload(d, &b.dst_off, h.dst_off, err) && upload(d, &b.dst_rows, h.dst_rows, err) &&
         upload(d, &b.term_ptr, h.term_ptr, err) && upload(d, &b.mat_off, h.mat_off, err) &&
         upload(d, &b.src_off, h.src_off, err) && upload(d, &b.src_cols, h.src_cols, err);
}

int launch_translate(const DevPlan& d, const DevBatch& b, const double2* src, double2* dst, int accumulate) {
  if (b.items == 0) return 0;
  int threads = 256;
  int blocks = (b.items * 32 + threads - 1) / threads;
  translate_kernel<<<blocks, threads, 0, d.stream>>>(b.items, b.dst_off, b.dst_rows, b.term_ptr, b.mat_off, b.src_off,
                                                     b.src_cols, d.ops, src, dst, accumulate);
  return 1;
}

}  // namespace

int upload_plan(const Packed& pk, const Plan& plan, DevPlan& d, std::string& err) {
  d.n = plan.n;
  d.kernel_mode = plan.opt.kernel_mode;
  d.kc = make_kernel_consts(plan.kappa);
  std::vector<double2> pts(plan.n), D(plan.n);
  for (int64_t t = 0; t < plan.n; ++t) {
    pts[t] = make_double2(pk.pts_t[2 * t], pk.pts_t[2 * t + 1]);
    D[t] = make_double2(pk.D_t[t].re, pk.D_t[t].im);
  }
  std::vector<double2> so(pk.n_mult), ti(pk.n_loc);
  for (int64_t k = 0; k < pk.n_mult; ++k) so[k] = make_double2(pk.so_xy[2 * k], pk.so_xy[2 * k + 1]);
  for (int64_t k = 0; k < pk.n_loc; ++k) ti[k] = make_double2(pk.ti_xy[2 * k], pk.ti_xy[2 * k + 1]);
  std::vector<double2> ops(pk.ops.size());
  for (size_t k = 0; k < pk.ops.size(); ++k) ops[k] = make_double2(pk.ops[k].re, pk.ops[k].im);
  d.n_mult = pk.n_mult;
  d.n_loc = pk.n_loc;
  d.ops_len = (int64_t)ops.size();
  bool ok = upload(d, &d.pts_t, pts, err) && upload(d, &d.w_t, pk.w_t, err) && upload(d, &d.qk2_t, pk.qk2_t, err) &&
            upload(d, &d.D_t, D, err) && upload(d, &d.perm, pk.perm, err) && upload(d, &d.so_xy, so, err) &&
            upload(d, &d.ti_xy, ti, err) && upload(d, &d.ops, ops, err) && upload_batch(d, d.p2m, pk.p2m, err);
  d.m2m.assign(pk.m2m.size(), DevBatch());
  for (size_t i = 0; ok && i < pk.m2m.size(); ++i) ok = upload_batch(d, d.m2m[i], pk.m2m[i], err);
  d.l2l.assign(pk.l2l.size(), DevBatch());
  for (size_t i = 0; ok && i < pk.l2l.size(); ++i) ok = upload_batch(d, d.l2l[i], pk.l2l[i], err);
  d.m2l_targets = (int)pk.m2l_loc_off.size();
  ok = ok && upload(d, &d.m2l_loc_off, pk.m2l_loc_off, err) && upload(d, &d.m2l_rows, pk.m2l_rows, err) &&
       upload(d, &d.m2l_src_ptr, pk.m2l_src_ptr, err) && upload(d, &d.m2l_src_off, pk.m2l_src_off, err) &&
       upload(d, &d.m2l_src_cnt, pk.m2l_src_cnt, err) && upload(d, &d.m2l_item_ptr, pk.m2l_item_ptr, err) &&
       upload(d, &d.m2l_item_code, pk.m2l_item_code, err) && upload(d, &d.m2l_item_begin, pk.m2l_item_begin, err) &&
       upload(d, &d.m2l_item_end, pk.m2l_item_end, err);
  d.nleaves = (int)pk.leaf_begin.size();
  d.max_leaf = pk.max_leaf;
  ok = ok && upload(d, &d.leaf_begin, pk.leaf_begin, err) && upload(d, &d.leaf_end, pk.leaf_end, err) &&
       upload(d, &d.near_ptr, pk.near_ptr, err) && upload(d, &d.near_begin, pk.near_begin, err) &&
       upload(d, &d.near_end, pk.near_end, err) && upload(d, &d.leaf_loc_off, pk.leaf_loc_off, err) &&
       upload(d, &d.leaf_rank, pk.leaf_rank, err) && upload(d, &d.leaf_U_off, pk.leaf_U_off, err) &&
       upload(d, &d.leaf_band, pk.leaf_band, err);
  ok = ok && alloc(d, &d.x_t, plan.n, err) && alloc(d, &d.v_t, plan.n, err) && alloc(d, &d.mult, pk.n_mult, err) &&
       alloc(d, &d.loc, pk.n_loc, err) && alloc(d, &d.host_stage, 2 * plan.n, err);
  if (!ok) return DAFMM_ECUDA;
  return DAFMM_OK;
}

void free_plan(DevPlan& d) {
  for (auto& e : d.prof_ev)
    if (e) {
      cudaEventDestroy(e);
      e = nullptr;
    }
  for (void* p : d.allocations) cudaFree(p);
  d.allocations.clear();
  if (d.gm_hostbuf) cudaFreeHost(d.gm_hostbuf);
  d.gm_hostbuf = nullptr;
}

int set_profiling(DevPlan& d, bool on, std::string& err) {
  if (on && !d.prof_ev[0])
    for (auto& e : d.prof_ev)
      if (!ck(cudaEventCreate(&e), err, "cudaEventCreate")) return DAFMM_ECUDA;
  d.prof = on;
  d.prof_pending = false;
  for (double& v : d.prof_ms) v = 0.0;
  d.prof_count = 0;
  d.launches = 0;
  return DAFMM_OK;
}

int harvest_profile(DevPlan& d, std::string& err) {
  if (!d.prof_pending) return DAFMM_OK;
  if (!ck(cudaEventSynchronize(d.prof_ev[kNumPasses]), err, "profile event sync")) return DAFMM_ECUDA;
  for (int p = 0; p < kNumPasses; ++p) {
    float ms = 0.f;
    if (!ck(cudaEventElapsedTime(&ms, d.prof_ev[p], d.prof_ev[p + 1]), err, "profile elapsed")) return DAFMM_ECUDA;
    d.prof_ms[p] += ms;
  }
  ++d.prof_count;
  d.prof_pending = false;
  return DAFMM_OK;
}

int run_matvec(DevPlan& d, const double2* x, double2* y, unsigned mask, std::string& err) {
  cudaStream_t s = d.stream;
  if (d.prof && harvest_profile(d, err) != DAFMM_OK) return DAFMM_ECUDA;
  // profiling marks: event p is recorded before pass p (p = 0..5) and event 6 after the last
  auto mark = [&](int p) {
    if (d.prof) cudaEventRecord(d.prof_ev[p], s);
  };
  mark(0);
  gather_kernel<<<grid_for(d.n, 256, 148 * 16), 256, 0, s>>>(d.n, d.perm, d.w_t, x, d.x_t, d.v_t);
  ++d.launches;
  const bool far = (mask & 2u) && d.n_mult > 0;
  if (far) {
    cudaMemsetAsync(d.mult, 0, sizeof(double2) * d.n_mult, s);
    cudaMemsetAsync(d.loc, 0, sizeof(double2) * d.n_loc, s);
  }
  mark(1);
  if (far) d.launches += launch_translate(d, d.p2m, d.v_t, d.mult, 0);  // P2M
  mark(2);
  if (far)
    for (auto& b : d.m2m) d.launches += launch_translate(d, b, d.mult, d.mult, 0);  // M2M
  mark(3);
  if (far && d.m2l_targets > 0) {  // M2L
    m2l_kernel<<<d.m2l_targets, kM2LThreads, 0, s>>>(d.m2l_loc_off, d.m2l_rows, d.m2l_item_ptr, d.m2l_item_code,
                                                      d.m2l_item_begin, d.m2l_item_end, d.m2l_src_off,
                                                      d.m2l_src_cnt, d.ti_xy, d.so_xy, d.mult, d.loc, d.kc);
    ++d.launches;
  }
  mark(4);
  if (far)
    for (auto& b : d.l2l) d.launches += launch_translate(d, b, d.loc, d.loc, 1);  // L2L
  mark(5);
  near_kernel<<<d.nleaves, kNearThreads, 0, s>>>(d.leaf_begin, d.leaf_end, d.near_ptr, d.near_begin, d.near_end,
                                                 d.leaf_band, d.leaf_loc_off, d.leaf_rank, d.leaf_U_off, d.ops, d.loc, d.pts_t,
                                                 d.v_t, d.x_t, d.qk2_t, d.D_t, d.perm, y, d.kc, d.kernel_mode,
                                                 far ? mask : (mask & 1u));
  ++d.launches;
  mark(6);
  if (d.prof) d.prof_pending = true;
  return ck(cudaGetLastError(), err, "matvec launch") ? DAFMM_OK : DAFMM_ECUDA;
}

// ============================================================================================
// Restarted GMRES (reading R14) with CGS2 orthogonalisation on the device.
int run_gmres(DevPlan& d, const double2* f, double2* psi, double tol, int maxit, int restart, int* iters_out,
              double* relres_out, double* history, std::string& err) {
  const int64_t n = d.n;
  const int m = restart > 0 ? restart : 50;
  if (m > 255) { err = "restart must be <= 255"; return DAFMM_EINVAL; }
  cudaStream_t s = d.stream;
  const int nb = grid_for(n, kVecThreads, 296);
  if (d.gm_restart != m) {
    if (d.gm_V) { err = "GMRES workspace already sized for another restart"; return DAFMM_EINVAL; }
    d.gm_restart = m;
    if (!alloc(d, &d.gm_V, (size_t)(m + 1) * n, err) || !alloc(d, &d.gm_w, n, err) || !alloc(d, &d.gm_r, n, err) ||
        !alloc(d, &d.gm_h, 3 * (m + 2), err) || !alloc(d, &d.gm_part, (size_t)nb * (m + 2), err))
      return DAFMM_ECUDA;
    if (!ck(cudaMallocHost((void**)&d.gm_hostbuf, sizeof(double2) * 3 * (m + 2)), err, "cudaMallocHost"))
      return DAFMM_ECUDA;
    d.gm_part_blocks = nb;
  }
  const int stride = m + 2;
  auto norm = [&](const double2* v, double& out) -> bool {
    norm2_kernel<<<nb, kVecThreads, 0, s>>>(n, v, d.gm_part);
    reduce_parts_kernel<<<1, 32, 0, s>>>(nb, 1, d.gm_part, 1, d.gm_h);
    if (!ck(cudaMemcpyAsync(d.gm_hostbuf, d.gm_h, sizeof(double2), cudaMemcpyDeviceToHost, s), err, "D2H") ||
        !ck(cudaStreamSynchronize(s), err, "sync"))
      return false;
    out = std::sqrt(d.gm_hostbuf[0]);
    return true;
  };
  double bnorm;
  if (!norm(f, bnorm)) return DAFMM_ECUDA;
  cudaMemsetAsync(psi, 0, sizeof(double2) * n, s);
  if (history) history[0] = 1.0;
  if (bnorm == 0.0) {
    *iters_out = 0;
    *relres_out = 0.0;
    return DAFMM_OK;
  }
  std::vector<std::complex<double>> H((size_t)(m + 1) * m), g(m + 1), sn(m);
  std::vector<double> cs(m);
  int iters = 0;
  bool converged = false;
  // r = f (psi0 = 0)
  cudaMemcpyAsync(d.gm_r, f, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s);
  while (iters < maxit && !converged) {
    double beta;
    if (!norm(d.gm_r, beta)) return DAFMM_ECUDA;
    if (beta / bnorm <= tol) { converged = true; break; }
    axpby_kernel<<<nb, kVecThreads, 0, s>>>(n, 1.0 / beta, d.gm_r, 0.0, d.gm_r, d.gm_V);
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int k = 0;
    for (int j = 0; j < m; ++j) {
      double2* vj = d.gm_V + (int64_t)j * n;
      double2* vj1 = d.gm_V + (int64_t)(j + 1) * n;
      if (run_matvec(d, vj, d.gm_w, 3u, err) != DAFMM_OK) return DAFMM_ECUDA;
      ++iters;
      // CGS2: two passes of h = V^H w, w -= V h
      for (int pass = 0; pass < 2; ++pass) {
        multidot_kernel<<<nb, kVecThreads, 0, s>>>(n, j + 1, d.gm_V, d.gm_w, d.gm_part, stride);
        reduce_parts_kernel<<<1, 256, 0, s>>>(nb, j + 1, d.gm_part, stride, d.gm_h + pass * (m + 2));
        combine_kernel<<<nb, kVecThreads, 0, s>>>(n, j + 1, d.gm_V, d.gm_h + pass * (m + 2), -1.0, d.gm_w);
      }
      norm2_kernel<<<nb, kVecThreads, 0, s>>>(n, d.gm_w, d.gm_part);
      reduce_parts_kernel<<<1, 32, 0, s>>>(nb, 1, d.gm_part, 1, d.gm_h + 2 * (m + 2));
      if (!ck(cudaMemcpyAsync(d.gm_hostbuf, d.gm_h, sizeof(double2) * (2 * (m + 2) + 1), cudaMemcpyDeviceToHost, s),
              err, "D2H") ||
          !ck(cudaStreamSynchronize(s), err, "sync"))
        return DAFMM_ECUDA;
      const double* hb = d.gm_hostbuf;
      for (int i = 0; i <= j; ++i)
        H[(size_t)i * m + j] = std::complex<double>(hb[2 * i] + hb[2 * ((m + 2) + i)], hb[2 * i + 1] + hb[2 * ((m + 2) + i) + 1]);
      double hnext = std::sqrt(hb[2 * 2 * (m + 2)]);
      H[(size_t)(j + 1) * m + j] = hnext;
      if (hnext != 0.0) axpby_kernel<<<nb, kVecThreads, 0, s>>>(n, 1.0 / hnext, d.gm_w, 0.0, d.gm_w, vj1);
      for (int i = 0; i < j; ++i) {
        std::complex<double> a = H[(size_t)i * m + j], b = H[(size_t)(i + 1) * m + j];
        H[(size_t)i * m + j] = cs[i] * a + sn[i] * b;
        H[(size_t)(i + 1) * m + j] = -std::conj(sn[i]) * a + cs[i] * b;
      }
      std::complex<double> a = H[(size_t)j * m + j], b = H[(size_t)(j + 1) * m + j];
      double c;
      std::complex<double> sg;
      if (b == 0.0) { c = 1.0; sg = 0.0; }
      else if (a == 0.0) { c = 0.0; sg = 1.0; }
      else {
        double rho = std::sqrt(std::norm(a) + std::norm(b));
        c = std::abs(a) / rho;
        sg = (a / std::abs(a)) * std::conj(b) / rho;
      }
      cs[j] = c;
      sn[j] = sg;
      H[(size_t)j * m + j] = c * a + sg * b;
      H[(size_t)(j + 1) * m + j] = 0.0;
      g[j + 1] = -std::conj(sg) * g[j];
      g[j] = c * g[j];
      k = j + 1;
      double res = std::abs(g[j + 1]) / bnorm;
      if (history) history[iters] = res;
      if (res <= tol) { converged = true; break; }
      if (iters >= maxit || hnext == 0.0) break;
    }
    // y = H^{-1} g, psi += V y
    std::vector<std::complex<double>> yv(k);
    for (int i = k - 1; i >= 0; --i) {
      std::complex<double> acc = g[i];
      for (int t = i + 1; t < k; ++t) acc -= H[(size_t)i * m + t] * yv[t];
      yv[i] = acc / H[(size_t)i * m + i];
    }
    std::vector<double2> yh(k);
    for (int i = 0; i < k; ++i) yh[i] = make_double2(yv[i].real(), yv[i].imag());
    cudaMemcpyAsync(d.gm_h, yh.data(), sizeof(double2) * k, cudaMemcpyHostToDevice, s);
    combine_kernel<<<nb, kVecThreads, 0, s>>>(n, k, d.gm_V, d.gm_h, 1.0, psi);
    // r = f - A psi
    if (run_matvec(d, psi, d.gm_w, 3u, err) != DAFMM_OK) return DAFMM_ECUDA;
    axpby_kernel<<<nb, kVecThreads, 0, s>>>(n, 1.0, f, -1.0, d.gm_w, d.gm_r);
    if (!ck(cudaStreamSynchronize(s), err, "sync")) return DAFMM_ECUDA;
  }
  double rn;
  if (!norm(d.gm_r, rn)) return DAFMM_ECUDA;  // gm_r = f - A psi of the final iterate
  *iters_out = iters;
  *relres_out = rn / bnorm;
  return converged ? DAFMM_OK : DAFMM_NOT_CONVERGED;
}

}  // namespace dafmm
