// sm_100a kernels of the DAFMM matvec and the GMRES vector work.
//
// Passes per matvec:
//   gather      x (caller order) -> x_t, v_t = w o x_t (tree order)                 HBM
//   p2m / m2m   batched GEMVs over column-major operator blocks (formed on the device
//               at create, setup_device.cu), a lane per output row
//               (translate_cm_kernel), one launch per level                        HBM
//   m2l         all levels in one persistent launch.  Default (m2l_store = -1 -> 1):
//               the kernel-entry blocks A_{t s}, evaluated once at create by
//               m2l_form_kernel, streamed from HBM by TMA bulk copies
//               (m2l_stored_kernel); m2l_store = 2: one block per node pair applied
//               as row and column sums by warp pairs (m2l_pairw_kernel, R22);
//               m2l_store = 0: entries
//               evaluated on the fly every matvec (m2l_kernel)                    HBM / fp64 ALU
//   l2l         batched GEMVs, coarse to fine                                      HBM
//   p2p         per leaf: near field with H0 on the fly (side stream, concurrent
//               with p2m..l2l); symmetric pairs evaluated once (column sums)       fp64 ALU
//   combine     L2P + near-field slots + self term + y = x + kappa^2 q phi, scattered
//               back to caller order                                               HBM
// Every kernel works in H0 units; the (i/4) of G is applied once per target in `combine`.
// GMRES (run_gmres): CGS2 multi-dot / combine / norm kernels, host Givens, optional right
// preconditioner (the HODLR of hodlr.cu, reading HR4).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <string>
#include <cstdio>
#include <cstring>
#include <vector>

#include "dafmm.h"
#include "device.h"
#include "setup_device.h"

namespace dafmm {

namespace {

constexpr int kNearThreads = 256;
#ifndef DAFMM_M2L_THREADS
#define DAFMM_M2L_THREADS 128
#endif
#ifndef DAFMM_M2L_STAGE
#define DAFMM_M2L_STAGE 320
#endif
#ifndef DAFMM_BANDS_CONST
#define DAFMM_BANDS_CONST 0
#endif
constexpr int kM2LThreads = DAFMM_M2L_THREADS;
constexpr int kM2LStage = DAFMM_M2L_STAGE;  // M2L: staged source pivots per chunk (32 B each, double-buffered)
constexpr int kNearStage = 320;  // near field: staged source points per chunk
constexpr int kCombineThreads = 64;
// kernel entries evaluated in lockstep per thread (each coefficient shared by TB FMAs); measured
// best: 8 for P2P, 4 for M2L (whose far-type evaluator needs more registers per entry)
#ifndef DAFMM_TB_P2P
#define DAFMM_TB_P2P 8
#endif
#ifndef DAFMM_TB_M2L
#define DAFMM_TB_M2L 4
#endif
constexpr int kTBP2P = DAFMM_TB_P2P;
constexpr int kTBM2L = DAFMM_TB_M2L;

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

// ---- batched translation (P2M, M2M, L2L): dst[dst_off + r] (+)= sum_c M[r][c] s_c -------------
// One warp per item.  The item's operator is one row-major block (its terms side by side), so
// every row is a contiguous run: the lanes first gather the item's sources for columns
// c = lane + 32 k (k < kTCK) into registers, then each row is one coalesced pass over the
// row (all 32 lanes busy) and a warp reduction.  Items wider than 32 kTCK columns are handled
// in column blocks.  HBM-bound: every operator element is read once per matvec.
#ifndef DAFMM_TCK
#define DAFMM_TCK 4
#endif
constexpr int kTCK = DAFMM_TCK;  // source columns per lane per pass (32 kTCK columns per pass)
#ifndef DAFMM_TRB
#define DAFMM_TRB 2  // with DAFMM_TCK 4: measured best (profiles/README.md, r34 and r36)
#endif
constexpr int kTRB = DAFMM_TRB;  // rows per step in translate_kernel
__global__ void translate_kernel(int items, const int64_t* __restrict__ dst_off, const int32_t* __restrict__ dst_rows,
                                 const int64_t* __restrict__ item_mat_off, const int32_t* __restrict__ item_cols,
                                 const int32_t* __restrict__ term_ptr, const int64_t* __restrict__ src_off,
                                 const int32_t* __restrict__ src_cols, const double2* __restrict__ ops,
                                 const double2* __restrict__ src, double2* __restrict__ dst, int accumulate) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= items) return;
  const int R = dst_rows[warp], C = item_cols[warp];
  const int tb = term_ptr[warp], te = term_ptr[warp + 1];
  const int64_t doff = dst_off[warp];
  const double2* M = ops + item_mat_off[warp];
  for (int cb = 0; cb < C; cb += 32 * kTCK) {
    double2 v[kTCK];
#pragma unroll
    for (int k = 0; k < kTCK; ++k) v[k] = make_double2(0.0, 0.0);
    int cs = 0;
    for (int t = tb; t < te; ++t) {  // sources of the columns this lane holds
      const int ce = cs + src_cols[t];
      if (ce > cb && cs < cb + 32 * kTCK) {
        const double2* sv = src + src_off[t] - cs;
#pragma unroll
        for (int k = 0; k < kTCK; ++k) {
          const int c = cb + lane + 32 * k;
          if (c >= cs && c < ce) v[k] = ld2(sv + c);
        }
      }
      cs = ce;
    }
    const int kmax = min(kTCK, (C - cb + 31) / 32);
    // kTRB rows per step: their loads are all in flight together and their warp reductions
    // interleave (one row at a time left the warp waiting on each shuffle tree)
    for (int r0 = 0; r0 < R; r0 += kTRB) {
      double ar[kTRB], ai[kTRB];
#pragma unroll
      for (int q = 0; q < kTRB; ++q) ar[q] = ai[q] = 0.0;
#pragma unroll
      for (int q = 0; q < kTRB; ++q) {
        if (r0 + q < R) {
          const double2* row = M + (int64_t)(r0 + q) * C + cb + lane;
#pragma unroll
          for (int k = 0; k < kTCK; ++k) {
            if (k < kmax && cb + lane + 32 * k < C) {
              const double2 m = ld2(row + 32 * k);
              ar[q] = fma(m.x, v[k].x, fma(-m.y, v[k].y, ar[q]));
              ai[q] = fma(m.x, v[k].y, fma(m.y, v[k].x, ai[q]));
            }
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int q = 0; q < kTRB; ++q) {
          ar[q] += __shfl_xor_sync(0xffffffffu, ar[q], o);
          ai[q] += __shfl_xor_sync(0xffffffffu, ai[q], o);
        }
      }
#pragma unroll
      for (int q = 0; q < kTRB; ++q) {
        if (lane == q && r0 + q < R) {
          double2 o = make_double2(ar[q], ai[q]);
          if (accumulate || cb > 0) {
            const double2 p = dst[doff + r0 + q];
            o.x += p.x;
            o.y += p.y;
          }
          dst[doff + r0 + q] = o;
        }
      }
    }
  }
}

// Narrow items (few columns, e.g. directional L2L with 2 parent cones): a group of g = 32 / ipw
// lanes per item (ipw items per warp, g >= the batch's largest row count when ipw > 1), lanes own
// rows and walk their contiguous row, 4 columns per step into 4 accumulators.
__global__ void translate_rows_kernel(int items, const int64_t* __restrict__ dst_off,
                                      const int32_t* __restrict__ dst_rows, const int64_t* __restrict__ item_mat_off,
                                      const int32_t* __restrict__ item_cols, const int32_t* __restrict__ term_ptr,
                                      const int64_t* __restrict__ src_off, const int32_t* __restrict__ src_cols,
                                      const double2* __restrict__ ops, const double2* __restrict__ src,
                                      double2* __restrict__ dst, int accumulate, int ipw) {
  const int g = 32 / ipw;
  const int lane = (threadIdx.x & 31) % g;
  const int item = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * ipw + (threadIdx.x & 31) / g;
  if (item >= items) return;
  const int R = dst_rows[item], C = item_cols[item];
  const int tb = term_ptr[item], te = term_ptr[item + 1];
  const int64_t doff = dst_off[item];
  const int warp = item;
  for (int r = lane; r < R; r += g) {
    const double2* row = ops + item_mat_off[warp] + (int64_t)r * C;
    double ar[4] = {0.0, 0.0, 0.0, 0.0}, ai[4] = {0.0, 0.0, 0.0, 0.0};
    int cs = 0;
    for (int t = tb; t < te; ++t) {
      const int n = src_cols[t];
      const double2* sv = src + src_off[t];
      const double2* m = row + cs;
      int c = 0;
      for (; c + 4 <= n; c += 4) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 a = ld2(m + c + q), b = ld2(sv + c + q);
          ar[q] = fma(a.x, b.x, fma(-a.y, b.y, ar[q]));
          ai[q] = fma(a.x, b.y, fma(a.y, b.x, ai[q]));
        }
      }
      for (; c < n; ++c) {
        const double2 a = ld2(m + c), b = ld2(sv + c);
        ar[0] = fma(a.x, b.x, fma(-a.y, b.y, ar[0]));
        ai[0] = fma(a.x, b.y, fma(a.y, b.x, ai[0]));
      }
      cs += n;
    }
    double2 o = make_double2((ar[0] + ar[1]) + (ar[2] + ar[3]), (ai[0] + ai[1]) + (ai[2] + ai[3]));
    if (accumulate) {
      const double2 p = dst[doff + r];
      o.x += p.x;
      o.y += p.y;
    }
    dst[doff + r] = o;
  }
}

// Column-major items (the default layout): entry (r, c) of the item at item_mat_off + c R + r.
// One warp per item, one lane per output row (row blocks of 32 when R > 32): each step reads one
// column of the operator as one coalesced run of R entries, eight columns in flight per lane, and
// the lane accumulates its own row, so there is no cross-lane reduction at all.  The sources of
// up to kTCMCols columns are staged in shared memory per warp and read as broadcasts.
constexpr int kTCMCols = 128;
constexpr int kTCMWarps = 8;
// GROUPS (batches whose items have at most 16 rows, i.e. the directional levels): the warp splits
// into G = 32 / P2 lane groups (P2 = the power of two >= R), group j takes the columns c = j (mod G)
// and the groups' partial rows are added at the end (one xor-shuffle tree per item, fixed order),
// so the small nodes still keep 32 lanes' worth of loads in flight.  Without GROUPS (48 registers
// instead of 64) every lane owns a row; measured per batch shape in profiles/README.md (r2w).
template <bool GROUPS>
__global__ void __launch_bounds__(32 * kTCMWarps) translate_cm_kernel(
    int items, const int64_t* __restrict__ dst_off, const int32_t* __restrict__ dst_rows,
    const int64_t* __restrict__ item_mat_off, const int32_t* __restrict__ item_cols,
    const int32_t* __restrict__ term_ptr, const int64_t* __restrict__ src_off, const int32_t* __restrict__ src_cols,
    const double2* __restrict__ ops, const double2* __restrict__ src, double2* __restrict__ dst, int accumulate) {
  __shared__ __align__(16) double2 xs_all[kTCMWarps][kTCMCols];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * kTCMWarps + w;
  if (item >= items) return;
  double2* xs = xs_all[w];
  const int R = dst_rows[item], C = item_cols[item];
  const int tb = term_ptr[item], te = term_ptr[item + 1];
  const int64_t doff = dst_off[item];
  const double2* M = ops + item_mat_off[item];
  int lg = 5;
  if (GROUPS) {
    lg = 0;
    while ((1 << lg) < min(R, 32)) ++lg;
  }
  const int P2 = 1 << lg, G = 32 >> lg, tl = lane & (P2 - 1), j = lane >> lg;
  for (int rb = 0; rb < R; rb += P2) {
    const int t = rb + tl;
    const bool act = t < R;
    double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
    for (int cb = 0; cb < C; cb += kTCMCols) {
      __syncwarp();
      int cs = 0;
      for (int q = tb; q < te; ++q) {  // stage the sources of columns [cb, cb + kTCMCols)
        const int ce = cs + src_cols[q];
        const int c0 = max(cs, cb), c1 = min(ce, cb + kTCMCols);
        if (c0 < c1) {
          const double2* sv = src + src_off[q] - cs;
          for (int c = c0 + lane; c < c1; c += 32) xs[c - cb] = ld2(sv + c);
        }
        cs = ce;
      }
      __syncwarp();
      if (act) {
        const int nc = min(kTCMCols, C - cb);
        const int64_t step = (int64_t)G * R;
        const double2* p = M + (int64_t)(cb + j) * R + t;
        int c = j;
        for (; c + 7 * G < nc; c += 8 * G, p += 8 * step) {
          double2 m[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) m[q] = ld2(p + q * step);
#pragma unroll
          for (int q = 0; q < 8; q += 2) {
            const double2 v0 = xs[c + q * G], v1 = xs[c + (q + 1) * G];
            ar = fma(m[q].x, v0.x, fma(-m[q].y, v0.y, ar));
            ai = fma(m[q].x, v0.y, fma(m[q].y, v0.x, ai));
            br = fma(m[q + 1].x, v1.x, fma(-m[q + 1].y, v1.y, br));
            bi = fma(m[q + 1].x, v1.y, fma(m[q + 1].y, v1.x, bi));
          }
        }
        for (; c < nc; c += G, p += step) {
          const double2 mm = ld2(p), v0 = xs[c];
          ar = fma(mm.x, v0.x, fma(-mm.y, v0.y, ar));
          ai = fma(mm.x, v0.y, fma(mm.y, v0.x, ai));
        }
      }
    }
    ar += br;
    ai += bi;
    if (GROUPS)
      for (int o = P2; o < 32; o <<= 1) {  // add the groups' partial rows
        ar += __shfl_xor_sync(0xffffffffu, ar, o);
        ai += __shfl_xor_sync(0xffffffffu, ai, o);
      }
    if (act && j == 0) {
      double2 o = make_double2(ar, ai);
      if (accumulate) {
        const double2 pv = dst[doff + t];
        o.x += pv.x;
        o.y += pv.y;
      }
      dst[doff + t] = o;
    }
  }
}

// ---- source streams ----------------------------------------------------------------------------
// P2P and M2L share one engine: a CTA owns a set of targets (the points of a leaf or the pivots
// of a node, one per thread "t", with nsl source slices) and a stream of sources given as a CSR
// list of contiguous runs (entry e -> (first, count)).  The stream is staged through shared
// memory in double-buffered chunks with cp.async (x, y, value: 32 B per source) while the
// previous chunk is consumed; the stream is cut into band-uniform items [pb, pe) (stream
// offsets) whose band code is CTA-uniform, so every inner loop is one templated evaluator.

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Stagers: copy the next chunk of a CTA's source stream into shared memory (asynchronous, one
// cp.async commit group per call; returns the number of sources staged, 0 at the end).
// IndexStager: the M2L stream is a flat list of multipole slots (idx), so every thread finds
// its source directly.  RunStager: the near-field stream is a few runs of consecutive points
// (the neighbour leaves), walked with a cursor that every thread advances identically.
template <int STAGE, int NT>
struct IndexStager {
  // idx of the chunk after the one being staged is prefetched into registers one chunk ahead,
  // so issuing its copies never waits on the index load
  static constexpr int kSlots = (STAGE + NT - 1) / NT;
  const int32_t* idx;
  int64_t base;
  int total;
  const double2* xy;
  const double2* val;
  int kreg[kSlots];
  __device__ __forceinline__ void prefetch(int c0) {
#pragma unroll
    for (int s = 0; s < kSlots; ++s) {
      const int q = threadIdx.x + s * NT;
      kreg[s] = (q < STAGE && c0 + q < total) ? __ldg(idx + base + c0 + q) : 0;
    }
  }
  __device__ __forceinline__ int issue(double4* buf, int c0) {
    const int fill = max(0, min(STAGE, total - c0));
#pragma unroll
    for (int s = 0; s < kSlots; ++s) {
      const int q = threadIdx.x + s * NT;
      if (q < fill) {
        double2* d = reinterpret_cast<double2*>(buf + q);
        cp_async16(d, xy + kreg[s]);
        cp_async16(d + 1, val + kreg[s]);
      }
    }
    cp_async_commit();
    return fill;
  }
  template <int S>
  __device__ __forceinline__ int first(double4* buf) {
    prefetch(0);
    const int fill = issue(buf, 0);
    prefetch(fill);
    return fill;
  }
  template <int S>
  __device__ __forceinline__ int next(double4* buf, int c0) {
    const int fill = issue(buf, c0);  // indices prefetched during the previous chunk
    prefetch(c0 + fill);
    return fill;
  }
};
struct RunStager {
  const int32_t* begin;
  const int32_t* end;
  int e, kin, pe;
  const double2* xy;
  const double2* val;
  template <int STAGE>
  __device__ __forceinline__ int stage(double4* buf, int) {
    int fill = 0;
    while (e < pe && fill < STAGE) {
      const int first = begin[e], cnt = end[e] - first;
      const int take = min(cnt - kin, STAGE - fill);
      const int64_t off = (int64_t)first + kin;
      for (int q = threadIdx.x; q < take; q += blockDim.x) {
        double2* d = reinterpret_cast<double2*>(buf + fill + q);
        cp_async16(d, xy + off + q);
        cp_async16(d + 1, val + off + q);
      }
      fill += take;
      kin += take;
      if (kin == cnt) {
        ++e;
        kin = 0;
      }
    }
    cp_async_commit();
    return fill;
  }
  template <int S>
  __device__ __forceinline__ int first(double4* buf) {
    return stage<S>(buf, 0);
  }
  template <int S>
  __device__ __forceinline__ int next(double4* buf, int c0) {
    return stage<S>(buf, c0);
  }
};

// Items of an M2L target: band code and stream range, from the packed plan.
// COLS (symmetric near field): the block's column sums sum_t H0(|x_t - s_q|) v_t over the
// warp's 32 targets are written to cs.slots[cs.base + pos + q] (one warp-half of the slots).
struct ColSink {
  double2* slots;
  int64_t base;
  double2 vt;  // this thread's target weight w_t x_t
};
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// Reduce N values per lane (N a power of 2, <= 32) over the warp's 32 lanes, reduce-scatter
// style: each halving step exchanges half of the values, N - 1 shuffles in all (instead of
// 5 N).  Returns the full sum of value index (lane >> (5 - log2 N)) & (N - 1)... for N = 16:
// value (lane >> 1), held by lanes 2k and 2k + 1.
template <int N>
__device__ __forceinline__ double warp_reduce_scatter(double* v) {
  const int lane = threadIdx.x & 31;
  int o = 16;
#pragma unroll
  for (int n = N; n > 1; n >>= 1, o >>= 1) {
    const bool up = lane & o;
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const double send = up ? v[i] : v[i + n / 2];
      const double keep = up ? v[i + n / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  double r = v[0];
#pragma unroll
  for (; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  return r;
}
struct M2LItems {
  static constexpr int kTB = kTBM2L;
  static constexpr bool kGuarded = false;  // no i == j pairs
  static constexpr bool kNearOnly = false;
  static constexpr bool kCols = false;
  const int4* it_;  // (code, pb, pe, -) in shared memory: read once per chunk by every thread
  int is, ie;
  __device__ __forceinline__ int code(int i) const { return it_[i].x; }
  __device__ __forceinline__ bool guard(int) const { return false; }
  __device__ __forceinline__ int pb(int i) const { return it_[i].y; }
  __device__ __forceinline__ int pe(int i) const { return it_[i].z; }
};
// Items of a near-field leaf: its own block [0, own) (contains i == j) and the rest.
struct NearItems {
  static constexpr int kTB = kTBP2P;
  static constexpr bool kGuarded = true;   // item 0 holds the i == j pairs
  static constexpr bool kNearOnly = true;  // bands: near-7, near-8, near-12 or generic
  static constexpr bool kCols = true;      // item 1 of a symmetric near field writes column sums
  int band, own, total, is, ie;
  int sym;
  double2* slots;     // this warp-half's slots
  int64_t slot_base;  // slot of stream position `own`
  double2 vt;
  __device__ __forceinline__ bool cols(int i) const { return sym && i == 1; }
  __device__ __forceinline__ ColSink sink(int c0) const { return ColSink{slots, slot_base - own + c0, vt}; }
  __device__ __forceinline__ int code(int) const { return band; }
  __device__ __forceinline__ bool guard(int i) const { return i == 0; }
  __device__ __forceinline__ int pb(int i) const { return i == 0 ? 0 : own; }
  __device__ __forceinline__ int pe(int i) const { return i == 0 ? own : total; }
};

// Band evaluator by code (compile time): generic, near 8, near 12, or a data band.
template <int CODE, int TB>
__device__ __forceinline__ void eval_band(const double* z2, double* re, double* im, const PolyTable& T,
                                          const FarBand* band) {
  if constexpr (CODE == kBandGeneric) h0_generic_vec<TB>(z2, re, im, T);
  else if constexpr (CODE == kBandNear8) h0_near_vec<8, TB>(z2, re, im, T);
  else if constexpr (CODE == kBandNear7) h0_near_vec<7, TB>(z2, re, im, T);
  else if constexpr (CODE == kBandNear12) h0_near_vec<12, TB>(z2, re, im, T);
  else h0_far_vec<TB>(z2, re, im, band->A, band->B, DataFarPQ<TB>{band}, T);
}

// One lockstep block of kTB staged sources p[0], p[stride], ...: acc += sum_q H0(|xt - s_q|) v_q.
// MASK: only the first `valid` sources count (tail block); GUARD: the pair i == j (own leaf of
// the near field; its value is the self term D_i) is excluded.  Excluded lanes get a safe z^2
// and a zero weight so the evaluator stays branch-free.
template <int CODE, int TB, bool GUARD, bool MASK, bool COLS = false>
__device__ __forceinline__ void consume_block(const double4* p, int stride, int valid, double2 xt, double& ar, double& ai,
                                              const PolyTable& T, const FarBand* band, const ColSink& cs = {}, int pos = 0) {
  if constexpr (CODE == kBandGeneric) {  // rare (straddling segments): one lane at a time
#pragma unroll 1
    for (int q = 0; q < (MASK ? valid : TB); ++q) {
      const double4 sv = p[q * stride];
      const double dx = xt.x - sv.x, dy = xt.y - sv.y;
      const double d2 = fma(dx, dx, dy * dy);
      if (GUARD && !(d2 > 0.0)) continue;
      double hr, hi;
      h0_generic_vec<1>(&d2, &hr, &hi, T);
      ar = fma(hr, sv.z, fma(-hi, sv.w, ar));
      ai = fma(hr, sv.w, fma(hi, sv.z, ai));
      if constexpr (COLS) {
        const double cr = warp_sum(fma(hr, cs.vt.x, -hi * cs.vt.y));
        const double ci = warp_sum(fma(hr, cs.vt.y, hi * cs.vt.x));
        if ((threadIdx.x & 31) == 0) cs.slots[cs.base + pos + q] = make_double2(cr, ci);
      }
    }
  } else {
  double z2[TB], hr[TB], hi[TB];
  bool use[TB];
#pragma unroll
  for (int q = 0; q < TB; ++q) {
    const bool ok = !MASK || q < valid;
    const double2 sp = *reinterpret_cast<const double2*>(p + ((MASK && !ok) ? 0 : q * stride));
    const double dx = xt.x - sp.x, dy = xt.y - sp.y;
    const double d2 = fma(dx, dx, dy * dy);
    use[q] = ok && (!GUARD || d2 > 0.0);
    z2[q] = (MASK || GUARD) ? (use[q] ? d2 : kZ2Safe) : d2;
  }
  eval_band<CODE, TB>(z2, hr, hi, T, band);
  // the weights are re-read from shared memory after the evaluation (not held in registers
  // across it: the evaluator needs every register it can get)
#pragma unroll
  for (int q = 0; q < TB; ++q) {
    double2 v = reinterpret_cast<const double2*>(p + ((MASK && q >= valid) ? 0 : q * stride))[1];
    if (MASK || GUARD) {
      v.x = use[q] ? v.x : 0.0;
      v.y = use[q] ? v.y : 0.0;
    }
    ar = fma(hr[q], v.x, fma(-hi[q], v.y, ar));
    ai = fma(hr[q], v.y, fma(hi[q], v.x, ai));
  }
  if constexpr (COLS) {  // the pairs' other direction: column sums over the warp's targets
    static_assert(2 * TB == 16, "the column reduce-scatter is written for 8 sources per block");
    double c[2 * TB];
#pragma unroll
    for (int q = 0; q < TB; ++q) {
      const bool u = !MASK || q < valid;
      c[2 * q] = u ? fma(hr[q], cs.vt.x, -hi[q] * cs.vt.y) : 0.0;
      c[2 * q + 1] = u ? fma(hr[q], cs.vt.y, hi[q] * cs.vt.x) : 0.0;
    }
    const double r = warp_reduce_scatter<2 * TB>(c);
    const int lane = threadIdx.x & 31, idx = lane >> 1, q = idx >> 1;
    if (!(lane & 1) && (!MASK || q < valid))
      reinterpret_cast<double*>(cs.slots + cs.base + pos + q)[idx & 1] = r;
  }
  }
}

// acc += sum_{j in [a, b)} H0(|xt - s_j|) v_j over staged sources (kappa-scaled coordinates).
// The range is cut into blocks of kTB consecutive sources, dealt to the slices cyclically
// (block k to slice k mod nsl); only the last block of the range can be partial (masked).
template <int CODE, int TB, bool GUARD, bool COLS = false>
__device__ __forceinline__ void consume(const double4* sb, int a, int b, double2 xt, int slice, int nsl, double& ar,
                                        double& ai, const PolyTable& T, const FarBand* band, const ColSink& cs = {}) {
  const int n = b - a;
  const int full = n / TB;
  for (int k = slice; k < full; k += nsl)
    consume_block<CODE, TB, GUARD, false, COLS>(sb + a + k * TB, 1, TB, xt, ar, ai, T, band, cs, a + k * TB);
  if ((n % TB) && slice == full % nsl)
    consume_block<CODE, TB, GUARD, true, COLS>(sb + a + full * TB, 1, n % TB, xt, ar, ai, T, band, cs, a + full * TB);
}

// Dispatch a CTA-uniform band code.  NEAR_ONLY (the P2P stream): only the near bands and generic
// occur, so no other band is instantiated (code size: the kernel stays in the i-cache).
template <int TB, bool GUARD, bool NEAR_ONLY, bool COLS = false>
__device__ __forceinline__ void consume_code(int code, const double4* sb, int a, int b, double2 xt, int slice, int nsl,
                                             double& ar, double& ai, const PolyTable& T, const FarBand* bands,
                                             const ColSink& cs = {}) {
  if constexpr (NEAR_ONLY) {
    if (code == kBandNear7) consume<kBandNear7, TB, GUARD, COLS>(sb, a, b, xt, slice, nsl, ar, ai, T, bands, cs);
    else if (code == kBandNear8) consume<kBandNear8, TB, GUARD, COLS>(sb, a, b, xt, slice, nsl, ar, ai, T, bands, cs);
    else if (code == kBandNear12) consume<kBandNear12, TB, GUARD, COLS>(sb, a, b, xt, slice, nsl, ar, ai, T, bands, cs);
    else consume<kBandGeneric, TB, GUARD, COLS>(sb, a, b, xt, slice, nsl, ar, ai, T, bands, cs);
  } else {
    switch (code) {  // the M2L stream: choose_band(.., allow_near7 = false) never yields near-7
      case kBandNear8:
        consume<kBandNear8, TB, GUARD>(sb, a, b, xt, slice, nsl, ar, ai, T, bands);
        break;
      case kBandNear12:
        consume<kBandNear12, TB, GUARD>(sb, a, b, xt, slice, nsl, ar, ai, T, bands);
        break;
      case kBandGeneric:
        consume<kBandGeneric, TB, GUARD>(sb, a, b, xt, slice, nsl, ar, ai, T, bands);
        break;
      default:
        consume<kBandFarData, TB, GUARD>(sb, a, b, xt, slice, nsl, ar, ai, T, bands + (code - kBandFarData));
    }
  }
}

// Run a CTA over one source stream (stager `st`, items of `items`).  CTA-uniform (barriers);
// `buf` holds 2 x STAGE double4: the next chunk is staged while the current one is consumed.
// Ends with a barrier.
template <int STAGE, class Stager, class Items>
__device__ __forceinline__ void stream_accumulate(double4* buf, Stager& st, const Items& items, double2 xt, bool active,
                                                  int slice, int nsl, double& ar, double& ai, const PolyTable& T,
                                                  const FarBand* bands) {
  int c0 = 0, which = 0, it0 = items.is;
  int fill = st.template first<STAGE>(buf);
  while (fill > 0) {
    cp_async_wait_all();
    __syncthreads();  // chunk `which` visible to all; everyone is done with the other buffer
    const int next = st.template next<STAGE>(buf + (which ^ 1) * STAGE, c0 + fill);
    const int c1 = c0 + fill;
    while (it0 < items.ie && items.pe(it0) <= c0) ++it0;
    if (active) {
      const double4* sb = buf + which * STAGE;
      for (int it = it0; it < items.ie && items.pb(it) < c1; ++it) {
        const int a = max(items.pb(it), c0) - c0, b = min(items.pe(it), c1) - c0;
        if (Items::kGuarded && items.guard(it))
          consume_code<Items::kTB, Items::kGuarded, Items::kNearOnly>(items.code(it), sb, a, b, xt, slice, nsl, ar,
                                                                      ai, T, bands);
        else {
          bool done = false;
          if constexpr (Items::kCols) {
            if (items.cols(it)) {  // symmetric near field: the column sums too
              consume_code<Items::kTB, false, Items::kNearOnly, true>(items.code(it), sb, a, b, xt, slice, nsl, ar, ai,
                                                                      T, bands, items.sink(c0));
              done = true;
            }
          }
          if (!done)
            consume_code<Items::kTB, false, Items::kNearOnly>(items.code(it), sb, a, b, xt, slice, nsl, ar, ai, T,
                                                              bands);
        }
      }
    }
    c0 = c1;
    fill = next;
    which ^= 1;
  }
  __syncthreads();
}

// ---- M2L: u[t] = sum_{src nodes} sum_k H0(kappa |t - s_k|) m_k --------------------
// One CTA per target node; its source stream is cut into band-uniform items.
#ifndef DAFMM_M2L_MINB
#define DAFMM_M2L_MINB 6
#endif
__global__ void __launch_bounds__(kM2LThreads, DAFMM_M2L_MINB) m2l_kernel(
    int ntargets, int* __restrict__ ticket, const int64_t* __restrict__ loc_off, const int32_t* __restrict__ rows,
    const int64_t* __restrict__ stream_ptr, const int32_t* __restrict__ stream_idx, const int32_t* __restrict__ item_ptr,
    const int32_t* __restrict__ item_code, const int32_t* __restrict__ item_pb, const int32_t* __restrict__ item_pe,
    const double2* __restrict__ ti_xy, const double2* __restrict__ so_xy,
    const double2* __restrict__ mult, double2* __restrict__ loc) {
  __shared__ __align__(16) double4 buf[2 * kM2LStage];
  __shared__ double2 red[kM2LThreads];
  __shared__ PolyTable T;
#if DAFMM_BANDS_CONST
  const FarBand* bands = dafmm_fit::kFarBandsDev;  // uniform constant-bank loads per coefficient pair
#else
  __shared__ FarBand bands[dafmm_fit::NUM_FAR];
#endif
  __shared__ int4 sitems[kNumBandCodes];
  __shared__ int next;
  load_poly_table(T);
#if !DAFMM_BANDS_CONST
  load_far_bands(bands);
#endif
  // persistent CTAs take target nodes from a ticket counter (targets are packed by
  // decreasing cost, so the dynamic order balances the tail)
  while (true) {
    if (threadIdx.x == 0) next = atomicAdd(ticket, 1);
    __syncthreads();
    const int tgt = next;
    __syncthreads();
    if (tgt >= ntargets) break;
    const int r = rows[tgt];
    const int64_t lo = loc_off[tgt];
    // the target's items (at most kNumBandCodes) into shared memory
    const int i0 = item_ptr[tgt], ni = item_ptr[tgt + 1] - i0;
    for (int i = threadIdx.x; i < ni; i += blockDim.x)
      sitems[i] = make_int4(item_code[i0 + i], item_pb[i0 + i], item_pe[i0 + i], 0);
    __syncthreads();
    const M2LItems items{sitems, 0, ni};
    for (int t0 = 0; t0 < r; t0 += kM2LThreads) {
      const int rc = min(kM2LThreads, r - t0);
      const int nsl = kM2LThreads / rc;
      const int t = threadIdx.x % rc;
      const int slice = threadIdx.x / rc;
      const bool active = slice < nsl;
      double2 xt = ld2(ti_xy + lo + t0 + t);
      double ar = 0.0, ai = 0.0;
      IndexStager<kM2LStage, kM2LThreads> st{stream_idx, stream_ptr[tgt], (int)(stream_ptr[tgt + 1] - stream_ptr[tgt]),
                                              so_xy, mult, {}};
      stream_accumulate<kM2LStage>(buf, st, items, xt, active, slice, nsl, ar, ai, T, bands);
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
}

// ---- stored M2L blocks (dafmm_options.m2l_store) ------------------------------------------
// The M2L operator of a target node is the block A_{t s} of kernel entries between its
// incoming pivots t and the outgoing pivots s of every node in its interaction lists (
// the kappa^2 q and w scalings are folded into the stored operators and multipoles, so the block
// is pure H0).  It depends only on the plan, so it can be evaluated once and kept in HBM: the
// matvec then streams 16 B per entry instead of evaluating ~100 fp64 flops per entry, and the
// M2L turns from fp64-ALU bound into HBM bound -- the other resource than the concurrent P2P's.
//
// Layout: per target node (r rows, L source columns in its source-stream order), column-major:
// entry (t, s) at m2l_mat_off[target] + s * r + t.  A CTA whose threads are mapped as
// (row t, slice sl) with nsl = floor(NT / r) slices, thread j = sl * r + t, touches entries
// e = j + k * nsl * r: one contiguous run per step, and every thread keeps one row.
//
constexpr int kMSConsumers = 128;  // consumer threads (4 warps); a node may have at most this many rows
constexpr int kMSThreads = kMSConsumers + 32;  // + one producer warp (one elected lane issues TMA)
#ifndef DAFMM_MS_STAGES
#define DAFMM_MS_STAGES 4
#endif
#ifndef DAFMM_MS_COLS
#define DAFMM_MS_COLS 512
#endif
#ifndef DAFMM_LEAF_SPLIT
#define DAFMM_LEAF_SPLIT 0  // 1: the deepest level's M2L on its own stream from the end of P2M
#endif
#ifndef DAFMM_M2M_SIDE
#define DAFMM_M2M_SIDE 0  // 1: M2M on a third stream beside the deepest level's stored M2L (flag handshake); measured slower at C4, C5 (profiles/README.md, r2p)
#endif
#ifndef DAFMM_NEAR_AFTER
#define DAFMM_NEAR_AFTER -1  // P2P held back until P2M (1) / M2M (2) has finished, never (0), or per plan (-1)
#endif
#ifndef DAFMM_NEAR_HIGH
#define DAFMM_NEAR_HIGH 0  // 1: the near-field stream gets the high priority instead of the far field
#endif
#ifndef DAFMM_MS_PER_SM
#define DAFMM_MS_PER_SM 2  // persistent stored-M2L CTAs per SM (they share the SMs with P2P CTAs)
#endif
#ifndef DAFMM_MS_MINB
#define DAFMM_MS_MINB 6  // register cap (<= 64): room for P2P CTAs beside the stored-M2L CTAs
#endif
#ifndef DAFMM_MS_STAGE_E
#define DAFMM_MS_STAGE_E 1024
#endif
constexpr int kMSStageE = DAFMM_MS_STAGE_E;     // entries per TMA bulk copy (16 KB)
constexpr int kMSStages = DAFMM_MS_STAGES;      // ring depth (x 16 KB in flight per CTA)
constexpr int kMSCols = DAFMM_MS_COLS;          // source columns per work unit (multipoles double-buffered)
constexpr int kMaxStoredRows = kMSConsumers;
constexpr int kMSFormThreads = 128;
constexpr size_t kMSDynSmem = sizeof(double2) * kMSStages * kMSStageE;

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
// wait until the phase with parity `parity` of barrier b has completed.  The suspend-time hint
// lets the waiting warp sleep until the phase completes (woken by the barrier) instead of
// re-polling: spinning waiters would take issue slots from the P2P warps sharing the SM.
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_addr(b)), "r"(parity), "r"(0x989680u)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__global__ void set_flag_kernel(int* flag) {
  __threadfence();
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(flag), "r"(1) : "memory");
}
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kMSConsumers) : "memory"); }
// TMA 1-D bulk copy global -> shared, completion counted in bytes on barrier b
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(b))
               : "memory");
}

// Evaluate the blocks once (at create time): one CTA per target node.
__global__ void __launch_bounds__(kMSFormThreads) m2l_form_kernel(const int64_t* __restrict__ loc_off,
                                                                const int32_t* __restrict__ rows,
                                                                const int64_t* __restrict__ stream_ptr,
                                                                const int32_t* __restrict__ stream_idx,
                                                                const int64_t* __restrict__ mat_off,
                                                                const double2* __restrict__ ti_xy,
                                                                const double2* __restrict__ so_xy,
                                                                double2* __restrict__ mat) {
  __shared__ PolyTable T;
  load_poly_table(T);
  const int tgt = blockIdx.x;
  const int r = rows[tgt];
  if (r <= 0) return;
  const int nsl = kMSFormThreads / r, t = threadIdx.x % r, sl = threadIdx.x / r;
  if (sl >= nsl) return;
  const double2 xt = ld2(ti_xy + loc_off[tgt] + t);
  const int64_t sp = stream_ptr[tgt];
  const int L = (int)(stream_ptr[tgt + 1] - sp);
  double2* M = mat + mat_off[tgt];
  for (int c = sl; c < L; c += nsl) {
    const double2 sv = ld2(so_xy + stream_idx[sp + c]);
    const double dx = xt.x - sv.x, dy = xt.y - sv.y;
    const double d2 = fma(dx, dx, dy * dy);
    double hr, hi;
    h0_generic_vec<1>(&d2, &hr, &hi, T);
    M[(int64_t)c * r + t] = make_double2(hr, hi);
  }
}

// Apply the stored blocks: u[t] = sum_s A_{t s} m_s.  Persistent CTAs; CTA b takes target nodes
// b, b + G, b + 2G, ... (packed by decreasing work).  Warp-specialised: one lane of the producer
// warp cuts each node into work units of at most kMSCols source columns, publishes the unit
// descriptors one unit ahead (a kMSUnits-slot ring), and streams each unit's entries through a
// kMSStages-deep ring of shared-memory stages with TMA bulk copies (mbarrier full/empty
// handshakes).  The 4 consumer warps accumulate their row over the staged entries; while they
// consume unit i they gather unit i+1's multipoles into the other half of a double buffer with
// cp.async (indices loaded one stage earlier), so the gather latency hides behind the stream.
// At a node's last unit the slices of each row are reduced and u is written.
struct MSUnit {
  int tgt, c0, c1, flags;  // flags: 1 first unit of the node, 2 last; tgt < 0: no more work
  int r, pad;              // the node's rows
  int64_t sp, lo;          // its source stream offset and output offset
};
constexpr int kMSUnits = 4;
constexpr int kMSIdx = kMSCols / kMSConsumers;  // multipole indices per consumer thread per unit
__global__ void __launch_bounds__(kMSThreads, DAFMM_MS_MINB) m2l_stored_kernel(
    int ntargets, const int64_t* __restrict__ loc_off, const int32_t* __restrict__ rows,
    const int64_t* __restrict__ stream_ptr, const int32_t* __restrict__ stream_idx,
    const int64_t* __restrict__ mat_off, const double2* __restrict__ mat, const double2* __restrict__ mult,
    double2* __restrict__ loc, int nfree, const int* __restrict__ upper_ready) {
  extern __shared__ __align__(128) double2 ms_dyn[];  // the TMA ring: kMSStages x kMSStageE entries
  double2(*ring)[kMSStageE] = reinterpret_cast<double2(*)[kMSStageE]>(ms_dyn);
  __shared__ __align__(16) double2 mb[2][kMSCols];
  __shared__ double2 red[kMSConsumers];
  __shared__ __align__(8) uint64_t full[kMSStages], empty[kMSStages], ufull[kMSUnits], uempty[kMSUnits];
  __shared__ MSUnit units[kMSUnits];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kMSStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kMSConsumers / 32);
    }
    for (int i = 0; i < kMSUnits; ++i) {
      mbar_init(&ufull[i], 1);
      mbar_init(&uempty[i], kMSConsumers / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == kMSConsumers / 32) {  // ---- producer
    if (lane != 0) return;
    int stage = 0, uslot = 0;
    uint32_t sphase = 0, uphase = 0;
    // the unit sequence: (tgt, c0, c1); next_unit() advances it, fetching tickets as needed
    // static schedule: this CTA's nodes are blockIdx.x + k gridDim.x (the list is sorted by
    // decreasing work, so round-robin balances to within one node); the metadata of node k+1
    // is loaded while node k streams (independent addresses: the loads do not stall the lane)
    int tgt = -2, L = 0, c0 = 0, r = 0;
    int64_t sp = 0, lo = 0, moff = 0;
    int ntgt = blockIdx.x, nr = 0;
    int64_t nsp = 0, nsp1 = 0, nlo = 0, nmoff = 0;
    bool waited = false;
    auto prefetch_node = [&]() {
      if (ntgt < ntargets) {
        nr = rows[ntgt];
        nsp = stream_ptr[ntgt];
        nsp1 = stream_ptr[ntgt + 1];
        nlo = loc_off[ntgt];
        nmoff = mat_off[ntgt];
      }
    };
    prefetch_node();
    auto next_unit = [&](MSUnit& u) {
      if (tgt == -1) {
        u = MSUnit{-1, 0, 0, 0, 0, 0, 0, 0};
        return;
      }
      if (tgt == -2 || c0 >= L) {  // next node
        if (ntgt >= ntargets) {
          tgt = -1;
          u = MSUnit{-1, 0, 0, 0, 0, 0, 0, 0};
          return;
        }
        tgt = ntgt;
        r = nr;
        sp = nsp;
        L = (int)(nsp1 - nsp);
        lo = nlo;
        moff = nmoff;
        c0 = 0;
        ntgt += gridDim.x;
        prefetch_node();
        // targets [nfree, ntargets) read multipoles that M2M writes on another stream while this
        // kernel works through the deepest level's targets: wait for its flag before the first of
        // them is published (the consumers gather a unit's multipoles only after its descriptor)
        if (tgt >= nfree && upper_ready != nullptr && !waited) {
          // (bounded: a flag that never comes is a scheduling bug; trap instead of hanging)
          for (int64_t spins = 0; ld_acquire_gpu(upper_ready) == 0; ++spins) {
            __nanosleep(256);
            if (spins > (int64_t)1 << 24) __trap();
          }
          waited = true;
        }
      }
      const int c1 = min(L, c0 + kMSCols);
      u = MSUnit{tgt, c0, c1, (c0 == 0 ? 1 : 0) | (c1 >= L ? 2 : 0), r, 0, sp, lo};
      c0 = c1;
    };
    auto publish = [&](const MSUnit& u) {
      mbar_wait(&uempty[uslot], uphase ^ 1);
      units[uslot] = u;
      mbar_arrive(&ufull[uslot]);
      if (++uslot == kMSUnits) {
        uslot = 0;
        uphase ^= 1;
      }
    };
    MSUnit cur, nxt;
    next_unit(cur);
    int64_t cur_moff = moff;
    publish(cur);
    while (cur.tgt >= 0) {
      next_unit(nxt);
      const int64_t nxt_moff = moff;
      publish(nxt);  // one unit ahead: the consumers prefetch its multipoles
      const double2* src = mat + cur_moff + (int64_t)cur.c0 * cur.r;
      const int ne = (cur.c1 - cur.c0) * cur.r;
      for (int e0 = 0; e0 < ne; e0 += kMSStageE) {
        const int cnt = min(kMSStageE, ne - e0);
        mbar_wait(&empty[stage], sphase ^ 1);
        mbar_arrive_tx(&full[stage], (uint32_t)cnt * 16u);
        bulk_load(ring[stage], src + e0, (uint32_t)cnt * 16u, &full[stage]);
        if (++stage == kMSStages) {
          stage = 0;
          sphase ^= 1;
        }
      }
      cur = nxt;
      cur_moff = nxt_moff;
    }
    return;
  }
  // ---- consumers (threads 0 .. kMSConsumers-1)
  const int j = threadIdx.x;
  int stage = 0, uslot = 0;
  uint32_t sphase = 0, uphase = 0;
  auto take = [&]() {
    mbar_wait(&ufull[uslot], uphase);
    const MSUnit u = units[uslot];
    __syncwarp();
    if (lane == 0) mbar_arrive(&uempty[uslot]);
    if (++uslot == kMSUnits) {
      uslot = 0;
      uphase ^= 1;
    }
    return u;
  };
  auto gather_idx = [&](const MSUnit& u, int* kidx) {
    const int64_t sp = u.sp + u.c0;
#pragma unroll
    for (int k = 0; k < kMSIdx; ++k) {
      const int c = j + k * kMSConsumers;
      kidx[k] = (u.tgt >= 0 && c < u.c1 - u.c0) ? __ldg(stream_idx + sp + c) : -1;
    }
  };
  auto gather_issue = [&](const int* kidx, double2* dst) {
#pragma unroll
    for (int k = 0; k < kMSIdx; ++k)
      if (kidx[k] >= 0) cp_async16(dst + j + k * kMSConsumers, mult + kidx[k]);
    cp_async_commit();
  };
  int nsl = 0, P = 1, buf = 0, sl = 0;
  bool act = false;
  double ar0 = 0.0, ai0 = 0.0, ar1 = 0.0, ai1 = 0.0;
  int kidx[kMSIdx];
  MSUnit u = take();
  gather_idx(u, kidx);
  gather_issue(kidx, mb[0]);
  while (u.tgt >= 0) {
    const MSUnit un = take();  // published before u's stages were issued
    gather_idx(un, kidx);      // in flight while the first half of u is consumed
    const int r = u.r;
    if (u.flags & 1) {
      nsl = r > 0 ? kMSConsumers / r : 0;
      P = max(1, nsl * r);
      sl = r > 0 ? j / r : 0;
      act = j < P;
      ar0 = ai0 = ar1 = ai1 = 0.0;
    }
    cp_async_wait_all();
    consumers_sync();  // u's multipoles (mb[buf]) complete; everyone is done with mb[buf ^ 1]
    const double2* mv = mb[buf];
    const int ne = (u.c1 - u.c0) * r;
    const int nst = (ne + kMSStageE - 1) / kMSStageE;
    // this thread's entries in the unit: e = j + k P (row t = j mod r, column c = sl + k nsl);
    // e and c run on across the stages
    int e = j, c = sl;
    for (int st = 0; st < nst; ++st) {
      const int e0 = st * kMSStageE, e1 = min(ne, e0 + kMSStageE);
      mbar_wait(&full[stage], sphase);
      if (act) {
        const double2* R = ring[stage] - e0;
        for (; e + 3 * P < e1; e += 4 * P, c += 4 * nsl) {
          const double2 m0 = R[e], v0 = mv[c];
          const double2 m1 = R[e + P], v1 = mv[c + nsl];
          const double2 m2 = R[e + 2 * P], v2 = mv[c + 2 * nsl];
          const double2 m3 = R[e + 3 * P], v3 = mv[c + 3 * nsl];
          ar0 = fma(m0.x, v0.x, fma(-m0.y, v0.y, ar0));
          ai0 = fma(m0.x, v0.y, fma(m0.y, v0.x, ai0));
          ar1 = fma(m1.x, v1.x, fma(-m1.y, v1.y, ar1));
          ai1 = fma(m1.x, v1.y, fma(m1.y, v1.x, ai1));
          ar0 = fma(m2.x, v2.x, fma(-m2.y, v2.y, ar0));
          ai0 = fma(m2.x, v2.y, fma(m2.y, v2.x, ai0));
          ar1 = fma(m3.x, v3.x, fma(-m3.y, v3.y, ar1));
          ai1 = fma(m3.x, v3.y, fma(m3.y, v3.x, ai1));
        }
        for (; e < e1; e += P, c += nsl) {
          const double2 m0 = R[e], v0 = mv[c];
          ar0 = fma(m0.x, v0.x, fma(-m0.y, v0.y, ar0));
          ai0 = fma(m0.x, v0.y, fma(m0.y, v0.x, ai0));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == kMSStages) {
        stage = 0;
        sphase ^= 1;
      }
      if (st == nst / 2) gather_issue(kidx, mb[buf ^ 1]);  // next unit's multipoles (indices have landed)
    }
    if (nst == 0) gather_issue(kidx, mb[buf ^ 1]);
    if (u.flags & 2) {  // reduce the slices of each row, write u
      red[j] = make_double2(ar0 + ar1, ai0 + ai1);
      consumers_sync();
      if (j < r) {
        double sr = 0.0, si = 0.0;
        for (int q = j; q < P; q += r) {
          sr += red[q].x;
          si += red[q].y;
        }
        loc[u.lo + j] = make_double2(sr, si);
      }
    }
    u = un;
    buf ^= 1;
  }
  cp_async_wait_all();
}

// ---- pair-stored M2L (reading R22, dafmm_options.m2l_store = 2) ---------------------------------
// With one skeleton per node (R19: s^{B,o} = t^{B,i}) the block of (B <- A) is the transpose of
// the block of (A <- B), G being symmetric, so each unordered interaction-list pair
// keeps one block, in the stream of its owner B.  The owner applies it twice per matvec:
//   row sums     u_B[t] += sum_c M[t, c] m_A[c]         (as m2l_stored_kernel)
//   column sums  slot[c] = sum_t M[t, c] m_B[t]          (u_A's share; added by m2l_slot_gather)
// so the HBM stream is half that of m2l_stored_kernel for the same work.  (A CTA-wide version --
// the stored kernel's ring with whole-column stages, 8 consumer warps doing both passes between
// CTA barriers -- took 3.9 ms at C4 against 2.15 ms for the warp pairs below.)
// The kernel: warp pairs.
// Every pair of warps is an independent worker: it owns whole nodes (node g, g + G, ... of the
// list sorted by decreasing work, G = warp pairs in the grid) and streams their blocks through
// its own kPWStages-deep ring of stages, with no CTA-level barrier, so the workers of an SM
// drift apart and one worker's wait is covered by the others' arithmetic.  A stage holds whole
// columns (at most 32 and at most kPWStageE entries), the multipoles of those columns and, for
// r <= 32, the owner's own multipole.  The two warps read every stage once each:
//   row warp     lane = row t:            acc_t  += sum_c M[t, c] m_A[c]   (kept in registers over
//                the node's stages, written at its last stage)
//   column warp  lane = (column, part i): slot_c  = sum_t M[t, c] m_B[t]   (rows visited from a
//                per-column rotation when r would otherwise put the lanes on few banks; parts
//                xor-shuffle reduced)
// The row warp also drives the ring: its lane 0 issues the TMA bulk copy of a stage's entries, and
// one step later (when the stage's column indices have landed in registers) its lanes gather the
// multipoles with cp.async; both complete on the stage's `full` mbarrier (1 expect_tx arrival + 32
// cp.async.mbarrier.arrive.noinc arrivals), which both warps wait on.  A slot is refilled when both
// warps have arrived on its `empty` mbarrier.
#ifndef DAFMM_PW_RINGS
#define DAFMM_PW_RINGS 6  // warp pairs per CTA
#endif
#ifndef DAFMM_PW_STAGES
#define DAFMM_PW_STAGES 3
#endif
#ifndef DAFMM_PW_STAGE_E
#define DAFMM_PW_STAGE_E 512
#endif
#ifndef DAFMM_PW_PER_SM
#define DAFMM_PW_PER_SM 1
#endif
#ifndef DAFMM_PW_SPIN
#define DAFMM_PW_SPIN 0
#endif
#ifndef DAFMM_PW_UNROLL4
#define DAFMM_PW_UNROLL4 0
#endif
#ifndef DAFMM_PW_MAXREG
#define DAFMM_PW_MAXREG 64  // 6 rings x 64 threads x 64 registers: two P2P CTAs fit beside the CTA
#endif
constexpr int kPWRings = DAFMM_PW_RINGS;
constexpr int kPWThreads = 64 * kPWRings;
constexpr int kPWStages = DAFMM_PW_STAGES;
constexpr int kPWStageE = DAFMM_PW_STAGE_E;
static_assert(kPWStageE >= kMaxStoredRows, "a stage holds at least one whole column");
static_assert(kPWStages >= 2, "ring depth");
struct PWStage {
  double2 ent[kPWStageE];  // whole columns of the block, column-major
  double2 mv[32];          // multipoles of the stage's columns
  double2 ms[32];          // the owner's own multipole (r <= 32)
};
struct PWDesc {
  int r, ncs, flags, lg;  // flags: 1 first stage of the node, 2 last; r < 0: no more work;
  int rot, pad;           // column pass: 2^lg lanes per column, row rotation per column
  int64_t lo, spc, sm;    // output offset, stream offset of the first column, own multipole
};
struct alignas(128) PWRing {
  PWStage st[kPWStages];
  PWDesc desc[kPWStages];
  uint64_t full[kPWStages], empty[kPWStages];
};
constexpr size_t kPWDynSmem = sizeof(PWRing) * kPWRings;
// polling wait (test_wait, no suspend): the warp-pair kernel's waits are short and on every warp's
// critical path
__device__ __forceinline__ void mbar_wait_poll(uint64_t* b, uint32_t parity) {
#if DAFMM_PW_SPIN
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_addr(b)), "r"(parity)
        : "memory");
  } while (!done);
#else
  mbar_wait(b, parity);
#endif
}
__device__ __forceinline__ void cmac(double& ar, double& ai, const double2 m, const double2 v) {
  ar = fma(m.x, v.x, fma(-m.y, v.y, ar));
  ai = fma(m.x, v.y, fma(m.y, v.x, ai));
}
__global__ void __maxnreg__(DAFMM_PW_MAXREG) m2l_pairw_kernel(
    int ntargets, const int64_t* __restrict__ loc_off, const int32_t* __restrict__ rows,
    const int64_t* __restrict__ stream_ptr, const int32_t* __restrict__ stream_idx,
    const int64_t* __restrict__ mat_off, const int64_t* __restrict__ self_moff, const int32_t* __restrict__ src_ptr,
    const int64_t* __restrict__ src_off, const int32_t* __restrict__ src_cnt, const double2* __restrict__ mat,
    const double2* __restrict__ mult, double2* __restrict__ loc, double2* __restrict__ slots) {
  extern __shared__ __align__(128) unsigned char pw_dyn[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ring = warp >> 1, role = warp & 1;
  PWRing& W = reinterpret_cast<PWRing*>(pw_dyn)[ring];  // (no pointer arithmetic on integers: keeps LDS)
  if (role == 0 && lane == 0) {
    for (int i = 0; i < kPWStages; ++i) {
      mbar_init(&W.full[i], 1);
      mbar_init(&W.empty[i], 2);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (role == 1) {  // ---- column warp
    for (int k = 0;; ++k) {
      const int slot = k % kPWStages;
      mbar_wait_poll(&W.full[slot], (uint32_t)(k / kPWStages) & 1u);
      const PWDesc d = W.desc[slot];
      if (d.r < 0) break;
      const int r = d.r, ncs = d.ncs, lg = d.lg, g = 1 << lg, rot = d.rot;
      const int cl = lane >> lg, i = lane & (g - 1);
      const double2* R = W.st[slot].ent;
      double sr = 0.0, si = 0.0, tr = 0.0, ti = 0.0;
      if (cl < ncs) {
        const double2* col = R + cl * r;
        if (r <= 32) {
          const double2* ms = W.st[slot].ms;
          if (rot == 0) {
            int t = i;
            for (; t + g < r; t += 2 * g) {
              cmac(sr, si, col[t], ms[t]);
              cmac(tr, ti, col[t + g], ms[t + g]);
            }
            if (t < r) cmac(sr, si, col[t], ms[t]);
          } else {
            int t = i + (rot * cl) % r;
            if (t >= r) t -= r;
            int v = i;
            for (; v + g < r; v += 2 * g) {
              int t1 = t + g;
              if (t1 >= r) t1 -= r;
              cmac(sr, si, col[t], ms[t]);
              cmac(tr, ti, col[t1], ms[t1]);
              t = t1 + g;
              if (t >= r) t -= r;
            }
            if (v < r) cmac(sr, si, col[t], ms[t]);
          }
        } else {  // more than 32 rows: the own multipole from L2
          for (int t = i; t < r; t += g) cmac(sr, si, col[t], ld2(mult + d.sm + t));
        }
        sr += tr;
        si += ti;
      }
      for (int o = g >> 1; o > 0; o >>= 1) {
        sr += __shfl_xor_sync(0xffffffffu, sr, o);
        si += __shfl_xor_sync(0xffffffffu, si, o);
      }
      if (i == 0 && cl < ncs) slots[d.spc + cl] = make_double2(sr, si);
      __syncwarp();
      if (lane == 0) mbar_arrive(&W.empty[slot]);
    }
    return;
  }
  // ---- row warp (drives the ring)
  const int G = gridDim.x * kPWRings;
  // The stage cursor (warp-uniform; lane 0 issues): nodes g, g + G, ...; within a node its source
  // runs (one per partner node A: r_A consecutive multipole slots = r_A columns of the block), cut
  // into chunks of at most `cps` columns.  The next node's metadata is loaded one node ahead (one
  // field per lane), the next run's one run ahead.
  int nn = blockIdx.x * kPWRings + ring;  // next node to enter
  int64_t nmeta = 0;
  auto prefetch_node = [&]() {
    if (nn < ntargets) {
      if (lane == 0) nmeta = rows[nn];
      else if (lane == 1) nmeta = stream_ptr[nn];
      else if (lane == 2) nmeta = src_ptr[nn];
      else if (lane == 3) nmeta = loc_off[nn];
      else if (lane == 4) nmeta = mat_off[nn];
      else if (lane == 5) nmeta = self_moff[nn];
      else if (lane == 6) nmeta = src_ptr[nn + 1];
      else if (lane == 7) nmeta = stream_ptr[nn + 1] - stream_ptr[nn];
    }
  };
  prefetch_node();
  int cr = 0, ccps = 1, crun = 0, cruns = 0;  // current node: rows, columns per stage, run cursor / end
  int cL = 0, cc = 0;                         // its columns, the next column
  int rc = 0, rcnt = 0;                       // the current run: columns taken, length
  int64_t csp = 0, clo = 0, cmoff = 0, csm = 0, roff = 0;
  int nrcnt = 0;  // the next run (loaded one run ahead)
  int64_t nroff = 0;
  bool done = false;
  auto next_run = [&]() {
    rc = 0;
    roff = nroff;
    rcnt = nrcnt;
    if (crun < cruns) {  // crun: the run to load ahead
      nroff = src_off[crun];
      nrcnt = src_cnt[crun];
    }
    ++crun;
  };
  // issue(): a stage = the next (at most ccps) columns of the node's stream, whatever runs they
  // belong to: one TMA for the entries, one per run segment for the multipoles, one for the own
  // multipole, all completing on the slot's `full` barrier
  auto issue = [&](int slot) {
    while (!done && cc >= cL) {  // next node (skipping nodes that own no block)
      if (nn >= ntargets) {
        done = true;
        break;
      }
      cr = (int)__shfl_sync(0xffffffffu, nmeta, 0);
      csp = __shfl_sync(0xffffffffu, nmeta, 1);
      crun = (int)__shfl_sync(0xffffffffu, nmeta, 2);
      clo = __shfl_sync(0xffffffffu, nmeta, 3);
      cmoff = __shfl_sync(0xffffffffu, nmeta, 4);
      csm = __shfl_sync(0xffffffffu, nmeta, 5);
      cruns = (int)__shfl_sync(0xffffffffu, nmeta, 6);
      cL = (int)__shfl_sync(0xffffffffu, nmeta, 7);
      nn += G;
      prefetch_node();
      if (cr <= 0) cL = 0;  // a node without pivots owns no entries (reading R11)
      ccps = min(32, kPWStageE / max(cr, 1));
      cc = 0;
      rc = rcnt = 0;
      if (crun < cruns) {
        nroff = src_off[crun];
        nrcnt = src_cnt[crun];
      }
      ++crun;
      if (cL > 0) next_run();
    }
    if (done) {
      if (lane == 0) {
        W.desc[slot] = PWDesc{-1, 0, 0, 0, 0, 0, 0, 0, 0};
        mbar_arrive_tx(&W.full[slot], 0u);
      }
      return;
    }
    const int ncs = min(ccps, cL - cc);
    const bool own = cr <= 32;
    if (lane == 0) {
      int lg = 0;
      while ((2 << lg) * ncs <= 32) ++lg;
      const int g = 1 << lg;
      const int rot = (g >= 8 || cr % (2 * g) == g) ? 0 : ((g - cr) & 7);
      W.desc[slot] = PWDesc{cr, ncs, (cc == 0 ? 1 : 0) | (cc + ncs >= cL ? 2 : 0), lg, rot, 0, clo, csp + cc, csm};
      mbar_arrive_tx(&W.full[slot], (uint32_t)(ncs * cr + ncs + (own ? cr : 0)) * 16u);
      bulk_load(W.st[slot].ent, mat + cmoff + (int64_t)cc * cr, (uint32_t)(ncs * cr) * 16u, &W.full[slot]);
      if (own) bulk_load(W.st[slot].ms, mult + csm, (uint32_t)cr * 16u, &W.full[slot]);
    }
    for (int c = 0; c < ncs;) {  // the multipoles, run segment by run segment
      while (rc >= rcnt) next_run();
      const int seg = min(ncs - c, rcnt - rc);
      if (lane == 0) bulk_load(W.st[slot].mv + c, mult + roff + rc, (uint32_t)seg * 16u, &W.full[slot]);
      rc += seg;
      c += seg;
    }
    cc += ncs;
  };
  for (int i = 0; i < kPWStages - 1; ++i) issue(i);  // prologue: stages 0 .. kPWStages - 2
  double ar = 0.0, ai = 0.0;  // the row sums of rows lane (r <= 32), over the node's stages
  for (int k = 0;; ++k) {
    const int slot = k % kPWStages;
    {  // refill the slot of stage k - 1 with stage k + kPWStages - 1
      const int ps = (slot + kPWStages - 1) % kPWStages;
      if (k >= 1) mbar_wait_poll(&W.empty[ps], (uint32_t)((k - 1) / kPWStages) & 1u);
      issue(ps);
    }
    mbar_wait_poll(&W.full[slot], (uint32_t)(k / kPWStages) & 1u);
    const PWDesc d = W.desc[slot];
    if (d.r < 0) break;
    const int r = d.r, ncs = d.ncs;
    const double2* R = W.st[slot].ent;
    const double2* mv = W.st[slot].mv;
    if (r <= 32) {
      if (d.flags & 1) ar = ai = 0.0;
      if (lane < r) {
        const double2* p = R + lane;
        double br = 0.0, bi = 0.0;
        int c = 0;
#if DAFMM_PW_UNROLL4
        for (; c + 4 <= ncs; c += 4, p += 4 * r) {
          const double2 m0 = p[0], m1 = p[r], m2 = p[2 * r], m3 = p[3 * r];
          const double2 v0 = mv[c], v1 = mv[c + 1], v2 = mv[c + 2], v3 = mv[c + 3];
          cmac(ar, ai, m0, v0);
          cmac(br, bi, m1, v1);
          cmac(ar, ai, m2, v2);
          cmac(br, bi, m3, v3);
        }
#endif
        for (; c + 2 <= ncs; c += 2, p += 2 * r) {
          const double2 m0 = p[0], m1 = p[r];
          const double2 v0 = mv[c], v1 = mv[c + 1];
          cmac(ar, ai, m0, v0);
          cmac(br, bi, m1, v1);
        }
        if (c < ncs) cmac(ar, ai, p[0], mv[c]);
        ar += br;
        ai += bi;
        if (d.flags & 2) loc[d.lo + lane] = make_double2(ar, ai);  // the node's last stage
      }
    } else {  // more than 32 rows (rare): per stage, the rows' partial sums are added to the node's
              // output directly (this warp is its only writer; M2L starts from zeroed outputs)
      for (int t = lane; t < r; t += 32) {
        double sr = 0.0, si = 0.0;
        for (int c = 0; c < ncs; ++c) cmac(sr, si, R[c * r + t], mv[c]);
        double2 o = loc[d.lo + t];
        o.x += sr;
        o.y += si;
        loc[d.lo + t] = o;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&W.empty[slot]);
  }
}

// loc[node] += sum of the column-sum slots the owners wrote for it (fixed order: deterministic).
// One warp per receiving node.
__global__ void m2l_slot_gather_kernel(int nodes, const int64_t* __restrict__ in_lo, const int32_t* __restrict__ in_rows,
                                       const int32_t* __restrict__ in_ptr, const int64_t* __restrict__ in_off,
                                       const double2* __restrict__ slots, double2* __restrict__ loc) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= nodes) return;
  const int r = in_rows[w], k0 = in_ptr[w], k1 = in_ptr[w + 1];
  const int64_t lo = in_lo[w];
  for (int c = lane; c < r; c += 32) {
    double2 acc = loc[lo + c];
    for (int k = k0; k < k1; ++k) {
      const double2 v = ld2(slots + in_off[k] + c);
      acc.x += v.x;
      acc.y += v.y;
    }
    loc[lo + c] = acc;
  }
}

// ---- near field P2P ------------------------------------------------------------
// phi_t = sum_{j in N(leaf), j != t} H0(kappa |x_t - x_j|) v_j   (H0 units, tree order).
// The leaf's own block is the first near entry (the only one with i == j pairs).
#ifndef DAFMM_P2P_MINB
#define DAFMM_P2P_MINB 3
#endif
#ifdef DAFMM_P2P_MAXREG
#define DAFMM_P2P_REGCAP __maxnreg__(DAFMM_P2P_MAXREG)
#else
#define DAFMM_P2P_REGCAP __launch_bounds__(kNearThreads, DAFMM_P2P_MINB)
#endif
__global__ void DAFMM_P2P_REGCAP p2p_kernel(
    const int32_t* __restrict__ leaf_begin, const int32_t* __restrict__ leaf_end, const int32_t* __restrict__ near_ptr,
    const int32_t* __restrict__ near_begin, const int32_t* __restrict__ near_end, const int32_t* __restrict__ leaf_band,
    const double2* __restrict__ pts_t, const double2* __restrict__ v_t, double2* __restrict__ phi, int sym,
    const int64_t* __restrict__ leaf_slot_base, double2* __restrict__ slots, int64_t slot_total) {
  __shared__ __align__(16) double4 buf[2 * kNearStage];
  __shared__ double2 red[kNearThreads];
  __shared__ PolyTable T;
  load_poly_table(T);
  const int leaf = blockIdx.x;
  const int tb = leaf_begin[leaf], m = leaf_end[leaf] - tb;
  const int ps = near_ptr[leaf], pe = near_ptr[leaf + 1];
  int total = 0;
  for (int e = ps; e < pe; ++e) total += near_end[e] - near_begin[e];
  for (int t0 = 0; t0 < m; t0 += kNearThreads) {
    const int rc = min(kNearThreads, m - t0);
    const int nsl = kNearThreads / rc;
    const int t = threadIdx.x % rc;
    const int slice = threadIdx.x / rc;
    const bool active = slice < nsl;
    double2 xt = ld2(pts_t + tb + t0 + t);
    // symmetric near field (every leaf has 32 or 64 points): slices are whole warps; warp
    // (t / 32) of the slice writes its half of the slots
    const NearItems items{leaf_band[leaf], pe > ps ? near_end[ps] - near_begin[ps] : 0, total, 0, 2, sym,
                          slots + (sym ? (int64_t)(t >> 5) * slot_total : 0), sym ? leaf_slot_base[leaf] : 0,
                          sym ? ld2(v_t + tb + t0 + t) : make_double2(0.0, 0.0)};
    double ar = 0.0, ai = 0.0;
    if (pe > ps) {
      RunStager st{near_begin, near_end, ps, 0, pe, pts_t, v_t};
      stream_accumulate<kNearStage>(buf, st, items, xt, active, slice, nsl, ar, ai, T, nullptr);
    }
    red[threadIdx.x] = make_double2(ar, ai);
    __syncthreads();
    if (threadIdx.x < rc) {
      double sr = 0.0, si = 0.0;
      for (int s = 0; s < nsl; ++s) {
        double2 v = red[threadIdx.x + s * rc];
        sr += v.x;
        si += v.y;
      }
      phi[tb + t0 + threadIdx.x] = make_double2(sr, si);
    }
    __syncthreads();
  }
}

// ---- L2P + combine + scatter ---------------------------------------------------
// phi_t = (i/4) [ P2P_t + (U u)_t ] + D_t x_t;   y[perm[t]] = x_t + kappa^2 q_t phi_t (mode 0)
// or phi_t (mode 1).  One CTA per leaf, one thread per point (coalesced columns of U).
__global__ void combine_kernel(const int32_t* __restrict__ leaf_begin, const int32_t* __restrict__ leaf_end,
                               const int64_t* __restrict__ leaf_loc_off, const int32_t* __restrict__ leaf_rank,
                               const int64_t* __restrict__ leaf_U_off, const double2* __restrict__ ops,
                               const double2* __restrict__ loc, const double2* __restrict__ phi,
                               const double2* __restrict__ x_t, const double* __restrict__ qk2_t,
                               const double2* __restrict__ D_t, const int32_t* __restrict__ perm,
                               double2* __restrict__ y, int kernel_mode, int do_near, int do_far_in,
                               const int32_t* __restrict__ in_ptr, const int64_t* __restrict__ in_off,
                               const double2* __restrict__ slots, int64_t slot_total) {
  const int leaf = blockIdx.x;
  const int tb = leaf_begin[leaf], m = leaf_end[leaf] - tb;
  const bool do_far = do_far_in && leaf_loc_off[leaf] >= 0;
  for (int tt = threadIdx.x; tt < m; tt += blockDim.x) {
    double sr = 0.0, si = 0.0;
    if (do_near) {
      const double2 p = phi[tb + tt];
      sr = p.x;
      si = p.y;
      if (in_ptr)  // symmetric near field: the pairs evaluated by earlier leaves (both slot halves)
        for (int k = in_ptr[leaf]; k < in_ptr[leaf + 1]; ++k) {
          const double2 a = slots[in_off[k] + tt], b = slots[slot_total + in_off[k] + tt];
          sr += a.x + b.x;
          si += a.y + b.y;
        }
    }
    if (do_far) {  // L2P: (U u)_t, U column-major m x r
      const int rk = leaf_rank[leaf];
      const double2* U = ops + leaf_U_off[leaf];
      const double2* u = loc + leaf_loc_off[leaf];
      double ar[2] = {0.0, 0.0}, ai[2] = {0.0, 0.0};
      int c = 0;
      for (; c + 2 <= rk; c += 2) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const double2 a = ld2(U + (int64_t)(c + q) * m + tt), b = ld2(u + c + q);
          ar[q] = fma(a.x, b.x, fma(-a.y, b.y, ar[q]));
          ai[q] = fma(a.x, b.y, fma(a.y, b.x, ai[q]));
        }
      }
      if (c < rk) {
        const double2 a = ld2(U + (int64_t)c * m + tt), b = ld2(u + c);
        ar[0] = fma(a.x, b.x, fma(-a.y, b.y, ar[0]));
        ai[0] = fma(a.x, b.y, fma(a.y, b.x, ai[0]));
      }
      sr += ar[0] + ar[1];
      si += ai[0] + ai[1];
    }
    // phi = (i/4) (sr + i si) + D x
    const double2 xv = x_t[tb + tt];
    double pr = -0.25 * si, pi = 0.25 * sr;
    if (do_near) {
      const double2 d = D_t[tb + tt];
      pr = fma(d.x, xv.x, fma(-d.y, xv.y, pr));
      pi = fma(d.x, xv.y, fma(d.y, xv.x, pi));
    }
    double2 out;
    if (kernel_mode == 0) {
      const double q = qk2_t[tb + tt];
      out = make_double2(q * pr, q * pi);
      if (do_near) {
        out.x += xv.x;
        out.y += xv.y;
      }
    } else {
      out = make_double2(pr, pi);
    }
    y[perm[tb + tt]] = out;
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

// part[bx * stride + i] = sum over block bx's slice of conj(V_i) w for the kMD vectors
// i = blockIdx.y * kMD + g of this block: w is read once per group of kMD basis vectors and
// each thread keeps kMD complex partial sums (one pass, no per-vector barriers).
#ifndef DAFMM_KMD
#define DAFMM_KMD 4  // measured: C3 GMRES(200) 2.43 s at 8, 2.26 s at 4, 2.24 s at 2, 2.63 s at 16
#endif
constexpr int kMD = DAFMM_KMD;  // basis vectors per multi-dot block row
#ifndef DAFMM_MD_BLOCKS
#define DAFMM_MD_BLOCKS 148
#endif
__global__ void multidot_kernel(int64_t n, int k, const double2* __restrict__ V, const double2* __restrict__ w,
                                double2* __restrict__ part, int stride) {
  __shared__ double2 sh[kMD][kVecThreads / 32];
  const int i0 = blockIdx.y * kMD;
  const int nv = min(kMD, k - i0);
  double ar[kMD], ai[kMD];
#pragma unroll
  for (int g = 0; g < kMD; ++g) ar[g] = ai[g] = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const double2 b = ld2(w + e);
#pragma unroll
    for (int g = 0; g < kMD; ++g) {
      if (g < nv) {
        const double2 a = ld2(V + (int64_t)(i0 + g) * n + e);
        ar[g] = fma(a.x, b.x, fma(a.y, b.y, ar[g]));
        ai[g] = fma(a.x, b.y, fma(-a.y, b.x, ai[g]));
      }
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int g = 0; g < kMD; ++g) {
    for (int o = 16; o > 0; o >>= 1) {
      ar[g] += __shfl_down_sync(0xffffffffu, ar[g], o);
      ai[g] += __shfl_down_sync(0xffffffffu, ai[g], o);
    }
    if (lane == 0) sh[g][wid] = make_double2(ar[g], ai[g]);
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double sr = 0.0, si = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
      sr += sh[threadIdx.x][q].x;
      si += sh[threadIdx.x][q].y;
    }
    part[(int64_t)blockIdx.x * stride + i0 + threadIdx.x] = make_double2(sr, si);
  }
}

// out[i] = sum_b part[b * stride + i]: one warp per output, lanes over the blocks, then a fixed
// shuffle tree (deterministic order).  Launch with reduce_launch().
__global__ void reduce_parts_kernel(int nblocks, int k, const double2* __restrict__ part, int stride,
                                    double2* __restrict__ out) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= k) return;
  double sr = 0.0, si = 0.0;
  for (int b = lane; b < nblocks; b += 32) {
    const double2 v = part[(int64_t)b * stride + i];
    sr += v.x;
    si += v.y;
  }
  for (int o = 16; o > 0; o >>= 1) {
    sr += __shfl_down_sync(0xffffffffu, sr, o);
    si += __shfl_down_sync(0xffffffffu, si, o);
  }
  if (lane == 0) out[i] = make_double2(sr, si);
}
void reduce_launch(int nblocks, int k, const double2* part, int stride, double2* out, cudaStream_t s) {
  reduce_parts_kernel<<<(k + 7) / 8, 256, 0, s>>>(nblocks, k, part, stride, out);
}

// w += sign * sum_{i<k} h_i V_i
__global__ void combine_kernel(int64_t n, int k, const double2* __restrict__ V, const double2* __restrict__ h,
                               double sign, double2* __restrict__ w) {
  __shared__ double2 hs[256];
  for (int i = threadIdx.x; i < k; i += blockDim.x) hs[i] = h[i];
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = w[e], acc1 = make_double2(0.0, 0.0);
    int i = 0;
    // 4 basis vectors per step, two accumulators: 4 loads in flight, half-length FMA chains
    for (; i + 4 <= k; i += 4) {
      double2 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = ld2(V + (int64_t)(i + q) * n + e);
#pragma unroll
      for (int q = 0; q < 4; q += 2) {
        const double2 c0 = make_double2(sign * hs[i + q].x, sign * hs[i + q].y);
        const double2 c1 = make_double2(sign * hs[i + q + 1].x, sign * hs[i + q + 1].y);
        acc.x = fma(c0.x, v[q].x, fma(-c0.y, v[q].y, acc.x));
        acc.y = fma(c0.x, v[q].y, fma(c0.y, v[q].x, acc.y));
        acc1.x = fma(c1.x, v[q + 1].x, fma(-c1.y, v[q + 1].y, acc1.x));
        acc1.y = fma(c1.x, v[q + 1].y, fma(c1.y, v[q + 1].x, acc1.y));
      }
    }
    for (; i < k; ++i) {
      const double2 v = ld2(V + (int64_t)i * n + e);
      const double2 c = make_double2(sign * hs[i].x, sign * hs[i].y);
      acc.x = fma(c.x, v.x, fma(-c.y, v.y, acc.x));
      acc.y = fma(c.x, v.y, fma(c.y, v.x, acc.y));
    }
    w[e] = make_double2(acc.x + acc1.x, acc.y + acc1.y);
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

// ---- H0 evaluator probe (dafmm_h0_eval) ------------------------------------------------------
// out[i] = H0^(1)(sqrt(z2[i])) by the band `code`'s evaluator, lane-blocked exactly as in P2P /
// M2L (kH0EvalTB entries per thread, coefficient tables in shared memory): it exposes the
// product's inner evaluator to the parity tests, band by band.
constexpr int kH0EvalTB = 4;
template <int CODE>
__device__ __forceinline__ void h0_eval_block(const double* z2, double* re, double* im, const PolyTable& T,
                                              const FarBand* band) {
  eval_band<CODE, kH0EvalTB>(z2, re, im, T, band);
}
__global__ void __launch_bounds__(128) h0_eval_kernel(const double* __restrict__ z2, double2* __restrict__ out,
                                                      int64_t n, int code) {
  __shared__ PolyTable T;
  __shared__ FarBand bands[dafmm_fit::NUM_FAR];
  load_poly_table(T);
  load_far_bands(bands);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * kH0EvalTB;
  for (int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kH0EvalTB; i0 < n; i0 += stride) {
    double z[kH0EvalTB], re[kH0EvalTB], im[kH0EvalTB];
#pragma unroll
    for (int q = 0; q < kH0EvalTB; ++q) z[q] = z2[i0 + q < n ? i0 + q : i0];
    switch (code) {
      case kBandGeneric: h0_eval_block<kBandGeneric>(z, re, im, T, nullptr); break;
      case kBandNear7: h0_eval_block<kBandNear7>(z, re, im, T, nullptr); break;
      case kBandNear8: h0_eval_block<kBandNear8>(z, re, im, T, nullptr); break;
      case kBandNear12: h0_eval_block<kBandNear12>(z, re, im, T, nullptr); break;
      default: h0_eval_block<kBandFarData>(z, re, im, T, bands + (code - kBandFarData));
    }
#pragma unroll
    for (int q = 0; q < kH0EvalTB; ++q)
      if (i0 + q < n) out[i0 + q] = make_double2(re[q], im[q]);
  }
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

// free one allocation made by alloc / upload (and forget it)
template <typename T>
void release(DevPlan& d, T** p) {
  if (!*p) return;
  auto it = std::find(d.allocations.begin(), d.allocations.end(), (void*)*p);
  if (it != d.allocations.end()) d.allocations.erase(it);
  cudaFree(*p);
  *p = nullptr;
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

bool upload_batch(DevPlan& d, DevBatch& b, const Packed::Batch& h, std::string& err, bool colmajor) {
  b.items = (int)h.dst_off.size();
  b.colmajor = colmajor;
  // kernel choice by shape: wide items (mean >= 48 columns) read each row with all 32 lanes
  // and reduce across the warp; narrow ones give each lane a row.  (A TMA-streamed variant on
  // column-major items, the stored-M2L kernel's ring, was measured slower: one gather latency
  // per small item; profiles/README.md, r2e.)
  int64_t cols = 0;
  for (int32_t c : h.item_cols) cols += c;
  b.wide = b.items > 0 && cols >= 48 * (int64_t)b.items;
  // narrow items: several per warp when their rows fit a lane group (16 or 8 lanes)
  int maxr = 0;
  for (int32_t r : h.dst_rows) maxr = std::max(maxr, (int)r);
  b.ipw = maxr <= 8 ? 4 : maxr <= 16 ? 2 : 1;
  int64_t rows_sum = 0;
  for (int32_t r : h.dst_rows) rows_sum += r;
  b.grouped = b.items > 0 && rows_sum <= 16 * (int64_t)b.items;
  return upload(d, &b.dst_off, h.dst_off, err) && upload(d, &b.dst_rows, h.dst_rows, err) &&
         upload(d, &b.term_ptr, h.term_ptr, err) && upload(d, &b.item_mat_off, h.item_mat_off, err) &&
         upload(d, &b.item_cols, h.item_cols, err) &&
         upload(d, &b.src_off, h.src_off, err) && upload(d, &b.src_cols, h.src_cols, err);
}

int launch_translate(const DevPlan& d, const DevBatch& b, const double2* src, double2* dst, int accumulate,
                     cudaStream_t st) {
  if (b.items == 0) return 0;
  int threads = 256;
  int blocks = (b.items * 32 + threads - 1) / threads;
  if (b.colmajor && b.grouped)  // small nodes (mean rows <= 16): lane groups
    translate_cm_kernel<true><<<(b.items + kTCMWarps - 1) / kTCMWarps, 32 * kTCMWarps, 0, st>>>(
        b.items, b.dst_off, b.dst_rows, b.item_mat_off, b.item_cols, b.term_ptr, b.src_off, b.src_cols, d.ops, src,
        dst, accumulate);
  else if (b.colmajor)
    translate_cm_kernel<false><<<(b.items + kTCMWarps - 1) / kTCMWarps, 32 * kTCMWarps, 0, st>>>(
        b.items, b.dst_off, b.dst_rows, b.item_mat_off, b.item_cols, b.term_ptr, b.src_off, b.src_cols, d.ops, src,
        dst, accumulate);
  else if (b.wide)
    translate_kernel<<<blocks, threads, 0, st>>>(b.items, b.dst_off, b.dst_rows, b.item_mat_off, b.item_cols,
                                                 b.term_ptr, b.src_off, b.src_cols, d.ops, src, dst, accumulate);
  else
    translate_rows_kernel<<<(b.items + 8 * b.ipw - 1) / (8 * b.ipw), threads, 0, st>>>(
        b.items, b.dst_off, b.dst_rows, b.item_mat_off, b.item_cols, b.term_ptr, b.src_off, b.src_cols, d.ops, src,
        dst, accumulate, b.ipw);
  return 1;
}

}  // namespace

int upload_plan(const Packed& pk, const Plan& plan, DevPlan& d, std::string& err) {
  d.n = plan.n;
  d.kernel_mode = plan.opt.kernel_mode;
  std::vector<double2> pts(plan.n), D(plan.n);
  for (int64_t t = 0; t < plan.n; ++t) {
    pts[t] = make_double2(pk.pts_t[2 * t], pk.pts_t[2 * t + 1]);
    D[t] = make_double2(pk.D_t[t].re, pk.D_t[t].im);
  }
  std::vector<double2> so(pk.n_mult), ti(pk.n_loc);
  for (int64_t k = 0; k < pk.n_mult; ++k) so[k] = make_double2(pk.so_xy[2 * k], pk.so_xy[2 * k + 1]);
  for (int64_t k = 0; k < pk.n_loc; ++k) ti[k] = make_double2(pk.ti_xy[2 * k], pk.ti_xy[2 * k + 1]);
  std::vector<double2> ops(pk.ops.size());
  std::memcpy(ops.data(), pk.ops.data(), sizeof(double2) * ops.size());
  d.n_mult = pk.n_mult;
  d.n_loc = pk.n_loc;
  d.ops_len = pk.ops_on_device ? pk.ops_len : (int64_t)ops.size();
  bool ok = upload(d, &d.pts_t, pts, err) && upload(d, &d.w_t, pk.w_t, err) && upload(d, &d.qk2_t, pk.qk2_t, err) &&
            upload(d, &d.D_t, D, err) && upload(d, &d.perm, pk.perm, err) && upload(d, &d.so_xy, so, err) &&
            upload(d, &d.ti_xy, ti, err) &&
            (pk.ops_on_device ? alloc(d, &d.ops, (size_t)pk.ops_len, err) : upload(d, &d.ops, ops, err)) && upload_batch(d, d.p2m, pk.p2m, err, pk.ops_colmajor != 0);
  d.m2m.assign(pk.m2m.size(), DevBatch());
  for (size_t i = 0; ok && i < pk.m2m.size(); ++i) ok = upload_batch(d, d.m2m[i], pk.m2m[i], err, pk.ops_colmajor != 0);
  d.l2l.assign(pk.l2l.size(), DevBatch());
  for (size_t i = 0; ok && i < pk.l2l.size(); ++i) ok = upload_batch(d, d.l2l[i], pk.l2l[i], err, pk.ops_colmajor != 0);
  if (ok && pk.ops_on_device) {  // F2: translation operators formed on the device
    std::vector<OpGroup> groups(pk.opd_groups.size());
    for (size_t g = 0; g < groups.size(); ++g) {
      const auto& a = pk.opd_groups[g];
      groups[g] = OpGroup{a[0], a[1], a[2], a[3], a[4], a[5]};
    }
    std::vector<OpJob> jobs(pk.opd_jobs.size());
    for (size_t j = 0; j < jobs.size(); ++j) {
      const auto& a = pk.opd_jobs[j];
      jobs[j] = OpJob{a.off, a.rows, a.col_start, a.stride, 0, a.src_off, a.src_len, 0};
    }
    const auto t0 = std::chrono::steady_clock::now();
    const int rc = form_ops_device(plan.pts.data(), plan.n, plan.kappa, pk.opd_piv, groups, jobs, d.ops, err);
    if (rc != DAFMM_OK) return rc;
    d.t_ops_device = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  d.m2l_targets = (int)pk.m2l_loc_off.size();
  d.m2l_leaf_targets = pk.m2l_leaf_targets;
  ok = ok && upload(d, &d.m2l_loc_off, pk.m2l_loc_off, err) && upload(d, &d.m2l_rows, pk.m2l_rows, err) &&
       upload(d, &d.m2l_stream_ptr, pk.m2l_stream_ptr, err) && upload(d, &d.m2l_stream_idx, pk.m2l_stream_idx, err) &&
       upload(d, &d.m2l_item_ptr, pk.m2l_item_ptr, err) &&
       upload(d, &d.m2l_item_code, pk.m2l_item_code, err) && upload(d, &d.m2l_item_begin, pk.m2l_item_begin, err) &&
       upload(d, &d.m2l_item_end, pk.m2l_item_end, err);
  d.nleaves = (int)pk.leaf_begin.size();
  d.max_leaf = pk.max_leaf;
  ok = ok && upload(d, &d.leaf_begin, pk.leaf_begin, err) && upload(d, &d.leaf_end, pk.leaf_end, err) &&
       upload(d, &d.near_ptr, pk.near_ptr, err) && upload(d, &d.near_begin, pk.near_begin, err) &&
       upload(d, &d.near_end, pk.near_end, err) && upload(d, &d.leaf_loc_off, pk.leaf_loc_off, err) &&
       upload(d, &d.leaf_rank, pk.leaf_rank, err) && upload(d, &d.leaf_U_off, pk.leaf_U_off, err) &&
       upload(d, &d.leaf_band, pk.leaf_band, err);
  d.p2p_sym = pk.p2p_sym;
  d.slot_total = pk.slot_total;
  if (ok && d.p2p_sym) {
    ok = upload(d, &d.leaf_slot_base, pk.leaf_slot_base, err) && upload(d, &d.in_ptr, pk.in_ptr, err) &&
         upload(d, &d.in_off, pk.in_off, err) && alloc(d, &d.slots, (size_t)(2 * d.slot_total), err) &&
         ck(cudaMemset(d.slots, 0, sizeof(double2) * (size_t)(2 * d.slot_total)), err, "slots memset");
  }
  if (ok && d.m2l_targets > 0 && plan.opt.m2l_store != 0) {  // stored M2L blocks
    std::vector<int64_t> moff(d.m2l_targets);
    int64_t tot = 0;
    int maxr = 0;
    for (int t = 0; t < d.m2l_targets; ++t) {
      moff[t] = tot;
      maxr = std::max(maxr, pk.m2l_rows[t]);
      tot += (int64_t)pk.m2l_rows[t] * (pk.m2l_stream_ptr[t + 1] - pk.m2l_stream_ptr[t]);
    }
    size_t free_b = 0, total_b = 0;
    if (!ck(cudaMemGetInfo(&free_b, &total_b), err, "cudaMemGetInfo")) return DAFMM_ECUDA;
    const size_t bytes = (size_t)tot * sizeof(double2);
    if (plan.opt.m2l_store == 1 && maxr > kMaxStoredRows) {
      err = "m2l_store=1: a node has " + std::to_string(maxr) + " pivots (at most " +
            std::to_string(kMaxStoredRows) + " supported)";
      return DAFMM_EINVAL;
    }
    if (plan.opt.m2l_store == 1 && bytes > free_b) {
      err = "m2l_store=1: the M2L blocks need " + std::to_string(bytes) + " bytes, " + std::to_string(free_b) +
            " free";
      return DAFMM_ENOMEM;
    }
    if (tot > 0 && maxr <= kMaxStoredRows && (plan.opt.m2l_store == 1 || pk.m2l_sym || bytes <= free_b / 2)) {
      ok = upload(d, &d.m2l_mat_off, moff, err) && alloc(d, &d.m2l_mat, (size_t)tot, err);
      if (ok) {
        m2l_form_kernel<<<d.m2l_targets, kMSFormThreads>>>(d.m2l_loc_off, d.m2l_rows, d.m2l_stream_ptr,
                                                         d.m2l_stream_idx, d.m2l_mat_off, d.ti_xy, d.so_xy,
                                                         d.m2l_mat);
        ok = ck(cudaGetLastError(), err, "m2l_form_kernel") && ck(cudaDeviceSynchronize(), err, "m2l_form_kernel");
      }
      if (!ok) return DAFMM_ECUDA;
    }
    if (pk.m2l_sym && !d.m2l_mat) {
      err = "pair-stored M2L (m2l_store=2): the blocks could not be stored";
      return DAFMM_ENOMEM;
    }
    if (pk.m2l_sym) {  // R22: own multipoles, column-sum slots, receiving nodes' slot lists
      d.m2l_sym = 1;
      d.m2l_in_nodes = (int)pk.m2l_in_lo.size();
      ok = upload(d, &d.m2l_self_moff, pk.m2l_self_moff, err) && upload(d, &d.m2l_src_ptr, pk.m2l_src_ptr, err) &&
           upload(d, &d.m2l_src_off, pk.m2l_src_off, err) && upload(d, &d.m2l_src_cnt, pk.m2l_src_cnt, err) &&
           upload(d, &d.m2l_in_lo, pk.m2l_in_lo, err) &&
           upload(d, &d.m2l_in_rows, pk.m2l_in_rows, err) && upload(d, &d.m2l_in_ptr, pk.m2l_in_ptr, err) &&
           upload(d, &d.m2l_in_off, pk.m2l_in_off, err) &&
           alloc(d, &d.m2l_slots, pk.m2l_stream_idx.size(), err);
      if (!ok) return DAFMM_ECUDA;
    }
  }
  if (ok) {
    int per_sm = 0, sms = 0, dev = 0;
    ok = ck(cudaGetDevice(&dev), err, "cudaGetDevice") &&
         ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), err, "SM count") &&
         ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, m2l_kernel, kM2LThreads, 0), err, "occupancy");
    d.m2l_grid = std::max(1, std::min(d.m2l_targets, std::max(1, per_sm) * sms));
    d.m2l_store_grid = std::max(1, std::min(d.m2l_targets, DAFMM_MS_PER_SM * sms));
    d.m2l_pair_grid = std::max(1, std::min((d.m2l_targets + kPWRings - 1) / kPWRings, DAFMM_PW_PER_SM * sms));
    if (d.m2l_mat)
      ok = ck(cudaFuncSetAttribute(m2l_stored_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMSDynSmem),
              err, "stored M2L shared memory") &&
           ck(cudaFuncSetAttribute(m2l_pairw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPWDynSmem),
              err, "pair M2L shared memory") &&
           ck(cudaFuncSetAttribute(m2l_pairw_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100), err,
              "carveout") &&
           ck(cudaFuncSetAttribute(m2l_stored_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100), err,
              "carveout") &&
           // the largest shared-memory carveout for P2P too, so an SM running three P2P CTAs has
           // room for the stored-M2L CTA beside them
           ck(cudaFuncSetAttribute(p2p_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100), err, "carveout");
  }
  {  // which chain is the critical path: the near field at its rate alone (4.2e11 point pairs / s)
     // against the far field's bytes (stored M2L blocks + translation operators) at 6 TB/s; the
     // on-the-fly M2L shares the fp64 pipe with the P2P, so nothing is held back then
    const double t_near = (double)pk.p2p_pairs / 4.2e11;
    const double t_far = d.m2l_mat ? (16.0 * (double)pk.m2l_stored_entries + 16.0 * (double)pk.ops_len) / 6.0e12 : 0.0;
    d.near_after = t_far > 1.15 * t_near ? 2 : 0;
  }
  int prio_lo = 0, prio_hi = 0;
  ok = ok && ck(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi), err, "stream priorities") &&
       ck(cudaStreamCreateWithPriority(&d.s_far, cudaStreamNonBlocking, DAFMM_NEAR_HIGH ? prio_lo : prio_hi), err,
          "far stream") &&
       ck(cudaStreamCreateWithPriority(&d.s_near, cudaStreamNonBlocking, DAFMM_NEAR_HIGH ? prio_hi : prio_lo), err,
          "near stream") &&
       ck(cudaStreamCreateWithPriority(&d.s_leaf, cudaStreamNonBlocking, DAFMM_NEAR_HIGH ? prio_lo : prio_hi), err,
          "leaf M2L stream") &&
       ck(cudaEventCreateWithFlags(&d.ev_p2m, cudaEventDisableTiming), err, "P2M event") &&
       ck(cudaEventCreateWithFlags(&d.ev_leaf, cudaEventDisableTiming), err, "leaf M2L event") &&
       ck(cudaEventCreateWithFlags(&d.ev_fork, cudaEventDisableTiming), err, "fork event") &&
       ck(cudaEventCreateWithFlags(&d.ev_join_far, cudaEventDisableTiming), err, "join event") &&
       ck(cudaEventCreateWithFlags(&d.ev_join_near, cudaEventDisableTiming), err, "join event") &&
       alloc(d, &d.phi, plan.n, err) && alloc(d, &d.m2l_ticket, 2, err) && alloc(d, &d.m2l_flag, 1, err) && alloc(d, &d.x_t, plan.n, err) && alloc(d, &d.v_t, plan.n, err) && alloc(d, &d.mult, pk.n_mult, err) &&
       alloc(d, &d.loc, pk.n_loc, err) && alloc(d, &d.host_stage, 2 * plan.n, err);
  if (!ok) return DAFMM_ECUDA;
  return DAFMM_OK;
}

void free_plan(DevPlan& d) {
  for (cudaEvent_t* e : {&d.ev_fork, &d.ev_join_far, &d.ev_join_near, &d.ev_p2m, &d.ev_leaf})
    if (*e) {
      cudaEventDestroy(*e);
      *e = nullptr;
    }
  for (cudaStream_t* st : {&d.s_far, &d.s_near, &d.s_leaf})
    if (*st) {
      cudaStreamDestroy(*st);
      *st = nullptr;
    }
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
  if (!ck(cudaEventSynchronize(d.prof_ev[EV_END]), err, "profile event sync")) return DAFMM_ECUDA;
  auto el = [&](int a, int b, double& out) -> bool {
    float ms = 0.f;
    if (!ck(cudaEventElapsedTime(&ms, d.prof_ev[a], d.prof_ev[b]), err, "profile elapsed")) return false;
    out = ms;
    return true;
  };
  double t[kNumPasses], near_end = 0.0, far_end = 0.0;
  // gather | memsets + P2M | M2M | M2L | L2L | P2P (side stream) | combine | fork-to-join span
  if (!el(EV_START, EV_FORK, t[0]) || !el(EV_FORK, EV_M2M, t[1]) || !el(EV_M2M, EV_M2L, t[2]) ||
      !el(EV_M2L, EV_L2L, t[3]) || !el(EV_L2L, EV_FAR_END, t[4]) || !el(EV_NEAR0, EV_NEAR1, t[5]) ||
      !el(EV_JOIN, EV_END, t[6]) || !el(EV_FORK, EV_NEAR1, near_end) || !el(EV_FORK, EV_FAR_END, far_end))
    return DAFMM_ECUDA;
  t[7] = std::max(near_end, far_end);
  if (!el(EV_LEAF0, EV_LEAF1, t[8])) return DAFMM_ECUDA;
  if (d.prof_side_m2m) {  // M2M ran on its own stream between the LEAF marks
    t[2] = t[8];
    t[8] = 0.0;
  }
  for (int p = 0; p < kNumPasses; ++p) d.prof_ms[p] += t[p];
  ++d.prof_count;
  d.prof_pending = false;
  return DAFMM_OK;
}

// y = A x.  The near field (P2P) only needs the gathered vector, so it runs on the side stream
// concurrently with the far field (P2M, M2M, M2L, L2L) on the handle's stream; the combine
// (L2P + identity + scatter) joins both.  No host synchronisation.
int run_matvec(DevPlan& d, const double2* x, double2* y, unsigned mask, std::string& err) {
  const cudaStream_t s = d.stream;
  if (d.prof && harvest_profile(d, err) != DAFMM_OK) return DAFMM_ECUDA;
  auto mark = [&](int e, cudaStream_t st) {
    if (d.prof) cudaEventRecord(d.prof_ev[e], st);
  };
  const bool near = mask & 1u;
  const bool far = (mask & 2u) && d.n_mult > 0;
  const bool fork = near && far && d.s_far != nullptr;
  // fork: the far field runs on a high-priority internal stream so its short, latency-bound
  // translation kernels and the persistent M2L CTAs are scheduled ahead of the pending P2P
  // CTAs (low-priority stream) as SM slots free up; both join back on the caller's stream
  const cudaStream_t fs = fork ? d.s_far : s, ns = fork ? d.s_near : s;
  mark(EV_START, s);
  gather_kernel<<<grid_for(d.n, 256, 148 * 16), 256, 0, s>>>(d.n, d.perm, d.w_t, x, d.x_t, d.v_t);
  ++d.launches;
  mark(EV_FORK, s);
  if (fork) {
    cudaEventRecord(d.ev_fork, s);
    cudaStreamWaitEvent(d.s_far, d.ev_fork, 0);
    cudaStreamWaitEvent(d.s_near, d.ev_fork, 0);
  }
  if (far) {
    cudaMemsetAsync(d.mult, 0, sizeof(double2) * d.n_mult, fs);
    cudaMemsetAsync(d.loc, 0, sizeof(double2) * d.n_loc, fs);
    if (d.m2l_targets > 0 && !d.m2l_mat) cudaMemsetAsync(d.m2l_ticket, 0, 2 * sizeof(int), fs);
  }
  // M2M beside the deepest level's M2L (DAFMM_M2M_SIDE): that level's M2L reads only the leaves'
  // multipoles, so the one persistent stored-M2L launch starts right after P2M and takes those
  // targets first (they are packed first) while M2M runs on a third stream and then raises a flag;
  // the M2L producers wait for the flag before their first coarser target.
  const bool side_m2m = DAFMM_M2M_SIDE && far && d.s_leaf != nullptr && d.m2l_mat != nullptr && !d.m2l_sym &&
                        !DAFMM_LEAF_SPLIT && !d.m2m.empty() && d.m2l_leaf_targets > 0 &&
                        d.m2l_leaf_targets < d.m2l_targets;
  if (side_m2m) cudaMemsetAsync(d.m2l_flag, 0, sizeof(int), fs);
  mark(EV_P2M, fs);
  if (far) d.launches += launch_translate(d, d.p2m, d.v_t, d.mult, 0, fs);  // P2M
  // The P2P can be held back until P2M (1) or M2M (2) has finished, so that the short translation
  // kernels at the head of the far chain do not queue behind resident P2P CTAs.  It pays when the
  // far chain is the critical path (d.near_after, chosen per plan in upload_plan: C4 3.24 -> 3.08 ms,
  // C3 0.95 -> 0.90 ms) and not when the P2P is (C5: 8.81 -> 8.90 ms); profiles/README.md, r2aa.
  const int near_after = DAFMM_NEAR_AFTER >= 0 ? DAFMM_NEAR_AFTER : d.near_after;
  if (near_after == 1 && fork && !side_m2m && !DAFMM_LEAF_SPLIT) {
    cudaEventRecord(d.ev_p2m, fs);
    cudaStreamWaitEvent(ns, d.ev_p2m, 0);
  }
  // M2L over targets [t0, t1) on stream st (ticket slot k for the on-the-fly kernel)
  auto m2l = [&](int t0, int t1, int k, cudaStream_t st) {
    if (t1 <= t0) return;
    if (d.m2l_sym) {  // one block per node pair: row sums and column sums (R22)
      m2l_pairw_kernel<<<d.m2l_pair_grid, kPWThreads, kPWDynSmem, st>>>(
          t1 - t0, d.m2l_loc_off + t0, d.m2l_rows + t0, d.m2l_stream_ptr + t0, d.m2l_stream_idx, d.m2l_mat_off + t0,
          d.m2l_self_moff + t0, d.m2l_src_ptr + t0, d.m2l_src_off, d.m2l_src_cnt, d.m2l_mat, d.mult, d.loc,
          d.m2l_slots);
      if (d.m2l_in_nodes > 0) {
        m2l_slot_gather_kernel<<<(d.m2l_in_nodes + 7) / 8, 256, 0, st>>>(d.m2l_in_nodes, d.m2l_in_lo, d.m2l_in_rows,
                                                                        d.m2l_in_ptr, d.m2l_in_off, d.m2l_slots,
                                                                        d.loc);
        ++d.launches;
      }
    } else if (d.m2l_mat) {  // from the stored blocks
      m2l_stored_kernel<<<d.m2l_store_grid, kMSThreads, kMSDynSmem, st>>>(
          t1 - t0, d.m2l_loc_off + t0, d.m2l_rows + t0, d.m2l_stream_ptr + t0, d.m2l_stream_idx, d.m2l_mat_off + t0,
          d.m2l_mat, d.mult, d.loc, side_m2m ? d.m2l_leaf_targets : t1 - t0, side_m2m ? d.m2l_flag : nullptr);
    } else {  // kernel entries on the fly, persistent CTAs
      m2l_kernel<<<d.m2l_grid, kM2LThreads, 0, st>>>(t1 - t0, d.m2l_ticket + k, d.m2l_loc_off + t0, d.m2l_rows + t0,
                                                      d.m2l_stream_ptr + t0, d.m2l_stream_idx, d.m2l_item_ptr + t0,
                                                      d.m2l_item_code, d.m2l_item_begin, d.m2l_item_end, d.ti_xy,
                                                      d.so_xy, d.mult, d.loc);
    }
    ++d.launches;
  };
  // DAFMM_LEAF_SPLIT: the deepest level's M2L needs only the leaves' multipoles, so it can run
  // on its own stream beside M2M and the coarser M2L / L2L, joining before the L2L into the
  // deepest level (the only other kernel touching those local expansions).  Measured slower
  // with stored blocks at C4 (4.18 vs 3.71 ms: two M2L launches crowd the P2P; profiles/README.md),
  // so it is off by default.
  const int nleaf = (DAFMM_LEAF_SPLIT && far && fork && d.l2l.size() > 0 && !d.m2l_sym) ? d.m2l_leaf_targets : 0;
  if (nleaf > 0) {
    cudaEventRecord(d.ev_p2m, fs);
    cudaStreamWaitEvent(d.s_leaf, d.ev_p2m, 0);
    mark(EV_LEAF0, d.s_leaf);
    m2l(0, nleaf, 0, d.s_leaf);
    mark(EV_LEAF1, d.s_leaf);
    cudaEventRecord(d.ev_leaf, d.s_leaf);
  } else if (!side_m2m) {
    mark(EV_LEAF0, fs);
    mark(EV_LEAF1, fs);
  }
  mark(EV_M2M, fs);
  if (side_m2m) {
    cudaEventRecord(d.ev_p2m, fs);
    cudaStreamWaitEvent(d.s_leaf, d.ev_p2m, 0);
    mark(EV_LEAF0, d.s_leaf);
    for (auto& b : d.m2m) d.launches += launch_translate(d, b, d.mult, d.mult, 0, d.s_leaf);  // M2M
    set_flag_kernel<<<1, 1, 0, d.s_leaf>>>(d.m2l_flag);
    ++d.launches;
    mark(EV_LEAF1, d.s_leaf);
    cudaEventRecord(d.ev_leaf, d.s_leaf);
  } else if (far) {
    for (auto& b : d.m2m) d.launches += launch_translate(d, b, d.mult, d.mult, 0, fs);  // M2M
  }
  if (near_after == 2 && fork && !side_m2m && !DAFMM_LEAF_SPLIT) {
    cudaEventRecord(d.ev_p2m, fs);
    cudaStreamWaitEvent(ns, d.ev_p2m, 0);
  }
  mark(EV_M2L, fs);
  if (far) m2l(nleaf, d.m2l_targets, 1, fs);  // M2L: all (remaining) levels
  if (side_m2m) cudaStreamWaitEvent(fs, d.ev_leaf, 0);  // join the M2M stream
  mark(EV_L2L, fs);
  if (far)
    for (size_t i = 0; i < d.l2l.size(); ++i) {  // L2L
      if (nleaf > 0 && i + 1 == d.l2l.size()) cudaStreamWaitEvent(fs, d.ev_leaf, 0);
      d.launches += launch_translate(d, d.l2l[i], d.loc, d.loc, 1, fs);
    }
  mark(EV_FAR_END, fs);
  mark(EV_NEAR0, ns);
  if (near) {  // P2P
    p2p_kernel<<<d.nleaves, kNearThreads, 0, ns>>>(d.leaf_begin, d.leaf_end, d.near_ptr, d.near_begin, d.near_end,
                                                   d.leaf_band, d.pts_t, d.v_t, d.phi, d.p2p_sym,
                                                   d.leaf_slot_base, d.slots, d.slot_total);
    ++d.launches;
  }
  mark(EV_NEAR1, ns);
  if (fork) {
    cudaEventRecord(d.ev_join_far, d.s_far);
    cudaEventRecord(d.ev_join_near, d.s_near);
    cudaStreamWaitEvent(s, d.ev_join_far, 0);
    cudaStreamWaitEvent(s, d.ev_join_near, 0);
  }
  mark(EV_JOIN, s);
  combine_kernel<<<d.nleaves, kCombineThreads, 0, s>>>(d.leaf_begin, d.leaf_end, d.leaf_loc_off, d.leaf_rank,
                                                        d.leaf_U_off, d.ops, d.loc, d.phi, d.x_t, d.qk2_t, d.D_t,
                                                        d.perm, y, d.kernel_mode, near ? 1 : 0, far ? 1 : 0,
                                                        d.p2p_sym ? d.in_ptr : nullptr, d.in_off, d.slots,
                                                        d.slot_total);
  ++d.launches;
  mark(EV_END, s);
  d.prof_side_m2m = side_m2m;
  if (d.prof) d.prof_pending = true;
  return ck(cudaGetLastError(), err, "matvec launch") ? DAFMM_OK : DAFMM_ECUDA;
}

// ============================================================================================
// Restarted GMRES (reading R14) with CGS2 orthogonalisation (R20) on the device.
int run_gmres(DevPlan& d, const double2* f, double2* psi, double tol, int maxit, int restart, int* iters_out,
              double* relres_out, double* history, std::string& err, const Precond& prec) {
  const int64_t n = d.n;
  const int m = restart > 0 ? restart : 50;
  if (m > 255) { err = "restart must be <= 255"; return DAFMM_EINVAL; }  // combine_kernel's coefficient cache
  cudaStream_t s = d.stream;
  const int nb = grid_for(n, kVecThreads, 296);
  if (d.gm_restart != m) {
    // (re)size the workspace for this restart: the previous one (another restart) is released
    for (void** p : {(void**)&d.gm_V, (void**)&d.gm_w, (void**)&d.gm_r, (void**)&d.gm_h, (void**)&d.gm_part,
                     (void**)&d.gm_z})
      release(d, p);
    if (d.gm_hostbuf) cudaFreeHost(d.gm_hostbuf);
    d.gm_hostbuf = nullptr;
    d.gm_restart = m;
    if (!alloc(d, &d.gm_V, (size_t)(m + 1) * n, err) || !alloc(d, &d.gm_w, n, err) || !alloc(d, &d.gm_r, n, err) ||
        !alloc(d, &d.gm_h, 3 * (m + 2), err) || !alloc(d, &d.gm_part, (size_t)nb * (m + 2), err) ||
        !alloc(d, &d.gm_z, n, err))
      return DAFMM_ECUDA;
    if (!ck(cudaMallocHost((void**)&d.gm_hostbuf, sizeof(double2) * 3 * (m + 2)), err, "cudaMallocHost"))
      return DAFMM_ECUDA;
    d.gm_part_blocks = nb;
  }
  const int stride = m + 2;
  // multi-dot blocks per vector group: fewer, longer blocks (their 2-D grid already has a
  // block row per group of kMD basis vectors)
  const int nb_md = std::min(nb, DAFMM_MD_BLOCKS);
  auto norm = [&](const double2* v, double& out) -> bool {
    norm2_kernel<<<nb, kVecThreads, 0, s>>>(n, v, d.gm_part);
    reduce_launch(nb, 1, d.gm_part, 1, d.gm_h, s);
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
  d.gm_reorth = 0;
  bool converged = false;
  // r = f (psi0 = 0).  Convergence is decided on the true residual r = f - A psi (recomputed at
  // every restart): a cycle that ends because its implicit (Givens) residual reached tol starts a
  // new cycle when the true residual has not (rounding makes the two differ slightly)
  cudaMemcpyAsync(d.gm_r, f, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s);
  while (true) {
    double beta;
    if (!norm(d.gm_r, beta)) return DAFMM_ECUDA;
    if (beta / bnorm <= tol) { converged = true; break; }
    if (iters >= maxit) break;
    axpby_kernel<<<nb, kVecThreads, 0, s>>>(n, 1.0 / beta, d.gm_r, 0.0, d.gm_r, d.gm_V);
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int k = 0;
    for (int j = 0; j < m; ++j) {
      double2* vj = d.gm_V + (int64_t)j * n;
      double2* vj1 = d.gm_V + (int64_t)(j + 1) * n;
      // right preconditioning (reading HR4): w = A M^{-1} v_j
      if (prec) {
        if (prec(vj, d.gm_z, err) != DAFMM_OK) return DAFMM_ECUDA;
        if (run_matvec(d, d.gm_z, d.gm_w, 3u, err) != DAFMM_OK) return DAFMM_ECUDA;
      } else if (run_matvec(d, vj, d.gm_w, 3u, err) != DAFMM_OK) {
        return DAFMM_ECUDA;
      }
      ++iters;
      // CGS2 (reading R20): two passes of h = V^H w, w -= V h, one host synchronisation.  (A DGKS
      // test that skips the second pass was measured: the projection cancels ||w|| below 1/sqrt(2)
      // in 98% of the C3 iterations, so it only added a synchronisation; profiles/README.md.)
      for (int pass = 0; pass < 2; ++pass) {
        multidot_kernel<<<dim3(nb_md, (j + 1 + kMD - 1) / kMD), kVecThreads, 0, s>>>(n, j + 1, d.gm_V, d.gm_w,
                                                                                    d.gm_part, stride);
        reduce_launch(nb_md, j + 1, d.gm_part, stride, d.gm_h + pass * (m + 2), s);
        combine_kernel<<<nb, kVecThreads, 0, s>>>(n, j + 1, d.gm_V, d.gm_h + pass * (m + 2), -1.0, d.gm_w);
      }
      ++d.gm_reorth;
      norm2_kernel<<<nb, kVecThreads, 0, s>>>(n, d.gm_w, d.gm_part);
      reduce_launch(nb, 1, d.gm_part, 1, d.gm_h + 2 * (m + 2), s);
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
      if (res <= tol || iters >= maxit || hnext == 0.0) break;
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
    if (prec) {  // psi += M^{-1} (V y)
      cudaMemsetAsync(d.gm_z, 0, sizeof(double2) * n, s);
      combine_kernel<<<nb, kVecThreads, 0, s>>>(n, k, d.gm_V, d.gm_h, 1.0, d.gm_z);
      if (prec(d.gm_z, d.gm_z, err) != DAFMM_OK) return DAFMM_ECUDA;
      axpby_kernel<<<nb, kVecThreads, 0, s>>>(n, 1.0, psi, 1.0, d.gm_z, psi);
    } else {
      combine_kernel<<<nb, kVecThreads, 0, s>>>(n, k, d.gm_V, d.gm_h, 1.0, psi);
    }
    // r = f - A psi
    if (run_matvec(d, psi, d.gm_w, 3u, err) != DAFMM_OK) return DAFMM_ECUDA;
    axpby_kernel<<<nb, kVecThreads, 0, s>>>(n, 1.0, f, -1.0, d.gm_w, d.gm_r);
    if (!ck(cudaStreamSynchronize(s), err, "sync")) return DAFMM_ECUDA;
  }
  double rn;
  if (!norm(d.gm_r, rn)) return DAFMM_ECUDA;  // gm_r = f - A psi of the final iterate
  *iters_out = iters;
  *relres_out = rn / bnorm;
  return (converged && rn / bnorm <= tol) ? DAFMM_OK : DAFMM_NOT_CONVERGED;
}

int h0_eval(const double* z2, double2* out, int64_t n, int code, cudaStream_t s, std::string& err) {
  if (n == 0) return DAFMM_OK;
  const int64_t blocks = std::min<int64_t>((n + 128 * kH0EvalTB - 1) / (128 * kH0EvalTB), 148 * 16);
  h0_eval_kernel<<<(int)blocks, 128, 0, s>>>(z2, out, n, code);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    err = std::string("h0_eval_kernel: ") + cudaGetErrorString(e);
    return DAFMM_ECUDA;
  }
  return DAFMM_OK;
}

}  // namespace dafmm
