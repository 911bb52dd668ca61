// Small dense complex fp64 helpers shared by the device setup kernels (setup_device.cu,
// hodlr.cu): complex arithmetic on double2 and a shared-memory LU with partial pivoting.
#pragma once
#include <cuda_runtime.h>

namespace dafmm {

static __device__ __forceinline__ void cfms2(double2& acc, double2 a, double2 b) {  // acc -= a b
  acc.x -= a.x * b.x - a.y * b.y;
  acc.y -= a.x * b.y + a.y * b.x;
}
static __device__ __forceinline__ void cfma2(double2& acc, double2 a, double2 b) {  // acc += a b
  acc.x += a.x * b.x - a.y * b.y;
  acc.y += a.x * b.y + a.y * b.x;
}
static __device__ __forceinline__ double2 cdiv2(double2 a, double2 b) {
  const double d = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
static __device__ __forceinline__ double cabs2h(double2 a) { return a.x * a.x + a.y * a.y; }

// In-place LU with partial pivoting of the n x n column-major matrix M in shared memory (all
// threads of the block; ties of the pivot search go to the lower row).  perm[i] = original
// row of row i of P M.  Sets *status on an exactly zero pivot.
static __device__ void block_lu(double2* M, int n, int* perm, int* s_piv, int* status) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < n; i += nt) perm[i] = i;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    if (tid < 32) {
      double best = -1.0;
      int bi = -1;
      for (int i = k + tid; i < n; i += 32) {
        const double a = cabs2h(M[k * n + i]);
        if (a > best) { best = a; bi = i; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (oi >= 0 && (bi < 0 || ob > best || (ob == best && oi < bi))) { best = ob; bi = oi; }
      }
      if (tid == 0) {
        *s_piv = bi;
        if (!(best > 0.0)) atomicExch(status, 1);
      }
    }
    __syncthreads();
    const int p = *s_piv;
    if (p != k) {
      for (int j = tid; j < n; j += nt) {
        const double2 a = M[j * n + k];
        M[j * n + k] = M[j * n + p];
        M[j * n + p] = a;
      }
      if (tid == 0) {
        const int a = perm[k];
        perm[k] = perm[p];
        perm[p] = a;
      }
    }
    __syncthreads();
    const double2 piv = M[k * n + k];
    for (int i = k + 1 + tid; i < n; i += nt) M[k * n + i] = cdiv2(M[k * n + i], piv);
    __syncthreads();
    const int m = n - k - 1;
    for (int e = tid; e < m * m; e += nt) {
      const int i = k + 1 + e % m, j = k + 1 + e / m;
      cfms2(M[j * n + i], M[k * n + i], M[j * n + k]);
    }
    __syncthreads();
  }
}

}  // namespace dafmm
