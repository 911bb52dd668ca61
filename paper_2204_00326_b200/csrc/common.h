// Shared product-side definitions: host/device qualifiers, error plumbing, complex helpers.
#pragma once
#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define DAFMM_HD __host__ __device__ __forceinline__
#else
#define DAFMM_HD inline
#endif

namespace dafmm {

// Complex fp64 value in registers / memory: identical layout to double2 and complex128.
struct alignas(16) cplx {
  double re, im;
};

DAFMM_HD cplx cmul(cplx a, cplx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
DAFMM_HD cplx cadd(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
// acc += a * b
DAFMM_HD void cfma(cplx& acc, cplx a, cplx b) {
  acc.re = fma(a.re, b.re, fma(-a.im, b.im, acc.re));
  acc.im = fma(a.re, b.im, fma(a.im, b.re, acc.im));
}

}  // namespace dafmm
