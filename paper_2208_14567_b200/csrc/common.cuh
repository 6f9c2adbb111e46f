// Shared helpers for the LINKS B200 kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include "links_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "links_b200 is built for sm_100a only"
#endif

namespace la {

constexpr unsigned FULL = 0xffffffffu;

// thread-local last-error text (la_last_error)
void set_error(const char* fmt, ...);

inline int fail(int code, const char* fmt, ...) {
  char buf[256];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  set_error("%s", buf);
  return code;
}

inline int cuda_status(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", where, cudaGetErrorString(e));
    return static_cast<int>(e);
  }
  return 0;
}

// SM count of the current device, cached per device
int sm_count();

__device__ __forceinline__ float2 ld_f2(const float2* p) { return *p; }

__device__ __forceinline__ void st_cs(float2* p, float2 v) { __stcs(p, v); }

// exact f64 ops without contraction (mirror numpy's operation order)
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// hypot for finite binary64 with the algorithm of glibc's __ieee754_hypot
// (Borges, "An Improved Algorithm for hypot(a,b)", 2019: corrected square
// root, the non-FMA kernel), the function numpy.hypot calls on Linux; explicit
// round-to-nearest ops so nothing is contracted.  Provenance: restated from
// the published algorithm to reproduce np.hypot bit for bit, not copied from
// glibc's sources (LGPL-2.1); bit-identical to np.hypot (checked on 2e7
// pairs, tests/test_gpu_filter.py, tests/test_gpu_solver.py).
__device__ __forceinline__ double np_hypot(double x, double y) {
  x = fabs(x);
  y = fabs(y);
  const double ax = x < y ? y : x;
  const double ay = x < y ? x : y;
  if (ay <= __dmul_rn(ax, 0x1p-54)) return __dadd_rn(ax, ay);
  double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
  double t1, t2;
  if (h <= __dmul_rn(2.0, ay)) {
    const double d = __dsub_rn(h, ay);
    t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, d), ax));
    t2 = __dmul_rn(__dsub_rn(d, __dmul_rn(2.0, __dsub_rn(ax, ay))), d);
  } else {
    const double d = __dsub_rn(h, ax);
    t1 = __dmul_rn(__dmul_rn(2.0, d), __dsub_rn(ax, __dmul_rn(2.0, ay)));
    t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, d), ay), ay), __dmul_rn(d, d));
  }
  return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}

}  // namespace la
