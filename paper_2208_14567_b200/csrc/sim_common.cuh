// Device helpers shared by the simulation kernels (sim.cu: warp-per-candidate
// replay and path writes; screen.cu: lane-per-candidate validity screen).
#pragma once
#include "common.cuh"
#include <cuda_fp16.h>

namespace la {

__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
// shared-space accesses by 32-bit address (one IADD per access in the dyad
// loop instead of generic-pointer arithmetic); "memory" keeps them ordered
// with the other shared-memory accesses of the warp
__device__ __forceinline__ float2 lds_f2(uint32_t a) {
  float2 v;
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_f2(uint32_t a, float2 v) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_f4(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 lds_u4(uint32_t a) {
  uint4 v;
  asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
// flag = 1 unless v >= bound (so a NaN sets it): one FSETP and a predicated move
__device__ __forceinline__ void flag_below(unsigned& flag, float v, float bound) {
  asm("{\n\t.reg .pred p;\n\tsetp.ltu.f32 p, %1, %2;\n\t@p mov.u32 %0, 1;\n\t}" : "+r"(flag) : "f"(v), "f"(bound));
}
__device__ __forceinline__ double2 lds_d2(uint32_t a) {
  double2 v;
  asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_d2(uint32_t a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
// 8-byte asynchronous global -> shared copy (LDGSTS) and its completion
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// fp32 screen error model (solve32): input rounding of the f64 pose and
// crank tip, per-dyad rounding of the fp32 evaluation (unit-box magnitudes,
// rsqrt/sqrt approximations included), and the margin's sensitivity factor
// with a safety factor of 2 on the first-order bound.
constexpr float kErr0 = 2e-7f;
constexpr float kErrStep = 5e-7f;
constexpr float kMarginK = 3.0f;
// fp16 storage of error bounds (8-byte-slot screens): rounded up on store
// so a stored bound never shrinks (bounds below 6.1e-5 are subnormal halves,
// absolute resolution 6e-8 -- far below the 2e-6 ambiguity floor)
__device__ __forceinline__ float lds_h16(uint32_t a) {
  unsigned short h;
  asm("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(a) : "memory");
  return __half2float(__ushort_as_half(h));
}
__device__ __forceinline__ void sts_h16(uint32_t a, float v) {
  const unsigned short h = __half_as_ushort(__float2half_ru(v));
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(h) : "memory");
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// f64 reciprocal square root and reciprocal: the MUFU seeds (RSQ64H / RCP64H,
// relative error 1e-6 measured, tools/micro/f64_seeds.cu) refined by one
// third-order step each -- Halley's y (1 + e/2 + 3 e^2/8), e = 1 - x y^2, and
// y (1 + e + e^2), e = 1 - x y -- to 1 ulp (2.2e-16 measured; two Newton
// steps give 2.6e-16 with two more DFMA).  Not correctly rounded, see
// dyads_f64.
__device__ __forceinline__ double rsqrt_f64(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y * y, 1.0);
  return fma(y * e, fma(0.375, e, 0.5), y);
}
__device__ __forceinline__ double rcp_f64(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);
  return fma(y, fma(e, e, e), y);
}

// exact-mode triage of an f64 replay: a fast (DFMA, Newton rsqrt) pass
// decides unless one of its lock tests is within this distance of its
// threshold; then the angle is redone in numpy's operation order
constexpr double kExactTriage = 1e-7;

// i-th fine angle of the coarse-first order (t = 4k + 1, 4k + 2, 4k + 3)
__device__ __forceinline__ int fine_angle(int i) { return (i / 3) * 4 + 1 + (i % 3); }

}  // namespace la
