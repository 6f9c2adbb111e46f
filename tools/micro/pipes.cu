// Throughput microbenchmark of FP32 instruction forms on sm_100a (one SM's worth of warps).
#include <cstdio>
#include <cuda_runtime.h>
#define N_ITER 4096
template <int MODE>
__global__ void k(float* out, float a, float b, int iters) {
  float2 x[8]; float s[8];
  for (int i = 0; i < 8; ++i) { x[i] = make_float2(a + i + threadIdx.x, b - i); s[i] = a * i + b; }
  float2 c2 = make_float2(a, b);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) x[i] = __ffma2_rn(x[i], c2, x[(i + 1) & 7]);                    // pair,pair,pair
      if (MODE == 1) x[i] = __ffma2_rn(x[i], make_float2(s[i], s[i]), make_float2(s[(i+3)&7], s[(i+3)&7])); // pair,bcast,bcast
      if (MODE == 2) s[i] = fmaf(s[i], a, s[(i + 1) & 7]);                           // scalar 3-reg
      if (MODE == 3) s[i] = fminf(fminf(s[i], s[(i + 1) & 7]), s[(i + 2) & 7]);      // FMNMX3
      if (MODE == 4) x[i] = __fadd2_rn(x[i], x[(i + 1) & 7]);                        // FADD2
      if (MODE == 5) { x[i] = __ffma2_rn(x[i], c2, x[(i + 1) & 7]); s[i] = fminf(fminf(s[i], s[(i + 1) & 7]), s[(i + 2) & 7]); }
      if (MODE == 6) { x[i].x = fmaf(x[i].x, a, x[(i + 1) & 7].x); s[i] = fminf(fminf(s[i], s[(i + 1) & 7]), s[(i + 2) & 7]); }
      if (MODE == 7) { x[i].x = fmaf(x[i].x, a, x[(i + 1) & 7].x); x[i].y = fmaf(x[i].y, b, x[(i + 2) & 7].y); s[i] = fminf(fminf(s[i], s[(i + 1) & 7]), s[(i + 2) & 7]); }
      if (MODE == 8) { x[i].x = fmaf(x[i].x, a, x[(i + 1) & 7].x); s[i] = fminf(s[i], s[(i + 1) & 7]); }
      if (MODE == 10) { s[i] = __int_as_float(__reduce_min_sync(0xffffffffu, __float_as_int(s[i]) + i)); }
      if (MODE == 11) { x[i].x = fmaf(x[i].x, a, x[(i + 1) & 7].x); x[i].y = fmaf(x[i].y, b, x[(i + 2) & 7].y); x[(i+4)&7].x = fmaf(x[i].y, a, x[(i + 3) & 7].x); s[i] = __int_as_float(__reduce_min_sync(0xffffffffu, __float_as_int(s[i]) + i)); }
      if (MODE == 9) { x[i] = __ffma2_rn(x[i], make_float2(s[(i+5)&7], s[(i+5)&7]), make_float2(s[(i+3)&7], s[(i+3)&7])); s[i] = fminf(fminf(s[i], s[(i + 1) & 7]), s[(i + 2) & 7]); }
    }
  }
  float r = 0; for (int i = 0; i < 8; ++i) r += x[i].x + x[i].y + s[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int MODE> void run(const char* name, int warps) {
  float* out; cudaMalloc(&out, 148 * 1024 * 4 * 8);
  int iters = N_ITER;
  k<MODE><<<148, warps * 32>>>(out, 1.0f, 2.0f, 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<148, warps * 32>>>(out, 1.0f, 2.0f, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double instr = 148.0 * warps * iters * 8 * (MODE == 5 || MODE == 6 || MODE == 8 || MODE == 9 ? 2 : MODE == 7 ? 3 : MODE == 11 ? 4 : 1);
  double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-28s warps/SM=%2d  warp-instr per SM-cycle = %.3f  (%.1f us)\n", name, warps, instr / 148 / cyc, ms * 1e3);
  cudaFree(out);
}
int main() {
  for (int w : {16, 32}) {
    run<10>("REDUX.MIN.S32", w);
    run<11>("3 FFMA + REDUX", w);
  }
  return 0;
}
