// TMEM read throughput on sm_100a: tcgen05.ld.32x32b.x32 (+ wait) issued by
// W warps of one CTA per SM (all SMs), with and without an FMNMX3 row-min
// over the loaded registers.  Sets the ceiling of any chamfer that takes its
// squared distances from tcgen05 accumulators: every distance is read out
// of TMEM once per direction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_ld tmem_ld.cu && ./tmem_ld
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

#define LD32(v, addr)                                                                                         \
  asm volatile(                                                                                               \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"       \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"                            \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),      \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), \
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),           \
        "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),           \
        "=r"(v[30]), "=r"(v[31])                                                                              \
      : "r"(addr))

// MODE 0: loads only (one wait per 2 loads); MODE 1: loads + FMNMX3 row min
template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base;
  // warp w reads lane quarter (w & 3), column block 64 * (w >> 2) (mod 512)
  const uint32_t base = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((64 * (warp >> 2)) & 511);
  float m0 = 3.0e38f, m1 = 3.0e38f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t a[32], b[32];
    LD32(a, base);
    LD32(b, base + 32);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    if (MODE == 1) {
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        m0 = fminf(fminf(m0, __uint_as_float(a[j])), __uint_as_float(a[j + 1]));
        m1 = fminf(fminf(m1, __uint_as_float(b[j])), __uint_as_float(b[j + 1]));
      }
    } else {
      m0 = fminf(m0, __uint_as_float(a[it & 31]));
      m1 = fminf(m1, __uint_as_float(b[(it + 7) & 31]));
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = fminf(m0, m1);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(512));
}

template <int MODE>
void run(int warps, int sms) {
  const int iters = 4096;
  float* out;
  long long* cyc;
  cudaMalloc(&out, (size_t)sms * warps * 32 * 4);
  cudaMalloc(&cyc, sms * 8);
  k<MODE><<<sms, warps * 32>>>(out, cyc, 16);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<sms, warps * 32>>>(out, cyc, iters);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(err));
    return;
  }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c0;
  cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
  // bytes read from TMEM per SM: warps * iters * 2 loads * 32 lanes * 32 cols * 4 B
  const double bytes = (double)warps * iters * 2 * 32 * 32 * 4;
  printf("mode %d warps %2d: %.1f B/clk/SM (clock64), %.2f TB/s chip (events, %d SMs), %.3f ms\n", MODE, warps,
         bytes / (double)c0, bytes * sms / (ms * 1e-3) / 1e12, sms, ms);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 16, 32}) run<0>(w, sms);
  for (int w : {4, 8, 16, 32}) run<1>(w, sms);
  return 0;
}
