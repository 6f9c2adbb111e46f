// Issue throughput of small tcgen05.mma.kind::tf32 tiles (M = 128, K = 8)
// as a function of N, one CTA per SM on every SM, one issuing thread,
// destination rotating over 4 TMEM column blocks (no accumulate).  With
// LOADERS = 1, 16 other warps read TMEM (tcgen05.ld x32 + FMNMX3) from the
// whole allocation at the same time (the chamfer epilogue's traffic).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_small umma_small.cu && ./umma_small
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

template <int LOADERS, int MODE = 0>
__global__ void rate(long long* cyc, int reps, int n, int per_commit, int acc) {
  __shared__ __align__(1024) unsigned char sa[4 * 128 * 32];
  __shared__ __align__(1024) unsigned char sb[2 * 256 * 32];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tmem_base;
  __shared__ volatile int done;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 4 * 128 * 32 / 4; i += blockDim.x) reinterpret_cast<float*>(sa)[i] = 0.25f;
  for (int i = tid; i < 2 * 256 * 32 / 4; i += blockDim.x) reinterpret_cast<float*>(sb)[i] = 0.5f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    done = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  if (warp == (blockDim.x >> 5) - 1) {
    const uint32_t idesc = idesc_tf32(128, n);
    const uint64_t ad = smem_desc(smem_u32(sa), 128, 256), bd = smem_desc(smem_u32(sb), 128, 256);
    const long long t0 = clock64();
    if (MODE == 0) {
      if ((tid & 31) == 0) {
        for (int r = 0; r < reps; ++r) {
          const uint32_t d = tmem + (acc ? 0u : (uint32_t)((r & 1) * 256));
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
              "l"(ad), "l"(bd), "r"(idesc), "r"(acc && r > 0 ? 1 : 0));
        }
      }
    } else if (MODE >= 3) {
      // MODE 3: commit after every MMA (throughput); MODE 4: MMA + commit + wait (latency)
      uint32_t ph = 0;
      for (int r = 0; r < reps; ++r) {
        const uint32_t d = tmem + (uint32_t)((r & 1) * 256);
        const uint64_t ad2 = MODE >= 5 ? smem_desc(smem_u32(sa) + (r & 3) * 4096, 128, 256) : ad;
        const uint64_t bd2 = MODE >= 5 ? smem_desc(smem_u32(sb) + ((r >> 2) & 1) * 8192, 128, 256) : bd;
        if (MODE == 6) asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if (MODE == 7) asm volatile(
              "{\n .reg .pred P1;\n W4:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
              " @!P1 bra W4;\n}\n" ::"r"(smem_u32(&bar2)), "r"(1));
        asm volatile(
            "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
            " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 0;\n"
            " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n}\n" ::"r"(d),
            "l"(ad2), "l"(bd2), "r"(idesc), "r"(smem_u32(&bar)));
        if (MODE == 4) {
          asm volatile(
              "{\n .reg .pred P1;\n W3:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
              " @!P1 bra W3;\n}\n" ::"r"(smem_u32(&bar)), "r"(ph));
          ph ^= 1u;
        }
      }
    } else {
      const int U = MODE == 2 ? 4 : 1;
      for (int r = 0; r < reps; r += U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t d = tmem + (acc ? 0u : (uint32_t)(((r + u) & 1) * 256));
          asm volatile(
              "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
              " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
              "l"(ad + (uint64_t)(u * 0)), "l"(bd + (uint64_t)(u * 0)), "r"(idesc), "r"(acc && (r + u) > 0 ? 1 : 0));
        }
      }
    }
    if ((tid & 31) == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(&bar2)));
      asm volatile(
          "{\n .reg .pred P1;\n W2:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
          " @!P1 bra W2;\n}\n" ::"r"(smem_u32(&bar2)),
          "r"(0));
      cyc[blockIdx.x] = clock64() - t0;
      done = 1;
    }
  } else if (LOADERS && warp < 16) {
    const uint32_t base = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(32 * (warp >> 2));
    float m = 3e38f;
    while (!done) {
      for (int s = 0; s < 4; ++s) {
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
              "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
              "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
              "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(base + (uint32_t)(s * 128)));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; j += 2) m = fminf(fminf(m, __uint_as_float(v[j])), __uint_as_float(v[j + 1]));
      }
    }
    if (m == 1.2345f) cyc[gridDim.x + blockIdx.x] = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

template <int L, int MODE = 0>
void run(int sms, int n, int per_commit, int acc = 0, int threads = 17 * 32) {
  long long* cyc;
  cudaMalloc(&cyc, 2 * sms * 8);
  const int reps = 4096;
  rate<L, MODE><<<sms, threads>>>(cyc, 64, n, per_commit, acc);
  rate<L, MODE><<<sms, threads>>>(cyc, reps, n, per_commit, acc);
  cudaError_t e = cudaDeviceSynchronize();
  long long c0 = 0;
  cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return;
  }
  printf("mode %d grid %d threads %d loaders %d acc %d N %3d commit/%d: %7.1f cycles per MMA, %6.0f MAC/clk\n", MODE, sms, threads, L, acc, n, per_commit, (double)c0 / reps,
         128.0 * n * 8 * reps / c0);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int n : {128, 208}) run<1, 5>(sms, n, 4096, 0, 17 * 32);
  for (int n : {128, 208}) run<1, 6>(sms, n, 4096, 0, 17 * 32);
  for (int n : {128, 208}) run<1, 7>(sms, n, 4096, 0, 17 * 32);
  return 0;
}
