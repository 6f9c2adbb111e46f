// Micro test: one tcgen05.mma.cta_group::1.kind::tf32 tile, D[128 x N] =
// A[128 x 16] . B[N x 16]^T, operands K-major in shared memory without
// swizzle (8-row x 16-byte core matrices), accumulator in TMEM, read back
// with tcgen05.ld.32x32b.  Checks the descriptor / layout conventions used
// by the chamfer tensor-core kernel against a CPU product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma umma_tf32.cu && ./umma
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

constexpr int M = 128, N = 208, K = 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// element (r, k) of a K-major operand with R rows: core matrices of 8 rows x 4
// tf32 (16 B); K-adjacent core matrices LBO = 128 B apart, 8-row groups
// SBO = (K / 4) * 128 B apart
__host__ __device__ __forceinline__ int kmajor_off(int r, int k) {
  return (r >> 3) * (K / 4) * 128 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4;
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100)
  return d;                // base offset 0, lbo mode 0, SWIZZLE_NONE
}

__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4)                 // D format F32
         | (2u << 7) | (2u << 10)  // A, B format TF32
         | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);  // K-major A and B
}

__global__ void umma_test(const float* A, const float* B, float* D, int swap_lbo_sbo) {
  __shared__ __align__(1024) unsigned char sa[M * K * 4];
  __shared__ __align__(1024) unsigned char sb[N * K * 4];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<float*>(sa + kmajor_off(r, k)) = A[i];
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<float*>(sb + kmajor_off(r, k)) = B[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n");  // st.shared -> async proxy (MMA operand reads)
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const uint32_t lbo = swap_lbo_sbo ? (K / 4) * 128 : 128, sbo = swap_lbo_sbo ? 128 : (K / 4) * 128;
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(M, N);
#pragma unroll
    for (int ks = 0; ks < K / 8; ++ks) {
      const uint64_t ad = smem_desc(smem_u32(sa) + ks * 256, lbo, sbo);
      const uint64_t bd = smem_desc(smem_u32(sb) + ks * 256, lbo, sbo);
      const uint32_t acc = ks > 0;
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
          " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)));
  }
  // wait for the MMA
  asm volatile(
      "{\n .reg .pred P1;\n WAIT:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT;\n}\n" ::"r"(smem_u32(&bar)),
      "r"(0));
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // warp w reads TMEM lanes [32w, 32w+32): thread = row
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(256));
}

__global__ void umma_rate(const float* A, const float* B, long long* cyc, int reps, int n_cols) {
  __shared__ __align__(1024) unsigned char sa[M * K * 4];
  __shared__ __align__(1024) unsigned char sb[256 * K * 4];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += blockDim.x) *reinterpret_cast<float*>(sa + kmajor_off(i / K, i % K)) = A[i];
  for (int i = tid; i < 256 * K; i += blockDim.x)
    *reinterpret_cast<float*>(sb + kmajor_off(i / K, i % K)) = B[i % (N * K)];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(M, n_cols);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int ks = 0; ks < K / 8; ++ks) {
        const uint64_t ad = smem_desc(smem_u32(sa) + ks * 256, 128, (K / 4) * 128);
        const uint64_t bd = smem_desc(smem_u32(sb) + ks * 256, 128, (K / 4) * 128);
        const uint32_t acc = (r | ks) > 0;
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)));
    asm volatile(
        "{\n .reg .pred P1;\n W2:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra W2;\n}\n" ::"r"(smem_u32(&bar)),
        "r"(0));
    cyc[0] = clock64() - t0;
    // single tile latency
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
  }
  __syncthreads();
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(256));
}

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N), R(M * N);
  srand(1);
  // values with <= 10 mantissa bits: tf32-exact, products exact in fp32
  auto rnd = [] { return (float)((rand() % 2048) - 1024) / 256.0f; };
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[n * K + k];
      R[m * N + n] = (float)s;
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  for (int swap = 0; swap < 2; ++swap) {
    cudaMemset(dD, 0, D.size() * 4);
    umma_test<<<1, 128>>>(dA, dB, dD, swap);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("swap=%d: CUDA error %s\n", swap, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    int bad = 0;
    for (int i = 0; i < M * N; ++i) {
      const double err = fabs((double)D[i] - R[i]);
      maxerr = fmax(maxerr, err);
      bad += err > 1e-3;
    }
    printf("swap_lbo_sbo=%d: max |D - ref| = %g, %d / %d mismatches; D[0]=%g ref %g, D[last]=%g ref %g\n", swap,
           maxerr, bad, M * N, D[0], R[0], D[M * N - 1], R[M * N - 1]);
  }
  long long* dc;
  cudaMalloc(&dc, 8);
  for (int n : {208, 256}) {
    for (int reps : {1, 16, 256}) {
      umma_rate<<<1, 128>>>(dA, dB, dc, reps, n);
      cudaDeviceSynchronize();
      long long cy;
      cudaMemcpy(&cy, dc, 8, cudaMemcpyDeviceToHost);
      const double macs = (double)reps * M * n * K;
      printf("N=%d reps=%d: %lld cycles, %.1f MAC/clk (tile = %d MACs)\n", n, reps, cy, macs / cy, M * n * K);
    }
  }
  return 0;
}
