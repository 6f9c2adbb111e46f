// Inner-loop variants of the chamfer scan (one query in registers, curve in smem).
#include <cstdio>
#include <cuda_runtime.h>
#define FULL 0xffffffffu
constexpr int P = 200, QS = 7, NP = 3;

__device__ __forceinline__ float min3f(float a, float b, float c) { return fminf(fminf(a, b), c); }

// VAR 0: expansion f32x2, REDUX per a (current)
// VAR 1: same, no REDUX (rowmin skipped) -> upper bound
// VAR 2: expansion f32x2, 4 a per iteration, REDUX per a
// VAR 3: direct f32x2 (FADD2 FADD2 FMUL2 FFMA2), REDUX per a
// VAR 4: expansion, rows via smem transpose-reduce every 32 a (no REDUX)
template <int VAR>
__global__ void __launch_bounds__(256) k(const float4* __restrict__ exg, const float2* __restrict__ eng, int ncurves,
                                         float* out, const float2* __restrict__ q) {
  __shared__ float4 ex[8][112];
  __shared__ float2 en[8][112];
  __shared__ float rowbuf[8][33 * 32 / 2 + 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float2 qx[NP], qy[NP], qn[NP];
  float tx, ty, tn;
  for (int s = 0; s < NP; ++s) {
    float2 a = q[lane + 64 * s], b = q[lane + 64 * s + 32];
    qx[s] = make_float2(a.x, b.x); qy[s] = make_float2(a.y, b.y);
    qn[s] = make_float2(a.x * a.x + a.y * a.y, b.x * b.x + b.y * b.y);
  }
  tx = q[lane + 192].x; ty = q[lane + 192].y; tn = tx * tx + ty * ty;
  for (int i = lane; i < 112; i += 32) { ex[w][i] = exg[i]; en[w][i] = eng[i]; }
  __syncwarp();
  float acc = 0.f;
  for (int c = blockIdx.x * 8 + w; c < ncurves; c += gridDim.x * 8) {
    float2 cmin[NP]; float cmint = INFINITY;
    for (int s = 0; s < NP; ++s) cmin[s] = make_float2(INFINITY, INFINITY);
    float rsum = 0.f;
#pragma unroll 1
    for (int a0 = 0; a0 < 224; a0 += 32) {
#pragma unroll
      for (int u = 0; u < 32; u += 2) {
        const int i = (a0 + u) >> 1;
        const float4 e = ex[w][i]; const float2 n = en[w][i];
        float rm0 = INFINITY, rm1 = INFINITY;
#pragma unroll
        for (int s = 0; s < NP; ++s) {
          float2 w0, w1;
          if (VAR == 3) {
            float2 dx0 = __ffma2_rn(make_float2(e.x, e.x), make_float2(0.5f, 0.5f), qx[s]);
            float2 dy0 = __ffma2_rn(make_float2(e.z, e.z), make_float2(0.5f, 0.5f), qy[s]);
            float2 dx1 = __ffma2_rn(make_float2(e.y, e.y), make_float2(0.5f, 0.5f), qx[s]);
            float2 dy1 = __ffma2_rn(make_float2(e.w, e.w), make_float2(0.5f, 0.5f), qy[s]);
            w0 = __ffma2_rn(dy0, dy0, __fmul2_rn(dx0, dx0));
            w1 = __ffma2_rn(dy1, dy1, __fmul2_rn(dx1, dx1));
          } else {
            w0 = __fadd2_rn(__ffma2_rn(qy[s], make_float2(e.z, e.z), __ffma2_rn(qx[s], make_float2(e.x, e.x), make_float2(n.x, n.x))), qn[s]);
            w1 = __fadd2_rn(__ffma2_rn(qy[s], make_float2(e.w, e.w), __ffma2_rn(qx[s], make_float2(e.y, e.y), make_float2(n.y, n.y))), qn[s]);
          }
          cmin[s].x = min3f(cmin[s].x, w0.x, w1.x);
          cmin[s].y = min3f(cmin[s].y, w0.y, w1.y);
          rm0 = min3f(rm0, w0.x, w0.y);
          rm1 = min3f(rm1, w1.x, w1.y);
        }
        float2 wt = __fadd2_rn(__ffma2_rn(make_float2(ty, ty), make_float2(e.z, e.w), __ffma2_rn(make_float2(tx, tx), make_float2(e.x, e.y), n)), make_float2(tn, tn));
        cmint = min3f(cmint, wt.x, wt.y);
        rm0 = fminf(rm0, wt.x); rm1 = fminf(rm1, wt.y);
        if (VAR == 0 || VAR == 2 || VAR == 3) {
          const int r0 = __reduce_min_sync(FULL, __float_as_int(rm0));
          const int r1 = __reduce_min_sync(FULL, __float_as_int(rm1));
          if (lane == 0) { rowbuf[w][u] = __int_as_float(r0); rowbuf[w][u + 1] = __int_as_float(r1); }
        } else if (VAR == 1) {
          rsum += rm0 + rm1;
        } else if (VAR == 4) {
          rowbuf[w][(u >> 1) * 33 + lane] = fminf(rm0, rm1);
        }
      }
      __syncwarp();
      if (VAR == 4) {
        float m = INFINITY;
#pragma unroll
        for (int l = 0; l < 16; l += 2) m = min3f(m, rowbuf[w][lane * 0 + l * 33 + (lane & 15)], rowbuf[w][(l + 1) * 33 + (lane & 15)]);
        rsum += sqrtf(fmaxf(m, 0.f));
      } else if (VAR != 1) {
        rsum += sqrtf(fmaxf(rowbuf[w][lane], 0.f));
      }
      __syncwarp();
    }
    float cs = cmint;
    for (int s = 0; s < NP; ++s) cs += cmin[s].x + cmin[s].y;
    acc += rsum + cs;
  }
  out[blockIdx.x * 256 + threadIdx.x] = acc;
}

template <int VAR> void run(const char* name, float4* ex, float2* en, float* out, float2* q) {
  int nc = 148 * 4 * 8 * 64;
  k<VAR><<<148 * 4, 256>>>(ex, en, 1000, out, q);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<VAR><<<148 * 4, 256>>>(ex, en, nc, out, q);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("%-40s %.1f M curve-pairs/s (P=200, Q=224 slots)\n", name, nc / ms / 1e3);
}
int main() {
  float4* ex; float2* en; float* out; float2* q;
  cudaMalloc(&ex, 112 * 16); cudaMalloc(&en, 112 * 8); cudaMalloc(&out, 148 * 4 * 256 * 4); cudaMalloc(&q, 256 * 8);
  cudaMemset(ex, 0, 112 * 16); cudaMemset(en, 0, 112 * 8); cudaMemset(q, 0, 256 * 8);
  run<0>("expansion f32x2 + REDUX (current)", ex, en, out, q);
  run<1>("expansion, no row reduce (bound)", ex, en, out, q);
  run<3>("direct f32x2 + REDUX", ex, en, out, q);
  run<4>("expansion + smem transpose rows", ex, en, out, q);
  return 0;
}
