// Chamfer scan with fused top-k / threshold selection (sm_100a).
//
// Reference semantics:
//   chamfer         curves.py:123-129  mean_a min_q |a-q| + mean_q min_a |a-q|
//   _chamfer_block  atlas.py:45-55     the same per curve of a (C, P, 2) block
//   Atlas.retrieve  atlas.py:179-236   walk the seeded shuffle order; hits are
//                                      d < threshold in scan order (first k),
//                                      padding is the best non-hits by
//                                      (d, scan position)
//
// Mapping (fast path, even P <= 256, Q <= 256).  The query lives in
// REGISTERS for the whole launch: lane l owns query points l, l+32, ... (QS
// slots, packed in pairs for the f32x2 FFMA2/FADD2 pipes).  Each warp walks
// its grid-stride share of scan positions; the database curve for the next
// position is fetched by a 1-D TMA bulk copy (cp.async.bulk + mbarrier) into
// a per-warp double buffer while the current curve is processed.  For every
// database point a (broadcast LDS.128, two points per step):
//   * column minima (per query point) stay in registers, FMNMX3-updated;
//   * the row minimum over the lane's slots is reduced across the warp by a
//     single REDUX.MIN on the non-negative float bit pattern.
// Square roots are taken only of the minima.  Distances use direct
// differences (no |a|^2+|q|^2-2a.q cancellation).
// Each warp keeps a lane-distributed sorted top-k (by (d, pos)) of non-hits
// and the first-k hits (by pos); a merge kernel reduces the per-warp lists.
#include "common.cuh"

#include <atomic>
#include <climits>
#include <cstdlib>
#include <cuda_fp16.h>

namespace la {
namespace {

#ifndef LA_CH_WARPS
#define LA_CH_WARPS 10  // x 2 CTAs at 96 registers: C4 8 / 10 / 12 warps 3.58 / 3.39 / 4.03 ms
#endif
constexpr int CW = LA_CH_WARPS;  // warps per CTA
constexpr int CT = CW * 32;
constexpr int PMAX = 256;       // database points per curve (fast path)
constexpr float BIG = 1.0e18f;  // padding coordinate: never a minimum

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "LAB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra LAB_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// the same on precomputed shared-space addresses (hot loops)
__device__ __forceinline__ void mbar_expect_tx_s(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d_s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "LAB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra LAB_WAIT_%=;\n\t}" ::"r"(bar),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ float min3f(float a, float b, float c) { return fminf(fminf(a, b), c); }

__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// lane-distributed sorted list of up to k entries; lane i holds entry i
struct WarpList {
  float d;
  long long pos;
  long long id;
};

__device__ __forceinline__ bool key_less(float d0, long long p0, float d1, long long p1) {
  return d0 < d1 || (d0 == d1 && p0 < p1);
}

// insert (d, pos, id) keeping ascending order by (d, pos); by_pos orders by
// position only.  Returns nothing; entries beyond k fall off.
__device__ __forceinline__ void list_insert(WarpList& L, int k, int lane, float d, long long pos, long long id,
                                            bool by_pos) {
  const bool less = lane < k && (by_pos ? (L.pos < pos) : key_less(L.d, L.pos, d, pos));
  const int idx = __popc(__ballot_sync(FULL, less));
  if (idx >= k) return;
  const float pd = __shfl_up_sync(FULL, L.d, 1);
  const long long pp = __shfl_up_sync(FULL, L.pos, 1);
  const long long pi = __shfl_up_sync(FULL, L.id, 1);
  if (lane > idx && lane < k) {
    L.d = pd;
    L.pos = pp;
    L.id = pi;
  }
  if (lane == idx) {
    L.d = d;
    L.pos = pos;
    L.id = id;
  }
}

struct ScanCtx {
  la_chamfer_args a;
  int nwarps_total;   // per query
  float* ws_top_d;    // [NQ][nwarps][k]
  long long* ws_top_pos;
  long long* ws_top_id;
  float* ws_hit_d;
  long long* ws_hit_pos;
  long long* ws_hit_id;
  long long* ws_nhit;  // [NQ][nwarps]
  float* dense;        // [NQ][N] (generic path) or NULL
  // exact pruning (fast path, top-k without all_d): per-query distance grid
  // of the query (lower bounds of the DB-to-query row minima) and a running
  // upper bound of the k-th best non-hit distance
  const __half* lb_dt;  // [NQ][LBV][LBV] vertex distances to the query, rounded down
  const float* lb_par;  // [NQ][8]: lo.x, lo.y, 1/h.x, 1/h.y, h.x, h.y
  unsigned* thr;        // [NQ] float bits of a k-th best upper bound
  unsigned* slots;      // [NQ][32] float bits: min d of the evaluated non-hits with id % 32 == slot
  int prune;
  float lb_slack;       // absolute slack subtracted from a curve's bound
  // indexed scans: number of scan positions actually present (the survivor
  // list's device-side count), or NULL: [pos_begin, pos_end)
  const long long* pos_count;
  // multi-query indexed scans: query qi's survivor list at order / pos_map +
  // qi * list_stride, its count at pos_count[qi] (0: one list for all queries)
  long long list_stride;
};

__device__ __forceinline__ void consider(WarpList& top, WarpList& hit, long long& nhit, const ScanCtx& c,
                                         int lane, float d, long long pos, long long id) {
  const int k = c.a.k;
  if (k <= 0) return;
  if (d < c.a.threshold) {
    ++nhit;
    const long long kp = __shfl_sync(FULL, hit.pos, k - 1);
    if (pos < kp) list_insert(hit, k, lane, d, pos, id, true);
  } else {
    const float kd = __shfl_sync(FULL, top.d, k - 1);
    const long long kp = __shfl_sync(FULL, top.pos, k - 1);
    if (key_less(d, pos, kd, kp)) list_insert(top, k, lane, d, pos, id, false);
  }
}

__device__ __forceinline__ void flush_lists(const ScanCtx& c, int qi, int gw, int lane, const WarpList& top,
                                            const WarpList& hit, long long nhit) {
  const int k = c.a.k;
  if (k <= 0) return;
  const size_t base = ((size_t)qi * c.nwarps_total + gw) * k;
  if (lane < k) {
    c.ws_top_d[base + lane] = top.d;
    c.ws_top_pos[base + lane] = top.pos;
    c.ws_top_id[base + lane] = top.id;
    c.ws_hit_d[base + lane] = hit.d;
    c.ws_hit_pos[base + lane] = hit.pos;
    c.ws_hit_id[base + lane] = hit.id;
  }
  if (lane == 0) c.ws_nhit[(size_t)qi * c.nwarps_total + gw] = nhit;
}

__device__ __forceinline__ void list_init(WarpList& L) {
  L.d = INFINITY;
  L.pos = LLONG_MAX;
  L.id = -1;
}

// ------------------------------------------------------------ fast path
// Expanded, pair-swizzled database curve in shared memory: for point pairs
// (2i, 2i+1), centred coordinates a' = a - (0.5, 0.5):
//   ex[i] = (-2x'_0, -2x'_1, -2y'_0, -2y'_1),  en[i] = (|a'_0|^2, |a'_1|^2)
// so  w(a, q) = |a'|^2 - 2 a'.q' + |q'|^2 = |a - q|^2  is two FFMA2 + one
// FADD2 per pair of query slots, and 0.5 * ex recovers -a' exactly for the
// direct-difference re-check.
constexpr float FAR_N = 1.0e30f;   // |a'|^2 of padding points: never a minimum
constexpr float U32 = 5.9604645e-8f;  // 2^-24, fp32 unit roundoff

template <int QS>
struct QueryRegs {
  static constexpr int NP = QS / 2;
  float2 qx[NP > 0 ? NP : 1], qy[NP > 0 ? NP : 1], qn[NP > 0 ? NP : 1];
  float tx = 0.f, ty = 0.f, tn = FAR_N;  // odd tail slot
  float r2 = 0.f;                        // max |q'|^2
};

// expanded-form minima for one database point pair (a0 = 2i, a1 = 2i+1).
// SCALAR selects one-lane FFMA/FADD/FMUL instead of the f32x2 forms (the
// two issue very differently against FMNMX3 on sm_100a; see tools/micro).
template <int QS, bool DIRECT, bool SCALAR>
__device__ __forceinline__ void pair_minima(const QueryRegs<QS>& Q, const float4 ex, const float2 en,
                                            float2 (&cmin)[QS / 2 > 0 ? QS / 2 : 1], float& cmint, float& rm0,
                                            float& rm1) {
  constexpr int NP = QS / 2;
  rm0 = INFINITY;
  rm1 = INFINITY;
#pragma unroll
  for (int s = 0; s < NP; ++s) {
    float2 w0, w1;
    if (SCALAR) {
      if (DIRECT) {
        float dx, dy;
        dx = fmaf(ex.x, 0.5f, Q.qx[s].x); dy = fmaf(ex.z, 0.5f, Q.qy[s].x); w0.x = fmaf(dy, dy, dx * dx);
        dx = fmaf(ex.x, 0.5f, Q.qx[s].y); dy = fmaf(ex.z, 0.5f, Q.qy[s].y); w0.y = fmaf(dy, dy, dx * dx);
        dx = fmaf(ex.y, 0.5f, Q.qx[s].x); dy = fmaf(ex.w, 0.5f, Q.qy[s].x); w1.x = fmaf(dy, dy, dx * dx);
        dx = fmaf(ex.y, 0.5f, Q.qx[s].y); dy = fmaf(ex.w, 0.5f, Q.qy[s].y); w1.y = fmaf(dy, dy, dx * dx);
      } else {
        w0.x = fmaf(Q.qy[s].x, ex.z, fmaf(Q.qx[s].x, ex.x, en.x)) + Q.qn[s].x;
        w0.y = fmaf(Q.qy[s].y, ex.z, fmaf(Q.qx[s].y, ex.x, en.x)) + Q.qn[s].y;
        w1.x = fmaf(Q.qy[s].x, ex.w, fmaf(Q.qx[s].x, ex.y, en.y)) + Q.qn[s].x;
        w1.y = fmaf(Q.qy[s].y, ex.w, fmaf(Q.qx[s].y, ex.y, en.y)) + Q.qn[s].y;
      }
    } else if (DIRECT) {
      const float2 dx0 = __ffma2_rn(make_float2(ex.x, ex.x), make_float2(0.5f, 0.5f), Q.qx[s]);
      const float2 dy0 = __ffma2_rn(make_float2(ex.z, ex.z), make_float2(0.5f, 0.5f), Q.qy[s]);
      const float2 dx1 = __ffma2_rn(make_float2(ex.y, ex.y), make_float2(0.5f, 0.5f), Q.qx[s]);
      const float2 dy1 = __ffma2_rn(make_float2(ex.w, ex.w), make_float2(0.5f, 0.5f), Q.qy[s]);
      w0 = __ffma2_rn(dy0, dy0, __fmul2_rn(dx0, dx0));
      w1 = __ffma2_rn(dy1, dy1, __fmul2_rn(dx1, dx1));
    } else {
      w0 = __fadd2_rn(__ffma2_rn(Q.qy[s], make_float2(ex.z, ex.z),
                                 __ffma2_rn(Q.qx[s], make_float2(ex.x, ex.x), make_float2(en.x, en.x))),
                      Q.qn[s]);
      w1 = __fadd2_rn(__ffma2_rn(Q.qy[s], make_float2(ex.w, ex.w),
                                 __ffma2_rn(Q.qx[s], make_float2(ex.y, ex.y), make_float2(en.y, en.y))),
                      Q.qn[s]);
    }
    cmin[s].x = min3f(cmin[s].x, w0.x, w1.x);
    cmin[s].y = min3f(cmin[s].y, w0.y, w1.y);
    rm0 = min3f(rm0, w0.x, w0.y);
    rm1 = min3f(rm1, w1.x, w1.y);
  }
  if (QS & 1) {
    // tail slot against both points at once: pairs over (a0, a1)
    float2 w;
    if (SCALAR) {
      if (DIRECT) {
        float dx = fmaf(ex.x, 0.5f, Q.tx), dy = fmaf(ex.z, 0.5f, Q.ty);
        w.x = fmaf(dy, dy, dx * dx);
        dx = fmaf(ex.y, 0.5f, Q.tx);
        dy = fmaf(ex.w, 0.5f, Q.ty);
        w.y = fmaf(dy, dy, dx * dx);
      } else {
        w.x = fmaf(Q.ty, ex.z, fmaf(Q.tx, ex.x, en.x)) + Q.tn;
        w.y = fmaf(Q.ty, ex.w, fmaf(Q.tx, ex.y, en.y)) + Q.tn;
      }
    } else if (DIRECT) {
      const float2 dx = __ffma2_rn(make_float2(ex.x, ex.y), make_float2(0.5f, 0.5f), make_float2(Q.tx, Q.tx));
      const float2 dy = __ffma2_rn(make_float2(ex.z, ex.w), make_float2(0.5f, 0.5f), make_float2(Q.ty, Q.ty));
      w = __ffma2_rn(dy, dy, __fmul2_rn(dx, dx));
    } else {
      w = __fadd2_rn(__ffma2_rn(make_float2(Q.ty, Q.ty), make_float2(ex.z, ex.w),
                                __ffma2_rn(make_float2(Q.tx, Q.tx), make_float2(ex.x, ex.y), en)),
                     make_float2(Q.tn, Q.tn));
    }
    cmint = min3f(cmint, w.x, w.y);
    rm0 = fminf(rm0, w.x);
    rm1 = fminf(rm1, w.y);
  }
}

// |sqrt(m_true) - sqrt(m)| bound when |m_true - m| <= delta
__device__ __forceinline__ float sqrt_err(float m, float delta) {
  return sqrtf(fmaxf(m, 0.f) + delta) - sqrtf(fmaxf(m - delta, 0.f));
}

// One curve against the register-resident query: returns the chamfer value
// and (EXPANSION) a rigorous bound on its fp32 expansion error.
template <int QS, bool DIRECT, bool SCALAR = false>
__device__ __forceinline__ float curve_chamfer(const QueryRegs<QS>& Q, const float4* __restrict__ ex,
                                               const float2* __restrict__ en, int P, int Q_, int lane,
                                               float delta, float& err, float* rowbuf) {
  constexpr int NP = QS / 2;
  float2 cmin[NP > 0 ? NP : 1];
#pragma unroll
  for (int s = 0; s < NP; ++s) cmin[s] = make_float2(INFINITY, INFINITY);
  float cmint = INFINITY;
  float row_sum = 0.f, row_err = 0.f;
  const int Ppad = (P + 31) & ~31;
  const bool leader = lane == 0;
#pragma unroll 1
  for (int a0 = 0; a0 < Ppad; a0 += 32) {
#pragma unroll
    for (int u = 0; u < 32; u += 2) {
      const int i = (a0 + u) >> 1;
      float rm0, rm1;
      pair_minima<QS, DIRECT, SCALAR>(Q, ex[i], en[i], cmin, cmint, rm0, rm1);
      // signed-int REDUX on the float bits: any negative rounding residue
      // (expansion form) sorts below every positive value and is clamped
      // to zero after the chunk
      const int r0 = __reduce_min_sync(FULL, __float_as_int(rm0));
      const int r1 = __reduce_min_sync(FULL, __float_as_int(rm1));
      if (leader) {
        rowbuf[u] = __int_as_float(r0);
        rowbuf[u + 1] = __int_as_float(r1);
      }
    }
    __syncwarp();
    const float mine = fmaxf(rowbuf[lane], 0.f);
    __syncwarp();
    if (a0 + lane < P) {
      row_sum += sqrtf(mine);
      if (!DIRECT) row_err += sqrt_err(mine, delta);
    }
  }
  float col_sum = 0.f, col_err = 0.f;
#pragma unroll
  for (int s = 0; s < NP; ++s) {
    if (lane + 32 * (2 * s) < Q_) {
      col_sum += sqrtf(fmaxf(cmin[s].x, 0.f));
      if (!DIRECT) col_err += sqrt_err(cmin[s].x, delta);
    }
    if (lane + 32 * (2 * s + 1) < Q_) {
      col_sum += sqrtf(fmaxf(cmin[s].y, 0.f));
      if (!DIRECT) col_err += sqrt_err(cmin[s].y, delta);
    }
  }
  if ((QS & 1) && lane + 32 * (QS - 1) < Q_) {
    col_sum += sqrtf(fmaxf(cmint, 0.f));
    if (!DIRECT) col_err += sqrt_err(cmint, delta);
  }
  if (!DIRECT) err = warp_sum(row_err) / (float)P + warp_sum(col_err) / (float)Q_;
  return warp_sum(row_sum) / (float)P + warp_sum(col_sum) / (float)Q_;
}

template <int QS>
__device__ void load_query(QueryRegs<QS>& Q, const float2* __restrict__ qsrc, int Qn, int lane) {
  constexpr int NP = QS / 2;
  float qr2 = 0.f;
#pragma unroll
  for (int s = 0; s < NP; ++s) {
    const int i0 = lane + 32 * (2 * s), i1 = lane + 32 * (2 * s + 1);
    float2 v0 = make_float2(BIG, BIG), v1 = make_float2(BIG, BIG);
    float n0 = FAR_N, n1 = FAR_N;
    if (i0 < Qn) {
      v0 = qsrc[i0];
      v0.x -= 0.5f;
      v0.y -= 0.5f;
      n0 = fmaf(v0.y, v0.y, v0.x * v0.x);
      qr2 = fmaxf(qr2, n0);
    }
    if (i1 < Qn) {
      v1 = qsrc[i1];
      v1.x -= 0.5f;
      v1.y -= 0.5f;
      n1 = fmaf(v1.y, v1.y, v1.x * v1.x);
      qr2 = fmaxf(qr2, n1);
    }
    Q.qx[s] = make_float2(v0.x, v1.x);
    Q.qy[s] = make_float2(v0.y, v1.y);
    Q.qn[s] = make_float2(n0, n1);
  }
  if (QS & 1) {
    const int it = lane + 32 * (QS - 1);
    Q.tx = BIG;
    Q.ty = BIG;
    Q.tn = FAR_N;
    if (it < Qn) {
      Q.tx = qsrc[it].x - 0.5f;
      Q.ty = qsrc[it].y - 0.5f;
      Q.tn = fmaf(Q.ty, Q.ty, Q.tx * Q.tx);
      qr2 = fmaxf(qr2, Q.tn);
    }
  }
  Q.r2 = __uint_as_float(__reduce_max_sync(FULL, __float_as_uint(qr2)));
}

// Column-term lower bound (prune stage 3): the database curve's points in
// runs of LB_RUN, each run's bounding box; min_a |q - a| >= distance from q
// to the nearest box.  Boxes (centred like the query registers) are built
// into `boxes` (one lane per run) and scanned by every lane for its query
// slots.  Returns mean_q of the bound (uniform across the warp).
template <int QS, int LB_RUN>
__device__ __forceinline__ float curve_col_bound(const QueryRegs<QS>& Q, const float2* __restrict__ cur, int P,
                                                 int Qn, float4* __restrict__ boxes, int lane) {
  constexpr int NP = QS / 2;
  const int nb = (P + LB_RUN - 1) / LB_RUN;
  if (lane < nb) {
    float lx = INFINITY, ly = INFINITY, hx = -INFINITY, hy = -INFINITY;
    const int e = min(P, (lane + 1) * LB_RUN);
    for (int i = lane * LB_RUN; i < e; ++i) {
      const float2 a = cur[i];
      lx = fminf(lx, a.x); ly = fminf(ly, a.y); hx = fmaxf(hx, a.x); hy = fmaxf(hy, a.y);
    }
    // (lo.x, lo.y, -hi.x, -hi.y), centred like the query registers
    boxes[lane] = make_float4(lx - 0.5f, ly - 0.5f, 0.5f - hx, 0.5f - hy);
  }
  __syncwarp();
  float2 m[NP > 0 ? NP : 1];
#pragma unroll
  for (int j = 0; j < NP; ++j) m[j] = make_float2(INFINITY, INFINITY);
  float mt = INFINITY;
  const float2 neg1 = make_float2(-1.f, -1.f);
  for (int b = 0; b < nb; ++b) {
    const float4 bx = boxes[b];
    const float2 lox = make_float2(bx.x, bx.x), loy = make_float2(bx.y, bx.y);
    const float2 nhx = make_float2(bx.z, bx.z), nhy = make_float2(bx.w, bx.w);
    // two query slots per f32x2 op: lo - q (FFMA2), q - hi (FADD2); the
    // same roundings as the scalar form
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const float2 ax = __ffma2_rn(Q.qx[j], neg1, lox), bxv = __fadd2_rn(Q.qx[j], nhx);
      const float2 ay = __ffma2_rn(Q.qy[j], neg1, loy), byv = __fadd2_rn(Q.qy[j], nhy);
      const float2 dx = make_float2(fmaxf(fmaxf(ax.x, bxv.x), 0.f), fmaxf(fmaxf(ax.y, bxv.y), 0.f));
      const float2 dy = make_float2(fmaxf(fmaxf(ay.x, byv.x), 0.f), fmaxf(fmaxf(ay.y, byv.y), 0.f));
      const float2 d2 = __ffma2_rn(dy, dy, __fmul2_rn(dx, dx));
      m[j].x = fminf(m[j].x, d2.x);
      m[j].y = fminf(m[j].y, d2.y);
    }
    if (QS & 1) {
      const float dx = fmaxf(fmaxf(bx.x - Q.tx, Q.tx + bx.z), 0.f);
      const float dy = fmaxf(fmaxf(bx.y - Q.ty, Q.ty + bx.w), 0.f);
      mt = fminf(mt, fmaf(dy, dy, dx * dx));
    }
  }
  __syncwarp();
  float sum = 0.f;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    if (lane + 32 * (2 * j) < Qn) sum += sqrt_approx(m[j].x);
    if (lane + 32 * (2 * j + 1) < Qn) sum += sqrt_approx(m[j].y);
  }
  if ((QS & 1) && lane + 32 * (QS - 1) < Qn) sum += sqrt_approx(mt);
  return warp_sum(sum) / (float)Qn;
}

// rare path: direct differences for a curve whose expansion error bound is
// too large (near-duplicates); own register file, query reloaded from L2
template <int QS>
__device__ __noinline__ float direct_chamfer(const float2* __restrict__ qsrc, int Qn, const float4* ex,
                                             const float2* en, int P, int lane, float* rowbuf) {
  QueryRegs<QS> Q;
  load_query<QS>(Q, qsrc, Qn, lane);
  float dummy;
  return curve_chamfer<QS, true>(Q, ex, en, P, Qn, lane, 0.f, dummy, rowbuf);
}

// ------------------------------------------------------------ exact pruning
// Row-term lower bound.  For a vertex v of a grid laid over the query's
// box, DT(v) = min_q |v - q|; for any database point a and any vertex v,
// min_q |a - q| >= DT(v) - |a - v| (triangle inequality).  Taking the best
// of the four corners of a's cell and averaging over the curve's points
// bounds the first chamfer term from below, and the second term is >= 0, so
//   chamfer(a, q) >= LB(a) = mean_i max(0, max_corners DT(v) - |a_i - v|).
// A curve whose bound (less slack for fp32 rounding) exceeds both the
// threshold (so it is no hit) and an upper bound of the k-th best non-hit
// distance found so far (thr) cannot enter the result and is skipped before
// its 40,000 point pairs are evaluated.  Three bounds of increasing cost
// and strength run in turn: the row term from the nearest grid vertex, from
// the best of the cell's four corners, and that plus the column term from
// bounding boxes of 10-point runs of the database curve
// (curve_col_bound).  thr falls as curves are evaluated: the k-th smallest
// of 32 per-query slot minima (slot = record id % 32, publish_kth), or
// optionally starts at the k-th best of a seed scan (LA_CH_SEED_DIV).  The
// result lists are identical to the unpruned scan: every curve in the
// final top-k has d <= (final k-th) <= thr at all times, and ties never
// prune (strict >).
#ifndef LA_CH_INDEX_MQ_SEED_DIV
#define LA_CH_INDEX_MQ_SEED_DIV 32  // multi-query indexed scans: seed prefix
#endif
#ifndef LA_CH_INDEX_SEED_DIV
#define LA_CH_INDEX_SEED_DIV 64  // indexed scans: the seed scan covers 1 / 64 of the positions (C4, 10M: 32 / 64 / 128 / 256 / 512 -> 1.74 / 1.70 / 1.75 / 1.86 / 2.01 ms)
#endif
constexpr int LBG = 64;             // grid cells per axis
constexpr int LBV = LBG + 1;        // vertices per axis
constexpr size_t LB_VTX_BYTES = ((size_t)LBV * LBV * sizeof(__half) + 15) & ~(size_t)15;
// per query: the vertex table (LBV x LBV) then the cell table (LBG x LBG)
#ifndef LA_CH_CELL_STRIDE
#define LA_CH_CELL_STRIDE (LBG + 2)
#endif
// cell table rows padded to LBS entries: neighbouring cells in x then fall
// into neighbouring shared-memory banks (with 64 two-byte entries per row a
// horizontal run of a curve -- the same iy in consecutive lanes -- would hit
// one bank)
constexpr int LBS = LA_CH_CELL_STRIDE;
constexpr size_t LB_DT_BYTES = (LB_VTX_BYTES + (size_t)LBG * LBS * sizeof(__half) + 15) & ~(size_t)15;
constexpr float LB_CELL_ONE = 16384.f;  // cell table fixed point: units of 2^-14
constexpr long long PRUNE_MIN_POS = 1 << 16;  // smaller scans: no seed launches

// grid over the query's bounding box joined with the unit square (the
// normalised-curve frame), padded by 1/32; DT rounded toward -inf after a
// 1e-6 slack for the fp32 distance evaluation.  grid (ceil, NQ), 256 threads.
__global__ void __launch_bounds__(256) lb_grid_kernel(const float* __restrict__ queries, int Q,
                                                      __half* __restrict__ dt, float* __restrict__ par) {
  const int qi = blockIdx.y;
  const float2* q = reinterpret_cast<const float2*>(queries) + (size_t)qi * Q;
  __shared__ float2 sq[256];
  __shared__ float red[4][8];
  float lx = 0.f, ly = 0.f, hx = 1.f, hy = 1.f;
  for (int i = threadIdx.x; i < Q; i += 256) {
    const float2 v = q[i];
    lx = fminf(lx, v.x); ly = fminf(ly, v.y); hx = fmaxf(hx, v.x); hy = fmaxf(hy, v.y);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lx = fminf(lx, __shfl_xor_sync(FULL, lx, o)); ly = fminf(ly, __shfl_xor_sync(FULL, ly, o));
    hx = fmaxf(hx, __shfl_xor_sync(FULL, hx, o)); hy = fmaxf(hy, __shfl_xor_sync(FULL, hy, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { red[0][w] = lx; red[1][w] = ly; red[2][w] = hx; red[3][w] = hy; }
  __syncthreads();
  lx = red[0][0]; ly = red[1][0]; hx = red[2][0]; hy = red[3][0];
  for (int j = 1; j < 8; ++j) {
    lx = fminf(lx, red[0][j]); ly = fminf(ly, red[1][j]); hx = fmaxf(hx, red[2][j]); hy = fmaxf(hy, red[3][j]);
  }
  const float padx = (hx - lx) / 32.f, pady = (hy - ly) / 32.f;
  lx -= padx; ly -= pady; hx += padx; hy += pady;
  const float cx = (hx - lx) / (float)LBG, cy = (hy - ly) / (float)LBG;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    float* pp = par + (size_t)qi * 8;
    pp[0] = lx; pp[1] = ly; pp[2] = 1.f / cx; pp[3] = 1.f / cy; pp[4] = cx; pp[5] = cy; pp[6] = 0.f; pp[7] = 0.f;
  }
  __half* out = dt + (size_t)qi * (LB_DT_BYTES / sizeof(__half));
  const int v = blockIdx.x * 256 + threadIdx.x;
  const bool live = v < LBV * LBV;
  const int ix = live ? v / LBV : 0, iy = live ? v % LBV : 0;
  const float vx = __fmaf_rn((float)ix, cx, lx), vy = __fmaf_rn((float)iy, cy, ly);
  // cell table: distance from the query to cell c's box, the border cells
  // open toward infinity (points outside the grid clamp into them) and
  // interior edges widened by 1e-6 (rounding of the scan's cell index)
  const bool lc = v < LBG * LBG;
  const int cxi = lc ? v / LBG : 0, cyi = lc ? v % LBG : 0;
  const float bx0 = cxi == 0 ? -INFINITY : __fmaf_rn((float)cxi, cx, lx) - 1e-6f;
  const float bx1 = cxi == LBG - 1 ? INFINITY : __fmaf_rn((float)(cxi + 1), cx, lx) + 1e-6f;
  const float by0 = cyi == 0 ? -INFINITY : __fmaf_rn((float)cyi, cy, ly) - 1e-6f;
  const float by1 = cyi == LBG - 1 ? INFINITY : __fmaf_rn((float)(cyi + 1), cy, ly) + 1e-6f;
  float m = INFINITY, mc = INFINITY;
  for (int b = 0; b < Q; b += 256) {
    __syncthreads();
    if (b + threadIdx.x < Q) sq[threadIdx.x] = q[b + threadIdx.x];
    __syncthreads();
    const int e = min(256, Q - b);
    for (int j = 0; j < e; ++j) {
      const float dx = vx - sq[j].x, dy = vy - sq[j].y;
      m = fminf(m, __fmaf_rn(dy, dy, dx * dx));
      const float ex = fmaxf(fmaxf(bx0 - sq[j].x, sq[j].x - bx1), 0.f);
      const float ey = fmaxf(fmaxf(by0 - sq[j].y, sq[j].y - by1), 0.f);
      mc = fminf(mc, __fmaf_rn(ey, ey, ex * ex));
    }
  }
  if (live) out[v] = __float2half_rd(fmaxf(sqrtf(m) * (1.f - 1e-6f) - 1e-6f, 0.f));
  // cell table in fixed point, floor(d * 2^14) (6.1e-5 resolution, finer
  // than fp16 above 0.125; integer sums of <= 256 terms fit 32 bits)
  if (lc) {
    const float dc = fmaxf(sqrtf(mc) * (1.f - 1e-6f) - 1e-6f, 0.f);
    reinterpret_cast<unsigned short*>(out + LB_VTX_BYTES / sizeof(__half))[cxi * LBS + cyi] =
        (unsigned short)min(__float2uint_rd(dc * (float)LB_CELL_ONE), 65535u);
  }
}

// k-th best of the seed scan's merged list -> thr (inf when fewer than k)
__global__ void thr_init_kernel(const float* __restrict__ seed_d, int k, int NQ, unsigned* __restrict__ thr,
                                unsigned* __restrict__ slots) {
  const int qi = blockIdx.x * blockDim.x + threadIdx.x;
  if (qi >= NQ) return;
  const float d = seed_d ? seed_d[(size_t)qi * k + k - 1] : INFINITY;
  thr[qi] = __float_as_uint(d < INFINITY && d >= 0.f ? d : INFINITY);
  for (int j = 0; j < 32; ++j) slots[(size_t)qi * 32 + j] = __float_as_uint(INFINITY);
}

// ------------------------------------------------------------ cell index
// The cheapest bound of the scan (curve_row_bound_cell: every database point
// a lies in grid cell c(a), and min_q |a - q| >= CT(c) = distance from the
// query to c's box) only needs each point's CELL.  la_chamfer_index stores
// the cells of every database point once, on a fixed 64 x 64 grid over the
// unit square padded by 1/32 (the frame of normalised curves; points outside
// clamp into the border cells, whose boxes are open toward infinity): 2 bytes
// per point instead of 8.  An indexed scan then runs in three steps:
//   seed   the pruned scan over a 1/64 prefix; its k-th best distance t0
//          bounds the final k-th best from above;
//   bound  every curve's cell row against the query's cell table (one u16
//          table load and an integer add per point, 400 bytes per curve
//          streamed): curves whose bound exceeds max(t0, threshold) can be
//          neither hits nor in the top k;
//   scan   the pruned scan over the ordered list of the others (running
//          bound, later stages, full evaluation as before), which reports
//          their original scan positions.
// Lists identical to the scan without an index: the bound is the first
// stage's (same slack rule), only taken against t0 instead of the running
// bound.
__device__ __forceinline__ unsigned lds_u16i(uint32_t a) {
  unsigned short h;
  asm("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(a));
  return h;
}
// table rows padded to 66 entries: cell (ix, iy) at ix * 66 + iy, so that
// neighbouring cells in x fall into neighbouring shared-memory banks (with a
// stride of 64 two-byte entries a horizontal run of a curve -- the same iy
// in every lane -- would hit one bank 32 ways)
constexpr int IDX_STRIDE = LBG + 2;
constexpr int IDX_TAB = LBG * IDX_STRIDE;  // table entries (8,448 bytes)
constexpr unsigned IDX_NULL = LBG;         // a padding slot of row 0: table value 0 (row padding cells)
// cells per index row: P rounded up to 16 (whole 32-byte sectors per curve)
__host__ __device__ constexpr int idx_row(int P) { return (P + 15) & ~15; }
constexpr float IDX_LO = -1.f / 32.f;
constexpr float IDX_CELL = (1.f + 2.f / 32.f) / (float)LBG;  // 17 / 1024, exact
constexpr float IDX_INV = 1.f / IDX_CELL;

__device__ __forceinline__ unsigned idx_cell(float2 a) {
  const unsigned ix = min(__float2uint_rd(fmaf(a.x, IDX_INV, -IDX_LO * IDX_INV)), (unsigned)(LBG - 1));
  const unsigned iy = min(__float2uint_rd(fmaf(a.y, IDX_INV, -IDX_LO * IDX_INV)), (unsigned)(LBG - 1));
  return ix * IDX_STRIDE + iy;
}

__global__ void __launch_bounds__(256) index_kernel(const float2* __restrict__ db, long long N, int P,
                                                    unsigned short* __restrict__ cells) {
  const int Pp = idx_row(P);
  const long long n = N * Pp;
  for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    const long long r = i / Pp;
    const int j = (int)(i - r * Pp);
    cells[i] = j < P ? (unsigned short)idx_cell(db[r * P + j]) : (unsigned short)IDX_NULL;
  }
}

// ---- coarse distance tables (the COLUMN term of the bound step).  For
// every database curve a and every cell c of a 16 x 16 grid over the same
// padded unit square, CD(a, c) = min_i dist(box(c), a_i), rounded down to
// 1/160 (one byte; border boxes open toward infinity, interior edges widened
// by 1e-6).  A query point q_j in cell c has min_i |q_j - a_i| >= CD(a, c),
// so mean_j CD(a, cell(q_j)) bounds the second chamfer term from below: with
// the query's cell histogram (cell, weight) that is a few dozen byte loads
// per curve.  Row and column bounds are complementary -- a query passing
// near every database point has a small row term and a large column term --
// and the scan compares their SUM with the threshold (numpy simulation,
// 3,000 curves x 6 queries: the row bound alone keeps 25-56 % of the curves,
// the sum 1-5 %).
constexpr int CDG = 16;                  // coarse cells per axis
constexpr int CD_CELLS = CDG * CDG;      // bytes per curve
constexpr float CD_ONE = 160.f;          // fixed point: units of 1 / 160 (255 = 1.59)
constexpr float kFrontFrac = 0.85f;      // second level: survivors with bound <= 0.85 t are scanned first
constexpr int CD2G = 32;                 // second level: 32 x 32 cells, 1 KB per curve
constexpr int CD2_CELLS = CD2G * CD2G;

template <int G>
__device__ __forceinline__ unsigned cd_cell(float2 a) {
  constexpr float inv = (float)G / (1.f + 2.f / 32.f);
  const unsigned ix = min(__float2uint_rd(fmaf(a.x, inv, -IDX_LO * inv)), (unsigned)(G - 1));
  const unsigned iy = min(__float2uint_rd(fmaf(a.y, inv, -IDX_LO * inv)), (unsigned)(G - 1));
  return ix * G + iy;
}

// one warp per curve; lane l owns cells l, l + 32, ...; the curve's points
// are read by every lane (L1 broadcast).  grid-stride over curves.  G = 16:
// the bound step's table (256 bytes); G = 32: the second level's (1 KB).
template <int G>
__global__ void __launch_bounds__(256) index_coarse_kernel(const float2* __restrict__ db, long long N, int P,
                                                           unsigned char* __restrict__ coarse) {
  constexpr float cell = (1.f + 2.f / 32.f) / (float)G;
  constexpr int CPL = G * G / 32;  // cells per lane
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * 8;
  for (long long r = (long long)blockIdx.x * 8 + (threadIdx.x >> 5); r < N; r += nw) {
    const float2* pts = db + r * P;
#pragma unroll 1
    for (int u0 = 0; u0 < CPL; u0 += 8) {
      float bx0[8], bx1[8], by0[8], by1[8], m[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = lane + 32 * (u0 + u), cx = c / G, cy = c % G;
        bx0[u] = cx == 0 ? -INFINITY : __fmaf_rn((float)cx, cell, IDX_LO) - 1e-6f;
        bx1[u] = cx == G - 1 ? INFINITY : __fmaf_rn((float)(cx + 1), cell, IDX_LO) + 1e-6f;
        by0[u] = cy == 0 ? -INFINITY : __fmaf_rn((float)cy, cell, IDX_LO) - 1e-6f;
        by1[u] = cy == G - 1 ? INFINITY : __fmaf_rn((float)(cy + 1), cell, IDX_LO) + 1e-6f;
        m[u] = INFINITY;
      }
      for (int i = 0; i < P; ++i) {
        const float2 a = __ldg(pts + i);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const float ex = fmaxf(fmaxf(bx0[u] - a.x, a.x - bx1[u]), 0.f);
          const float ey = fmaxf(fmaxf(by0[u] - a.y, a.y - by1[u]), 0.f);
          m[u] = fminf(m[u], __fmaf_rn(ey, ey, ex * ex));
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        // rounded down, after the slack of the fp32 distance evaluation
        const float d = fmaxf(sqrtf(m[u]) * (1.f - 1e-6f) - 1e-6f, 0.f);
        coarse[r * (G * G) + lane + 32 * (u0 + u)] = (unsigned char)min(__float2uint_rd(d * CD_ONE), 255u);
      }
    }
  }
}

// the query's cell histogram on the G x G grid as G * G weight bytes
// (G * G / 4 words after qw[0], the number of words to use: G * G / 4, or 0
// when Q > 255 and a weight could overflow its byte -- the column term is
// then left out).  One CTA of 256 threads.
template <int G>
__global__ void __launch_bounds__(256) index_qlist_kernel(const float* __restrict__ query, int Q,
                                                          unsigned* __restrict__ qw) {
  __shared__ unsigned hist[G * G];
  for (int c = threadIdx.x; c < G * G; c += 256) hist[c] = 0u;
  __syncthreads();
  const float2* q = reinterpret_cast<const float2*>(query) + (size_t)blockIdx.x * Q;  // one CTA per query
  qw += (size_t)blockIdx.x * (G * G / 4 + 1);
  for (int j = threadIdx.x; j < Q; j += 256) atomicAdd(&hist[cd_cell<G>(q[j])], 1u);
  __syncthreads();
  for (int w = threadIdx.x; w < G * G / 4; w += 256) {
    const int c = 4 * w;
    qw[1 + w] = hist[c] | (hist[c + 1] << 8) | (hist[c + 2] << 16) | (hist[c + 3] << 24);
  }
  if (threadIdx.x == 0) qw[0] = Q <= 255 ? G * G / 4 : 0;
}

// the query's cell table on the index grid: floor(2^14 x distance from the
// query to the cell's box), boxes widened by 1e-6 (rounding of idx_cell),
// border cells open, the distance rounded down as in lb_grid_kernel.
// grid (ceil(IDX_TAB / 256), queries), 256 threads.
__global__ void __launch_bounds__(256) index_table_kernel(const float* __restrict__ queries, int Q,
                                                          unsigned short* __restrict__ tables) {
  __shared__ float2 sq[256];
  const float2* q = reinterpret_cast<const float2*>(queries) + (size_t)blockIdx.y * Q;
  unsigned short* table = tables + (size_t)blockIdx.y * IDX_TAB;
  const int v = blockIdx.x * 256 + threadIdx.x;  // table slot
  const int cxi = min(v / IDX_STRIDE, LBG - 1), cyi = min(v % IDX_STRIDE, LBG - 1);
  const float bx0 = cxi == 0 ? -INFINITY : __fmaf_rn((float)cxi, IDX_CELL, IDX_LO) - 1e-6f;
  const float bx1 = cxi == LBG - 1 ? INFINITY : __fmaf_rn((float)(cxi + 1), IDX_CELL, IDX_LO) + 1e-6f;
  const float by0 = cyi == 0 ? -INFINITY : __fmaf_rn((float)cyi, IDX_CELL, IDX_LO) - 1e-6f;
  const float by1 = cyi == LBG - 1 ? INFINITY : __fmaf_rn((float)(cyi + 1), IDX_CELL, IDX_LO) + 1e-6f;
  float mc = INFINITY;
  for (int b = 0; b < Q; b += 256) {
    __syncthreads();
    if (b + threadIdx.x < Q) sq[threadIdx.x] = q[b + threadIdx.x];
    __syncthreads();
    const int e = min(256, Q - b);
    for (int j = 0; j < e; ++j) {
      const float ex = fmaxf(fmaxf(bx0 - sq[j].x, sq[j].x - bx1), 0.f);
      const float ey = fmaxf(fmaxf(by0 - sq[j].y, sq[j].y - by1), 0.f);
      mc = fminf(mc, __fmaf_rn(ey, ey, ex * ex));
    }
  }
  const float dc = fmaxf(sqrtf(mc) * (1.f - 1e-6f) - 1e-6f, 0.f);
  // padding slots (iy >= LBG) hold 0: IDX_NULL, the cell of row padding, adds nothing
  if (v < IDX_TAB)
    table[v] = v % IDX_STRIDE >= LBG ? (unsigned short)0
                                     : (unsigned short)min(__float2uint_rd(dc * (float)LB_CELL_ONE), 65535u);
}

// bound step: one THREAD per curve (no warp reduction, ~4 instructions per
// point; a warp per curve measured 3.2 ms per 10M curves against 1.45 ms).
// A curve that is not pruned is
// appended (one atomic per warp) to the survivor list as (record, reported
// scan position); the list's order does not matter: the scan's lists are
// keyed by (distance, position) and its hit lists by position.
#ifndef LA_IB_T
#define LA_IB_T 512  // 128x16 / 256x8 / 512x4 threads x CTAs per SM measured 1.71 / 1.69 / 1.66 ms per C4 scan
#endif
#ifndef LA_IB_MINB
#define LA_IB_MINB 4
#endif
#ifndef LA_IB_UNROLL
#define LA_IB_UNROLL 2
#endif
constexpr int IB_T = LA_IB_T;
constexpr int IB_UNROLL = LA_IB_UNROLL;
__global__ void __launch_bounds__(IB_T, LA_IB_MINB) index_bound_kernel(const unsigned short* __restrict__ cells, int P,
                                                           const int64_t* __restrict__ order,
                                                           const int64_t* __restrict__ pos_map, long long pos_begin,
                                                           long long pos_base, long long npos,
                                                           const unsigned short* __restrict__ table,
                                                           const unsigned* __restrict__ thr, float threshold,
                                                           float lb_slack, int64_t* __restrict__ order2,
                                                           int64_t* __restrict__ pos_map2,
                                                           unsigned long long* __restrict__ count,
                                                           const unsigned char* __restrict__ coarse,
                                                           const unsigned* __restrict__ qlist, int Q) {
  __shared__ unsigned short tab[IDX_TAB];
  __shared__ __align__(16) unsigned ql[CD_CELLS / 4];  // the query's weight bytes, cell-major
  for (int i = threadIdx.x; i < IDX_TAB / 2; i += IB_T)
    reinterpret_cast<unsigned*>(tab)[i] = reinterpret_cast<const unsigned*>(table)[i];
  const int nql = coarse ? (int)qlist[0] : 0;
  for (int i = threadIdx.x; i < nql; i += IB_T) ql[i] = qlist[1 + i];
  __syncthreads();
  const float cscale = 1.f / (CD_ONE * (float)Q);
  const int lane = threadIdx.x & 31;
  const float t = fmaxf(__uint_as_float(*thr), threshold);
  const float scale = 1.f / (LB_CELL_ONE * (float)P);
  const uint32_t tab_s = smem_u32(tab);
  auto look = [&](unsigned c) -> unsigned { return lds_u16i(tab_s + 2u * c); };
  auto rec_of = [&](long long i) -> long long { return order ? order[pos_begin + i] : pos_begin + i; };
  // the warp's kept curves (lane l: relative position i, record rec) are appended together
  auto append = [&](bool keep, long long i, long long rec) {
    const unsigned mask = __ballot_sync(FULL, keep);
    if (!mask) return;
    unsigned long long base = 0ull;
    if (lane == 0) base = atomicAdd(count, (unsigned long long)__popc(mask));
    base = __shfl_sync(FULL, base, 0);
    if (keep) {
      const long long at = (long long)base + __popc(mask & ((1u << lane) - 1u));
      const long long pos = pos_begin + i;
      order2[at] = rec;
      pos_map2[at] = pos_map ? pos_map[pos] : pos + pos_base;
    }
  };
  // one THREAD per curve: its row as whole 32-byte sectors (padding cells
  // are IDX_NULL, table value 0)
  const int Pp = idx_row(P);
  const int W = Pp / 16;  // sectors per curve
  const long long nth = (long long)gridDim.x * IB_T;
  for (long long i0 = (long long)blockIdx.x * IB_T + (threadIdx.x & ~31); i0 < npos; i0 += nth) {
    const long long i = i0 + lane;
    const bool live = i < npos;
    const long long rec = live ? rec_of(i) : 0;
    const uint4* row = reinterpret_cast<const uint4*>(cells + (size_t)rec * Pp);
    unsigned s0 = 0u, s1 = 0u;
    // column term first: the query's cell histogram against the curve's
    // coarse distance bytes (a lower bound of the second chamfer term)
    float col = 0.f;
    if (live && nql) {
      // 256 distance bytes x 256 weight bytes: eight 32-byte loads, one
      // byte-wise dot product (DP4A) per word against the broadcast weights
      const unsigned char* drow = coarse + (size_t)rec * CD_CELLS;
      unsigned cs = 0u;
#pragma unroll 2
      for (int k = 0; k < CD_CELLS / 32; ++k) {
        uint4 v, u;
        asm volatile("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w), "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
                     : "l"(drow + 32 * k));
        const uint4 wa = reinterpret_cast<const uint4*>(ql)[2 * k], wb = reinterpret_cast<const uint4*>(ql)[2 * k + 1];
        cs = __dp4a(v.x, wa.x, cs); cs = __dp4a(v.y, wa.y, cs); cs = __dp4a(v.z, wa.z, cs); cs = __dp4a(v.w, wa.w, cs);
        cs = __dp4a(u.x, wb.x, cs); cs = __dp4a(u.y, wb.y, cs); cs = __dp4a(u.z, wb.z, cs); cs = __dp4a(u.w, wb.w, cs);
      }
      col = (float)cs * cscale;
    }
    if (live && !(fmaf(col, 1.f - 1e-4f, -lb_slack) > t)) {
#pragma unroll IB_UNROLL
      for (int k = 0; k < W; ++k) {
        uint4 v, u;  // one 32-byte sector (LDG.256; two 16-byte loads fetched every sector twice)
        asm volatile("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w), "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
                     : "l"(row + 2 * k));
        s0 += look(v.x & 0xffffu) + look(v.y & 0xffffu) + look(v.z & 0xffffu) + look(v.w & 0xffffu);
        s1 += look(v.x >> 16) + look(v.y >> 16) + look(v.z >> 16) + look(v.w >> 16);
        s0 += look(u.x & 0xffffu) + look(u.y & 0xffffu) + look(u.z & 0xffffu) + look(u.w & 0xffffu);
        s1 += look(u.x >> 16) + look(u.y >> 16) + look(u.z >> 16) + look(u.w >> 16);
        // the terms are >= 0: once a partial sum prunes, so does the total
        if (fmaf(fmaf((float)(s0 + s1), scale, col), 1.f - 1e-4f, -lb_slack) > t) break;
      }
    }
    append(live && !(fmaf(fmaf((float)(s0 + s1), scale, col), 1.f - 1e-4f, -lb_slack) > t), i, rec);
  }
}

// bound step for several queries: a CTA holds the cell tables of a group of
// IBM_QG queries INTERLEAVED in shared memory (entry (cell, query) at
// cell * IBM_QG + query), and a half-warp owns one curve with lane = query:
// the 16 lanes look up the same cell in 16 consecutive two-byte entries (one
// 32-byte run: no bank conflict inside a half-warp), the curve's cells come
// from a per-warp staging buffer as 16-byte broadcasts.  Every query keeps
// its own survivor list (order2 / pos_map2 + q * cap, count[q]).
constexpr int IBM_QG = 16;
constexpr int IBM_T = 512;
constexpr int IBM_ROW = 512 + CD_CELLS;  // staging bytes per curve: cells (P <= 256), coarse distance bytes
constexpr int IBM_WQ = (CD_CELLS / 4) * IBM_QG * 4;  // the group's weight words, interleaved like the tables
constexpr size_t IBM_SMEM = (size_t)IDX_TAB * IBM_QG * 2 + IBM_WQ + (size_t)(IBM_T / 32) * 2 * IBM_ROW;
__global__ void __launch_bounds__(IBM_T, 1) index_bound_mq_kernel(const unsigned short* __restrict__ cells, int P,
                                                                  const int64_t* __restrict__ order,
                                                                  const int64_t* __restrict__ pos_map,
                                                                  long long pos_begin, long long pos_base,
                                                                  long long npos, int NQ,
                                                                  const unsigned short* __restrict__ tables,
                                                                  const unsigned* __restrict__ thr, float threshold,
                                                                  float lb_slack, long long cap,
                                                                  int64_t* __restrict__ order2,
                                                                  int64_t* __restrict__ pos_map2,
                                                                  unsigned long long* __restrict__ count,
                                                                  const unsigned char* __restrict__ coarse,
                                                                  const unsigned* __restrict__ qw, int Q) {
  extern __shared__ __align__(16) unsigned char ibm_smem[];
  unsigned short* tab = reinterpret_cast<unsigned short*>(ibm_smem);
  unsigned* wq = reinterpret_cast<unsigned*>(ibm_smem + (size_t)IDX_TAB * IBM_QG * 2);
  const int q0 = blockIdx.y * IBM_QG;
  for (int i = threadIdx.x; i < IDX_TAB * IBM_QG; i += IBM_T) {
    const int cell = i / IBM_QG, ql = i % IBM_QG;
    tab[i] = q0 + ql < NQ ? tables[(size_t)(q0 + ql) * IDX_TAB + cell] : (unsigned short)0;
  }
  // weight word w of query ql at wq[w * IBM_QG + ql] (zero: no column term)
  for (int i = threadIdx.x; i < (CD_CELLS / 4) * IBM_QG; i += IBM_T) {
    const int w = i / IBM_QG, ql = i % IBM_QG;
    const unsigned* src = qw + (size_t)(q0 + ql) * (CD_CELLS / 4 + 1);
    wq[i] = (coarse && q0 + ql < NQ && src[0]) ? src[1 + w] : 0u;
  }
  __syncthreads();
  const float cscale = 1.f / (CD_ONE * (float)Q);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int h = lane >> 4, ql = lane & 15;
  const int q = q0 + ql;
  const bool qlive = q < NQ;
  const float t = qlive ? fmaxf(__uint_as_float(thr[q]), threshold) : -INFINITY;
  const float scale = 1.f / (LB_CELL_ONE * (float)P);
  const int Pp = idx_row(P);
  const int W = Pp / 16;  // sectors per curve (<= 16)
  unsigned char* stage = ibm_smem + (size_t)IDX_TAB * IBM_QG * 2 + IBM_WQ + ((size_t)w * 2 + h) * IBM_ROW;
  const uint32_t stage_s = smem_u32(stage);
  const uint32_t lane_tab = smem_u32(tab) + 2u * (uint32_t)ql;
  auto look = [&](unsigned c) -> unsigned { return lds_u16i(lane_tab + c * (2u * IBM_QG)); };
  const long long npairs = (npos + 1) / 2;
  for (long long pr = (long long)blockIdx.x * (IBM_T / 32) + w; pr < npairs; pr += (long long)gridDim.x * (IBM_T / 32)) {
    const long long i = 2 * pr + h;
    const bool live = i < npos;
    const long long rec = live ? (order ? order[pos_begin + i] : pos_begin + i) : 0;
    __syncwarp();
    if (live && ql < W) {
      uint4 v, u;
      asm volatile("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w), "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
                   : "l"(cells + (size_t)rec * Pp + 16 * ql));
      reinterpret_cast<uint4*>(stage)[2 * ql] = v;
      reinterpret_cast<uint4*>(stage)[2 * ql + 1] = u;
    }
    if (live && coarse && ql < CD_CELLS / 32) {  // the curve's 256 coarse distance bytes
      uint4 v, u;
      asm volatile("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w), "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
                   : "l"(coarse + (size_t)rec * CD_CELLS + 32 * ql));
      reinterpret_cast<uint4*>(stage + 512)[2 * ql] = v;
      reinterpret_cast<uint4*>(stage + 512)[2 * ql + 1] = u;
    }
    __syncwarp();
    unsigned s0 = 0u, s1 = 0u;
    // column term: the curve's bytes (a broadcast) against this lane's query's weights
    float col = 0.f;
    if (live && qlive && coarse) {
      unsigned cs = 0u;
#pragma unroll 4
      for (int k = 0; k < CD_CELLS / 16; ++k) {
        uint4 v;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "r"(stage_s + 512u + 16u * (uint32_t)k));
        const unsigned* wk = wq + (4 * k) * IBM_QG + ql;
        cs = __dp4a(v.x, wk[0], cs);
        cs = __dp4a(v.y, wk[IBM_QG], cs);
        cs = __dp4a(v.z, wk[2 * IBM_QG], cs);
        cs = __dp4a(v.w, wk[3 * IBM_QG], cs);
      }
      col = (float)cs * cscale;
    }
    bool alive = live && qlive && !(fmaf(col, 1.f - 1e-4f, -lb_slack) > t);
#pragma unroll 1
    for (int k = 0; k < W; ++k) {
      if (alive) {
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint4 v;
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                       : "r"(stage_s + 32u * (uint32_t)k + 16u * (uint32_t)half));
          s0 += look(v.x & 0xffffu) + look(v.y & 0xffffu) + look(v.z & 0xffffu) + look(v.w & 0xffffu);
          s1 += look(v.x >> 16) + look(v.y >> 16) + look(v.z >> 16) + look(v.w >> 16);
        }
        // the terms are >= 0: once a partial sum prunes, so does the total
        if (fmaf(fmaf((float)(s0 + s1), scale, col), 1.f - 1e-4f, -lb_slack) > t) alive = false;
      }
      if (!__any_sync(FULL, alive)) break;
    }
    if (alive) {  // not pruned: into query q's list
      const long long at = (long long)atomicAdd(count + q, 1ull);
      const long long pos = pos_begin + i;
      order2[(size_t)q * cap + at] = rec;
      pos_map2[(size_t)q * cap + at] = pos_map ? pos_map[pos] : pos + pos_base;
    }
  }
}

__global__ void index_count_mq_kernel(const long long* __restrict__ count, int NQ, int64_t* __restrict__ n_stage) {
  long long sum = 0;
  for (int q = 0; q < NQ; ++q) sum += count[q];
  n_stage[0] += sum;  // (query, curve) pairs surviving the bound step
}

// second level of the bound step, over the first level's survivors only:
// the column term from the curve's 32 x 32 table (1 KB, thirty-two 32-byte
// loads against the query's 1,024 weight bytes), then the whole cell row on
// top of it with the early exit.  Survivor i of (order_in, pos_in) that still
// is not pruned goes to (order_out, pos_out).  One thread per survivor.
__global__ void __launch_bounds__(IB_T, LA_IB_MINB) index_bound2_kernel(
    const unsigned short* __restrict__ cells, int P, const unsigned char* __restrict__ fine,
    const long long* __restrict__ count_in, const int64_t* __restrict__ order_in, const int64_t* __restrict__ pos_in,
    const unsigned short* __restrict__ table, const unsigned* __restrict__ qw2, int Q,
    const unsigned* __restrict__ thr, float threshold, float lb_slack, int64_t* __restrict__ order_out,
    int64_t* __restrict__ pos_out, unsigned long long* __restrict__ count_out, long long cap) {
  __shared__ unsigned short tab[IDX_TAB];
  __shared__ __align__(16) unsigned qwt[CD2_CELLS / 4];
  for (int i = threadIdx.x; i < IDX_TAB / 2; i += IB_T)
    reinterpret_cast<unsigned*>(tab)[i] = reinterpret_cast<const unsigned*>(table)[i];
  const int nql = (int)qw2[0];
  for (int i = threadIdx.x; i < CD2_CELLS / 4; i += IB_T) qwt[i] = i < nql ? qw2[1 + i] : 0u;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const float t = fmaxf(__uint_as_float(*thr), threshold);
  const float scale = 1.f / (LB_CELL_ONE * (float)P);
  const float cscale = 1.f / (CD_ONE * (float)Q);
  const uint32_t tab_s = smem_u32(tab);
  auto look = [&](unsigned c) -> unsigned { return lds_u16i(tab_s + 2u * c); };
  const int Pp = idx_row(P);
  const int W = Pp / 16;
  const long long n = *count_in;
  const long long nth = (long long)gridDim.x * IB_T;
  for (long long i0 = (long long)blockIdx.x * IB_T + (threadIdx.x & ~31); i0 < n; i0 += nth) {
    const long long i = i0 + lane;
    const bool live = i < n;
    const long long rec = live ? order_in[i] : 0;
    unsigned cs = 0u;
    if (live) {
      const unsigned char* drow = fine + (size_t)rec * CD2_CELLS;
#pragma unroll 4
      for (int k = 0; k < CD2_CELLS / 32; ++k) {
        uint4 v, u;
        asm volatile("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w), "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
                     : "l"(drow + 32 * k));
        const uint4 wa = reinterpret_cast<const uint4*>(qwt)[2 * k], wb = reinterpret_cast<const uint4*>(qwt)[2 * k + 1];
        cs = __dp4a(v.x, wa.x, cs); cs = __dp4a(v.y, wa.y, cs); cs = __dp4a(v.z, wa.z, cs); cs = __dp4a(v.w, wa.w, cs);
        cs = __dp4a(u.x, wb.x, cs); cs = __dp4a(u.y, wb.y, cs); cs = __dp4a(u.z, wb.z, cs); cs = __dp4a(u.w, wb.w, cs);
      }
    }
    const float col = (float)cs * cscale;
    unsigned s0 = 0u, s1 = 0u;
    if (live && !(fmaf(col, 1.f - 1e-4f, -lb_slack) > t)) {
      const uint4* row = reinterpret_cast<const uint4*>(cells + (size_t)rec * Pp);
#pragma unroll 2
      for (int k = 0; k < W; ++k) {
        uint4 v, u;
        asm volatile("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w), "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
                     : "l"(row + 2 * k));
        s0 += look(v.x & 0xffffu) + look(v.y & 0xffffu) + look(v.z & 0xffffu) + look(v.w & 0xffffu);
        s1 += look(v.x >> 16) + look(v.y >> 16) + look(v.z >> 16) + look(v.w >> 16);
        s0 += look(u.x & 0xffffu) + look(u.y & 0xffffu) + look(u.z & 0xffffu) + look(u.w & 0xffffu);
        s1 += look(u.x >> 16) + look(u.y >> 16) + look(u.z >> 16) + look(u.w >> 16);
        if (fmaf(fmaf((float)(s0 + s1), scale, col), 1.f - 1e-4f, -lb_slack) > t) break;
      }
    }
    const float bnd = fmaf(fmaf((float)(s0 + s1), scale, col), 1.f - 1e-4f, -lb_slack);
    const bool keep = live && !(bnd > t);
    // survivors whose bound is well below the threshold (the final top k is
    // among them unless the seed's bound was far off) fill the list from the
    // front, the others from the back (count_out[1]); index_close_kernel then
    // joins the two parts, so the scan meets the promising curves first and
    // its running k-th best falls early.  Order only: every survivor is kept.
    const bool front = keep && bnd <= kFrontFrac * t;
    const unsigned mf = __ballot_sync(FULL, front), mb = __ballot_sync(FULL, keep && !front);
    if (mf | mb) {
      unsigned long long bf = 0ull, bb = 0ull;
      if (lane == 0) {
        if (mf) bf = atomicAdd(count_out, (unsigned long long)__popc(mf));
        if (mb) bb = atomicAdd(count_out + 1, (unsigned long long)__popc(mb));
      }
      bf = __shfl_sync(FULL, bf, 0);
      bb = __shfl_sync(FULL, bb, 0);
      if (keep) {
        const unsigned below = (1u << lane) - 1u;
        const long long at = front ? (long long)bf + __popc(mf & below) : cap - 1 - ((long long)bb + __popc(mb & below));
        order_out[at] = rec;
        pos_out[at] = pos_in[i];
      }
    }
  }
}

// joins the back part of index_bound2_kernel's list to its front part:
// entries cap-1-j (j < count[1]) move to count[0] + j; count[0] becomes the
// total.  A grid-wide pass reading the old counts, then one thread updating
// them, are two launches (index_close_kernel, index_close_count_kernel).
__global__ void index_close_kernel(int64_t* __restrict__ order, int64_t* __restrict__ pos,
                                   const unsigned long long* __restrict__ count, long long cap) {
  const long long c0 = (long long)count[0], c1 = (long long)count[1];
  // back entries already inside the joined range [c0, c0 + c1) stay where
  // they are; the others (sources >= c0 + c1, never a target) fill the
  // slots [c0, cap - c1) the stayers leave free
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < c1; j += (long long)gridDim.x * blockDim.x) {
    const long long src = cap - 1 - j, dst = c0 + j;
    if (src >= c0 + c1) {  // sources inside [c0, c0 + c1) are already in the joined range
      order[dst] = order[src];
      pos[dst] = pos[src];
    }
  }
}
__global__ void index_close_count_kernel(unsigned long long* __restrict__ count) {
  count[0] += count[1];
}


__global__ void index_count_kernel(const long long* __restrict__ count, int64_t* __restrict__ n_stage) {
  n_stage[0] += *count;  // curves surviving the bound step
}

// A fully evaluated non-hit with d below thr: lower its slot (id % 32) and,
// when that changed the slot, publish the k-th smallest slot minimum.  The
// 32 slot minima are distances of 32 distinct evaluated records, so their
// k-th smallest bounds the final k-th best from above.  Lock-free; after the
// first wave of curves it triggers only for new near-best curves.  Whole
// warp (d, id uniform).
// the rank-(k-1) ballot below needs k <= 32 (one slot minimum per lane)
static_assert(LA_MAX_TOPK <= 32, "publish_kth assumes k <= 32");
__device__ __forceinline__ void publish_kth(unsigned* __restrict__ thr, unsigned* __restrict__ slots, int k,
                                            int lane, float d, long long id) {
  unsigned old = 0u;
  if (lane == 0) old = atomicMin(&slots[id & 31], __float_as_uint(d));
  old = __shfl_sync(FULL, old, 0);
  if (old <= __float_as_uint(d)) return;
  const unsigned v = __ldcg(&slots[lane]);
  int rank = 0;
#pragma unroll 8
  for (int j = 0; j < 32; ++j) {
    const unsigned o = __shfl_sync(FULL, v, j);
    rank += (o < v) || (o == v && j < lane);
  }
  const unsigned kth_lane = __ballot_sync(FULL, rank == k - 1);
  const unsigned kth = __shfl_sync(FULL, v, __ffs(kth_lane) - 1);
  if (lane == 0 && kth < __float_as_uint(INFINITY)) atomicMin(thr, kth);
}

// cheapest first stage: every point a lies in (or clamps into) grid cell
// c(a), and min_q |a - q| >= CT(c) = distance from the query to c's box
// (lb_grid_kernel's cell table): one table load per point, no square root.
// cur_s / ct_s: shared-space addresses of the curve and the cell table.
__device__ __forceinline__ float2 lds_f2p(uint32_t a) {
  float2 v;
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ unsigned lds_u16p(uint32_t a) {
  unsigned short h;
  asm("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(a));
  return h;
}
__device__ __forceinline__ float curve_row_bound_cell(uint32_t cur_s, int P, uint32_t ct_s, float lx, float ly,
                                                      float ihx, float ihy, int lane, float early) {
  const float ox = -lx * ihx, oy = -ly * ihy;
  // fixed-point table entries (floors) summed as integers: the sum is itself
  // a floor, and the warp total is one REDUX
  auto point = [&](int i) -> unsigned {
    const float2 a = lds_f2p(cur_s + 8u * (uint32_t)i);
    const unsigned ix = min(__float2uint_rd(fmaf(a.x, ihx, ox)), (unsigned)(LBG - 1));
    const unsigned iy = min(__float2uint_rd(fmaf(a.y, ihy, oy)), (unsigned)(LBG - 1));
    return lds_u16p(ct_s + 2u * (ix * LBS + iy));
  };
  const float scale = 1.f / (LB_CELL_ONE * (float)P);
  unsigned s = 0u;
  int P1;
  if (P >= 128) {
    // the first 128 points, four per lane, independent loads
    P1 = 128;
#pragma unroll
    for (int u = 0; u < 4; ++u) s += point(lane + 32 * u);
  } else {
    P1 = P;
    for (int i = lane; i < P; i += 32) s += point(i);
  }
  // the terms are >= 0: a partial sum is already a (weaker) bound
  const unsigned t1 = __reduce_add_sync(FULL, s);
  const float s1 = (float)t1 * scale;
  if (s1 > early || P1 == P) return s1;
  s = 0u;
  for (int i = P1 + lane; i < P; i += 32) s += point(i);
  return (float)(t1 + __reduce_add_sync(FULL, s)) * scale;
}

// mean over the curve's points of the per-point bound (whole warp; all
// lanes return the same value)
__device__ __forceinline__ float curve_row_bound(const float2* __restrict__ cur, int P, const __half* __restrict__ dt,
                                                 float lx, float ly, float ihx, float ihy, float cx, float cy,
                                                 int lane) {
  float s = 0.f;
  for (int i = lane; i < P; i += 32) {
    const float2 a = cur[i];
    const int ix = min(max(__float2int_rd((a.x - lx) * ihx), 0), LBG - 1);
    const int iy = min(max(__float2int_rd((a.y - ly) * ihy), 0), LBG - 1);
    const float x0 = __fmaf_rn((float)ix, cx, lx), x1 = __fmaf_rn((float)(ix + 1), cx, lx);
    const float y0 = __fmaf_rn((float)iy, cy, ly), y1 = __fmaf_rn((float)(iy + 1), cy, ly);
    const float ex0 = a.x - x0, ex1 = a.x - x1, ey0 = a.y - y0, ey1 = a.y - y1;
    const float sx0 = ex0 * ex0, sx1 = ex1 * ex1, sy0 = ey0 * ey0, sy1 = ey1 * ey1;
    const __half* d0 = dt + ix * LBV + iy;
    float L = __half2float(d0[0]) - sqrt_approx(sx0 + sy0);
    L = fmaxf(L, __half2float(d0[1]) - sqrt_approx(sx0 + sy1));
    L = fmaxf(L, __half2float(d0[LBV]) - sqrt_approx(sx1 + sy0));
    L = fmaxf(L, __half2float(d0[LBV + 1]) - sqrt_approx(sx1 + sy1));
    s += fmaxf(L, 0.f);
  }
  return warp_sum(s) / (float)P;
}

constexpr size_t SCAN_SMEM_PER_WARP =
    2 * PMAX * sizeof(float2) + (PMAX / 2) * (sizeof(float4) + sizeof(float2)) + 32 * sizeof(float);
constexpr size_t SCAN_SMEM = CW * SCAN_SMEM_PER_WARP + CW * 2 * sizeof(uint64_t) + LB_DT_BYTES;

// The CTA's 8 warp lists -> one list (warp 0 inserts the other warps'
// entries), flushed as list blockIdx.x of gridDim.x: the merge kernel then
// scans 8x fewer entries (most warp lists are short once pruning starts).
__device__ __forceinline__ void cta_flush_lists(const ScanCtx& c, int qi, int w, int lane, WarpList& top,
                                                WarpList& hit, long long nhit, unsigned char* smem) {
  const int k = c.a.k;
  if (k <= 0) return;
  struct Ent { float d; long long pos, id; };
  Ent* et = reinterpret_cast<Ent*>(smem);                  // [CW][32] top
  Ent* eh = et + CW * 32;                                   // [CW][32] hits
  long long* nh = reinterpret_cast<long long*>(eh + CW * 32);  // [CW]
  __syncthreads();  // every warp is done with the shared buffers
  et[w * 32 + lane] = Ent{top.d, top.pos, top.id};
  eh[w * 32 + lane] = Ent{hit.d, hit.pos, hit.id};
  if (lane == 0) nh[w] = nhit;
  __syncthreads();
  if (w != 0) return;
  long long tot = nhit;
  for (int v = 1; v < CW; ++v) {
    tot += nh[v];
    for (int j = 0; j < k; ++j) {
      const Ent e = et[v * 32 + j];
      if (e.pos == LLONG_MAX) break;  // sorted: the rest is empty
      const float kd = __shfl_sync(FULL, top.d, k - 1);
      const long long kp = __shfl_sync(FULL, top.pos, k - 1);
      if (!key_less(e.d, e.pos, kd, kp)) break;
      list_insert(top, k, lane, e.d, e.pos, e.id, false);
    }
    for (int j = 0; j < k; ++j) {
      const Ent e = eh[v * 32 + j];
      if (e.pos == LLONG_MAX) break;
      const long long kp = __shfl_sync(FULL, hit.pos, k - 1);
      if (!(e.pos < kp)) break;
      list_insert(hit, k, lane, e.d, e.pos, e.id, true);
    }
  }
  ScanCtx cc = c;
  cc.nwarps_total = gridDim.x;
  flush_lists(cc, qi, blockIdx.x, lane, top, hit, tot);
}

#ifndef LA_CH_MINB
#define LA_CH_MINB 2  // resident CTAs per SM the register budget targets (3: 80 registers with spills, 12 % slower on C4)
#endif
template <int QS>
__global__ void __launch_bounds__(CT, LA_CH_MINB) chamfer_scan_kernel(const ScanCtx c) {
  extern __shared__ __align__(128) unsigned char scan_smem[];
  auto raw = reinterpret_cast<float2(*)[2][PMAX]>(scan_smem);                                  // [CW][2][PMAX]
  auto exs = reinterpret_cast<float4(*)[PMAX / 2]>(scan_smem + CW * 2 * PMAX * sizeof(float2));  // [CW][PMAX/2]
  auto ens = reinterpret_cast<float2(*)[PMAX / 2]>(scan_smem + CW * 2 * PMAX * sizeof(float2) +
                                                   CW * (PMAX / 2) * sizeof(float4));
  float* rowbuf = reinterpret_cast<float*>(scan_smem + CW * 2 * PMAX * sizeof(float2) +
                                           CW * (PMAX / 2) * (sizeof(float4) + sizeof(float2))) +
                  32 * (threadIdx.x >> 5);
  auto bars = reinterpret_cast<uint64_t(*)[2]>(scan_smem + CW * SCAN_SMEM_PER_WARP);
  __half* lb_dt = reinterpret_cast<__half*>(scan_smem + CW * SCAN_SMEM_PER_WARP + CW * 2 * sizeof(uint64_t));
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int qi = blockIdx.y;
  const la_chamfer_args& A = c.a;
  const int P = A.P, Qn = A.Q;
  const int gw = blockIdx.x * CW + w;
  const long long stride = (long long)gridDim.x * CW;
  const bool expansion = (A.flags & LA_CH_EXPANSION) != 0;
  const float fix_tol = A.fixup_below;

  // query slots in registers, centred at (0.5, 0.5); padding far away
  QueryRegs<QS> Q;
  const float2* qsrc = reinterpret_cast<const float2*>(A.queries) + (size_t)qi * Qn;
  load_query<QS>(Q, qsrc, Qn, lane);

  WarpList top, hit;
  list_init(top);
  list_init(hit);
  long long nhit = 0;

  // pruning: the query's distance grid in shared memory
  const bool prune = c.prune != 0;
  float lb_lx = 0.f, lb_ly = 0.f, lb_ihx = 0.f, lb_ihy = 0.f, lb_cx = 0.f, lb_cy = 0.f;
  if (prune) {
    const uint4* src = reinterpret_cast<const uint4*>(c.lb_dt + (size_t)qi * (LB_DT_BYTES / sizeof(__half)));
    uint4* dst = reinterpret_cast<uint4*>(lb_dt);
    for (int i = threadIdx.x; i < (int)(LB_DT_BYTES / 16); i += CT) dst[i] = src[i];
    const float* pp = c.lb_par + (size_t)qi * 8;
    lb_lx = pp[0]; lb_ly = pp[1]; lb_ihx = pp[2]; lb_ihy = pp[3]; lb_cx = pp[4]; lb_cy = pp[5];
    __syncthreads();
  }
  const unsigned* thr_q = prune ? c.thr + qi : nullptr;
  long long nfull = 0;
  const float lb_slack = c.lb_slack;

  const long long first = A.pos_begin + gw;
  long long pos_end = A.pos_end;
  if (c.pos_count) pos_end = min(pos_end, A.pos_begin + c.pos_count[c.list_stride ? qi : 0]);
  const int64_t* const ord = A.order ? A.order + (size_t)qi * c.list_stride : nullptr;
  const int64_t* const pmap = A.pos_map ? A.pos_map + (size_t)qi * c.list_stride : nullptr;
  const long long count = first < pos_end ? (pos_end - first + stride - 1) / stride : 0;
  const bool use_tma = (P % 2) == 0;
  const uint32_t bytes = (uint32_t)P * 8u;
  const int Ppad = (P + 31) & ~31;
  if (lane == 0) {
    mbar_init(&bars[w][0], 1);
    mbar_init(&bars[w][1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto rec_of = [&](long long pos) -> long long { return ord ? ord[pos] : pos; };
  if (use_tma && count > 0 && lane == 0) {
    const long long id = rec_of(first);
    mbar_expect_tx(&bars[w][0], bytes);
    tma_load_1d(&raw[w][0][0], A.db + (size_t)id * P * 2, bytes, &bars[w][0]);
  }
  uint32_t phase = 0;
  // running bound read one curve ahead (an older value is larger, still an
  // upper bound of the final k-th best)
  float thr_c = prune ? __uint_as_float(__ldcg(thr_q)) : INFINITY;
  const uint32_t lbc_s = smem_u32(lb_dt) + (uint32_t)LB_VTX_BYTES;  // cell table
  const uint32_t bar_s = smem_u32(&bars[w][0]);                     // + 8 * buffer
  const uint32_t raw_s = smem_u32(&raw[w][0][0]);                   // + PMAX * 8 * buffer

  for (long long it = 0; it < count; ++it) {
    const int bi = (int)(it & 1);
    const long long pos = first + it * stride;
    const long long id = rec_of(pos);
    __syncwarp();
    const float2* cur;
    if (use_tma) {
      if (it + 1 < count && lane == 0) {
        fence_proxy_async();
        const long long nid = rec_of(pos + stride);
        const uint32_t nb = (uint32_t)(bi ^ 1);
        mbar_expect_tx_s(bar_s + 8u * nb, bytes);
        tma_load_1d_s(raw_s + (uint32_t)(PMAX * 8) * nb, A.db + (size_t)nid * P * 2, bytes, bar_s + 8u * nb);
      }
      mbar_wait_s(bar_s + 8u * (uint32_t)bi, (phase >> bi) & 1u);
      phase ^= (1u << bi);
      cur = &raw[w][bi][0];
    } else {
      const float2* src = reinterpret_cast<const float2*>(A.db) + (size_t)id * P;
      for (int k = lane; k < P; k += 32) raw[w][0][k] = src[k];
      __syncwarp();
      cur = &raw[w][0][0];
    }
    if (id == A.exclude_id) continue;
    if (prune) {
      // bounds of increasing cost; d > lb: neither a hit nor in the top k.
      // thr as loaded one curve earlier (the load's latency hides behind
      // this curve; an older, larger value still bounds the final k-th best
      // from above)
      const float t = fmaxf(thr_c, A.threshold);
      thr_c = __uint_as_float(__ldcg(thr_q));  // for the next curve (measured: two in flight was slower)
      const uint32_t cur_s = use_tma ? raw_s + (uint32_t)(PMAX * 8 * bi) : raw_s;  // = cur
      // (a survivor list of the index's bound step already passed this
      // stage's bound, against a looser threshold; it rarely prunes there)
      if (!c.pos_count) {
        const float lb1 = curve_row_bound_cell(cur_s, P, lbc_s, lb_lx, lb_ly, lb_ihx, lb_ihy, lane,
                                               (t + lb_slack) * (1.f + 2e-4f));
        if (fmaf(lb1, 1.f - 1e-4f, -lb_slack) > t) continue;
      }
      const float lb4 = curve_row_bound(cur, P, lb_dt, lb_lx, lb_ly, lb_ihx, lb_ihy, lb_cx, lb_cy, lane);
      if (fmaf(lb4, 1.f - 1e-4f, -lb_slack) > t) continue;
      // column term from 10-point runs (a 40-point pre-stage measured slower)
      const float lbc = curve_col_bound<QS, 10>(Q, cur, P, Qn, exs[w], lane);
      if (fmaf(lb4 + lbc, 1.f - 1e-4f, -lb_slack) > t) continue;
    }
    ++nfull;
    // expand + swizzle (each lane handles pairs lane, lane+32, ...)
    float ar2 = 0.f;
    for (int i = lane; i < Ppad / 2; i += 32) {
      // padding points sit far away in both forms (-0.5*ex = 1e18, |a'|^2 = 1e30)
      float4 e4 = make_float4(-2.f * BIG, -2.f * BIG, -2.f * BIG, -2.f * BIG);
      float2 n2 = make_float2(FAR_N, FAR_N);
      if (2 * i < P) {
        const float2 p0 = cur[2 * i];
        const float x = p0.x - 0.5f, y = p0.y - 0.5f;
        e4.x = -2.f * x;
        e4.z = -2.f * y;
        n2.x = fmaf(y, y, x * x);
        ar2 = fmaxf(ar2, n2.x);
      }
      if (2 * i + 1 < P) {
        const float2 p1 = cur[2 * i + 1];
        const float x = p1.x - 0.5f, y = p1.y - 0.5f;
        e4.y = -2.f * x;
        e4.w = -2.f * y;
        n2.y = fmaf(y, y, x * x);
        ar2 = fmaxf(ar2, n2.y);
      }
      exs[w][i] = e4;
      ens[w][i] = n2;
    }
    ar2 = __uint_as_float(__reduce_max_sync(FULL, __float_as_uint(ar2)));
    __syncwarp();
    float d;
    if (expansion) {
      // rounding of the FFMA2/FADD2 chain is <= 18 u R^2
      const float delta = 20.f * U32 * fmaxf(ar2, Q.r2);
      float err = 0.f;
      if (A.flags & LA_CH_SCALAR_PIPE)
        d = curve_chamfer<QS, false, true>(Q, exs[w], ens[w], P, Qn, lane, delta, err, rowbuf);
      else
        d = curve_chamfer<QS, false>(Q, exs[w], ens[w], P, Qn, lane, delta, err, rowbuf);
      if (!(err <= fix_tol)) d = direct_chamfer<QS>(qsrc, Qn, exs[w], ens[w], P, lane, rowbuf);
    } else {
      float dummy;
      if (A.flags & LA_CH_SCALAR_PIPE)
        d = curve_chamfer<QS, true, true>(Q, exs[w], ens[w], P, Qn, lane, 0.f, dummy, rowbuf);
      else
        d = curve_chamfer<QS, true>(Q, exs[w], ens[w], P, Qn, lane, 0.f, dummy, rowbuf);
    }
    if (A.all_d && lane == 0) A.all_d[(size_t)qi * A.N + id] = d;
    const long long rpos = pmap ? pmap[pos] : pos + A.pos_base;
    consider(top, hit, nhit, c, lane, d, rpos, id + A.id_base);
    if (prune && d >= A.threshold && d < __uint_as_float(__shfl_sync(FULL, __ldcg(thr_q), 0)))
      publish_kth(c.thr + qi, c.slots + (size_t)qi * 32, A.k, lane, d, id);
  }
  cta_flush_lists(c, qi, w, lane, top, hit, nhit, scan_smem);
  if (A.n_full && lane == 0 && nfull) atomicAdd(reinterpret_cast<unsigned long long*>(A.n_full + qi),
                                                 (unsigned long long)nfull);
}

// ------------------------------------------------------------ multi-query scan
// (fast path, pruned top-k, NQ >= 2)  chamfer_scan_kernel gives every query
// its own CTAs, so each query re-streams the whole database and re-derives
// each curve's grid cells.  Here a CTA holds a GROUP of QG queries: every
// database curve is fetched once per group (TMA), each of its points is
// placed once on a grid COMMON to all queries (nearest vertex v, e = |a - v|),
// and the stage-0 bound of the first chamfer term,
//   LB0(a, q) = mean_i max(0, DT_q(v_i) - e_i),   DT_q(v) <= min_q |v - q|,
// costs one shared-memory half load and three FP ops per (point, query).
// The per-lane partial sums of 8 queries are reduced across the warp by a
// transposed butterfly (9 shuffles for 8 sums).  A (query, curve) pair whose
// LB0 exceeds max(threshold, thr_q) is dropped; the survivors go through the
// single-query stages (4-corner bound on the query's own 64x64 grid, column
// bound from run boxes) and, if still alive, the exact evaluation.  Lists
// live per (CTA, query) in shared memory (a per-query lock; insertions are
// rare), are flushed as list blockIdx.x of the query and merged by
// merge_kernel.  Lists are identical to the unpruned scan for the same
// reasons as chamfer_scan_kernel (every bound is a valid lower bound after
// the (1 - 1e-4) / slack margins; ties never prune).
#ifndef LA_MQ_WARPS
#define LA_MQ_WARPS 16  // C5: 8 / 12 / 16 warps 25.7 / 18.4 / 17.0 ms (16 still fits 32-query groups)
#endif
constexpr int MQ_W = LA_MQ_WARPS;  // warps per CTA
constexpr int MQ_T = MQ_W * 32;
constexpr int MQ_MAXG = 64;       // queries per group (bits of the pass mask)
constexpr int MQ_TAB_N = 129;     // grid lines of the column-term gap tables
#ifndef LA_MQ_DIAG
#define LA_MQ_DIAG 0  // gap tables along the diagonals too (measured: no extra pruning on C5)
#endif
constexpr int MQ_NTAB = LA_MQ_DIAG ? 8 : 4;
constexpr int MQ_TAB_BYTES = LA_MQ_DIAG ? 2068 : 1036;  // MQ_NTAB tables of MQ_TAB_N halves + pad (odd word stride)

template <int G0>
struct MQGrid {
  static constexpr int V = G0 + 1;
  static constexpr int NV = V * V;
  static constexpr int STRIDE = (NV + 7) & ~7;  // halves per query
};

// common grid: bounding box of every query point joined with the unit
// square, padded by 1/32 of its extent; par = lo.x, lo.y, 1/h.x, 1/h.y, h.x, h.y
__global__ void __launch_bounds__(1024) mq_box_kernel(const float* __restrict__ queries, long long n, int G0,
                                                      float* __restrict__ par) {
  const float2* q = reinterpret_cast<const float2*>(queries);
  float lx = 0.f, ly = 0.f, hx = 1.f, hy = 1.f;
  for (long long i = threadIdx.x; i < n; i += 1024) {
    const float2 v = q[i];
    lx = fminf(lx, v.x); ly = fminf(ly, v.y); hx = fmaxf(hx, v.x); hy = fmaxf(hy, v.y);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lx = fminf(lx, __shfl_xor_sync(FULL, lx, o)); ly = fminf(ly, __shfl_xor_sync(FULL, ly, o));
    hx = fmaxf(hx, __shfl_xor_sync(FULL, hx, o)); hy = fmaxf(hy, __shfl_xor_sync(FULL, hy, o));
  }
  __shared__ float red[4][32];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { red[0][w] = lx; red[1][w] = ly; red[2][w] = hx; red[3][w] = hy; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 1; j < 32; ++j) {
      lx = fminf(lx, red[0][j]); ly = fminf(ly, red[1][j]); hx = fmaxf(hx, red[2][j]); hy = fmaxf(hy, red[3][j]);
    }
    const float padx = (hx - lx) / 32.f, pady = (hy - ly) / 32.f;
    lx -= padx; ly -= pady; hx += padx; hy += pady;
    const float cx = (hx - lx) / (float)G0, cy = (hy - ly) / (float)G0;
    par[0] = lx; par[1] = ly; par[2] = 1.f / cx; par[3] = 1.f / cy; par[4] = cx; par[5] = cy;
    const float ccx = (hx - lx) / (float)(MQ_TAB_N - 1), ccy = (hy - ly) / (float)(MQ_TAB_N - 1);
    par[6] = ccx; par[7] = ccy; par[8] = 1.f / ccx; par[9] = 1.f / ccy;
    // rotated axes u = x + y, v = x - y (unnormalised) over the box's range
    const float lu = lx + ly, lv = lx - hy;
    const float ccu = ((hx + hy) - lu) / (float)(MQ_TAB_N - 1), ccv = ((hx - ly) - lv) / (float)(MQ_TAB_N - 1);
    par[10] = lu; par[11] = ccu; par[12] = 1.f / ccu; par[13] = lv; par[14] = ccv; par[15] = 1.f / ccv;
  }
}

// DT_q on the common grid, rounded toward -inf after a 1e-6 slack (as
// lb_grid_kernel); grid (ceil(NV / 256), NQ)
__global__ void __launch_bounds__(256) mq_dt_kernel(const float* __restrict__ queries, int Q, int G0, int stride,
                                                    const float* __restrict__ par, __half* __restrict__ dt) {
  const int qi = blockIdx.y;
  const float2* q = reinterpret_cast<const float2*>(queries) + (size_t)qi * Q;
  __shared__ float2 sq[256];
  const int V = G0 + 1;
  const float lx = par[0], ly = par[1], cx = par[4], cy = par[5];
  const int v = blockIdx.x * 256 + threadIdx.x;
  const bool live = v < V * V;
  const int ix = live ? v / V : 0, iy = live ? v % V : 0;
  const float vx = __fmaf_rn((float)ix, cx, lx), vy = __fmaf_rn((float)iy, cy, ly);
  float m = INFINITY;
  for (int b = 0; b < Q; b += 256) {
    __syncthreads();
    if (b + threadIdx.x < Q) sq[threadIdx.x] = q[b + threadIdx.x];
    __syncthreads();
    const int e = min(256, Q - b);
    for (int j = 0; j < e; ++j) {
      const float dx = vx - sq[j].x, dy = vy - sq[j].y;
      m = fminf(m, __fmaf_rn(dy, dy, dx * dx));
    }
  }
  if (live) dt[(size_t)qi * stride + v] = __float2half_rd(fmaxf(sqrtf(m) * (1.f - 1e-6f) - 1e-6f, 0.f));
}

// column-term gap tables per query: for grid lines g_m = lo + m * cc
// (m = 0..MQ_TAB_N-1, cc = box / (MQ_TAB_N - 1)) along x and y,
//   A(m) = mean_q max(g_m - q, 0),  B(m) = mean_q max(q - g_m, 0),
// rounded down; 4 tables of MQ_TAB_N halves, padded so that consecutive
// queries' tables start in different banks (259 words per query)
__global__ void __launch_bounds__(160) mq_tab_kernel(const float* __restrict__ queries, int Q,
                                                     const float* __restrict__ par, __half* __restrict__ tab) {
  const int qi = blockIdx.x;
  const float2* q = reinterpret_cast<const float2*>(queries) + (size_t)qi * Q;
  const int m = threadIdx.x;
  const float gx = __fmaf_rn((float)m, par[6], par[0]), gy = __fmaf_rn((float)m, par[7], par[1]);
  const float gu = __fmaf_rn((float)m, par[11], par[10]), gv = __fmaf_rn((float)m, par[14], par[13]);
  float ax = 0.f, bx = 0.f, ay = 0.f, by = 0.f, au = 0.f, bu = 0.f, av = 0.f, bv = 0.f;
  for (int i = 0; i < Q; ++i) {
    const float2 v = q[i];
    ax += fmaxf(gx - v.x, 0.f); bx += fmaxf(v.x - gx, 0.f);
    ay += fmaxf(gy - v.y, 0.f); by += fmaxf(v.y - gy, 0.f);
    const float u = v.x + v.y, w = v.x - v.y;
    au += fmaxf(gu - u, 0.f); bu += fmaxf(u - gu, 0.f);
    av += fmaxf(gv - w, 0.f); bv += fmaxf(w - gv, 0.f);
  }
  if (m < MQ_TAB_N) {
    // fp32 sums of <= 256 terms: relative error < 2e-5, covered by 1 - 1e-4
    const float sc = (1.f - 1e-4f) / (float)Q;
    __half* t = tab + (size_t)qi * (MQ_TAB_BYTES / 2);
    t[m] = __float2half_rd(ax * sc);
    t[MQ_TAB_N + m] = __float2half_rd(bx * sc);
    t[2 * MQ_TAB_N + m] = __float2half_rd(ay * sc);
    t[3 * MQ_TAB_N + m] = __float2half_rd(by * sc);
    // rounding of u, v (<= 2.4e-7 absolute) is covered by the scan's lb_slack
    if (LA_MQ_DIAG) {
      t[4 * MQ_TAB_N + m] = __float2half_rd(au * sc);
      t[5 * MQ_TAB_N + m] = __float2half_rd(bu * sc);
      t[6 * MQ_TAB_N + m] = __float2half_rd(av * sc);
      t[7 * MQ_TAB_N + m] = __float2half_rd(bv * sc);
    }
  }
  if (m < (MQ_TAB_BYTES / 2 - MQ_NTAB * MQ_TAB_N))
    tab[(size_t)qi * (MQ_TAB_BYTES / 2) + MQ_NTAB * MQ_TAB_N + m] = __float2half(0.f);
}

// highest grid line <= v (0 below the box: A vanishes there) / lowest >= v
__device__ __forceinline__ int mq_line_lo(float v, float lo, float cc, float icc) {
  int m = (int)floorf((v - lo) * icc);
  m = max(min(m, MQ_TAB_N - 1), 0);
  if (m > 0 && __fmaf_rn((float)m, cc, lo) > v) --m;
  return v >= lo ? m : 0;
}
__device__ __forceinline__ int mq_line_hi(float v, float lo, float cc, float icc) {
  int m = (int)ceilf((v - lo) * icc);
  m = max(min(m, MQ_TAB_N - 1), 0);
  if (m < MQ_TAB_N - 1 && __fmaf_rn((float)m, cc, lo) < v) ++m;
  return __fmaf_rn((float)m, cc, lo) >= v ? m : MQ_TAB_N - 1;
}

struct MQSmem {
  // per CTA: dt [QG][STRIDE] halves, lists, counters; per warp: buffers
  size_t dt, tab, top_d, top_pos, top_id, hit_d, hit_pos, hit_id, nh, lock, cnt, warp0, per_warp, total;
};

__host__ __device__ inline MQSmem mq_smem(int QG, int k, int stride, int P) {
  MQSmem m{};
  auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
  const int kk = k > 0 ? k : 1;
  size_t o = 0;
  m.dt = o; o = al(o + (size_t)((QG + 7) & ~7) * stride * 2);
  m.tab = o; o = al(o + (size_t)QG * MQ_TAB_BYTES);
  m.top_d = o; o = al(o + (size_t)QG * kk * 4);
  m.hit_d = o; o = al(o + (size_t)QG * kk * 4);
  m.top_pos = o; o = al(o + (size_t)QG * kk * 8);
  m.top_id = o; o = al(o + (size_t)QG * kk * 8);
  m.hit_pos = o; o = al(o + (size_t)QG * kk * 8);
  m.hit_id = o; o = al(o + (size_t)QG * kk * 8);
  m.nh = o; o = al(o + (size_t)QG * 8);
  m.lock = o; o = al(o + (size_t)QG * 4);
  m.cnt = o; o = al(o + (size_t)(QG + 5) * 4);  // survivors of the 5 bound stages, then n_full per query
  o = (o + 127) & ~(size_t)127;
  m.warp0 = o;
  const int Pe = (P + 1) & ~1, Ppad = (P + 31) & ~31;
  // curve double buffer, expanded pairs padded to whole 32-point chunks
  // (float4 + float2, read by curve_chamfer), 32 run boxes, row buffer,
  // 2 mbarriers
  m.per_warp = al(2 * (size_t)Pe * 8) + al((size_t)(Ppad / 2) * 16) + al((size_t)(Ppad / 2) * 8) + 32 * 16 + 32 * 4 + 16;
  m.per_warp = (m.per_warp + 127) & ~(size_t)127;
  m.total = m.warp0 + MQ_W * m.per_warp;
  return m;
}

__device__ __forceinline__ float lds_half(uint32_t a) {
  unsigned short h;
  asm("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(a));
  return __half2float(__ushort_as_half(h));
}

// insert into the CTA's list of query q under its lock (whole warp)
__device__ __forceinline__ void mq_insert(float* ld, long long* lp, long long* li, int* lock, int k, int lane,
                                          float d, long long pos, long long id, bool by_pos) {
  if (lane == 0) {
    while (atomicCAS(lock, 0, 1) != 0) __nanosleep(20);
  }
  __syncwarp();
  __threadfence_block();
  const float cd = lane < k ? ld[lane] : INFINITY;
  const long long cp = lane < k ? lp[lane] : LLONG_MAX;
  const long long ci = lane < k ? li[lane] : -1;
  const bool less = lane < k && (by_pos ? (cp < pos) : key_less(cd, cp, d, pos));
  const int idx = __popc(__ballot_sync(FULL, less));
  const float pd = __shfl_up_sync(FULL, cd, 1);
  const long long pp = __shfl_up_sync(FULL, cp, 1);
  const long long pi = __shfl_up_sync(FULL, ci, 1);
  if (idx < k) {
    if (lane > idx && lane < k) {
      ld[lane] = pd;
      lp[lane] = pp;
      li[lane] = pi;
    }
    if (lane == idx) {
      ld[lane] = d;
      lp[lane] = pos;
      li[lane] = id;
    }
  }
  __threadfence_block();
  __syncwarp();
  if (lane == 0) atomicExch(lock, 0);
}

template <int QS, int G0>
__global__ void __launch_bounds__(MQ_T, 1) chamfer_mq_kernel(const ScanCtx c, int QG, const __half* __restrict__ dt0,
                                                             const __half* __restrict__ tab0,
                                                             const float* __restrict__ par0) {
  using GR = MQGrid<G0>;
  extern __shared__ __align__(128) unsigned char mq_smem_raw[];
  const la_chamfer_args& A = c.a;
  const int P = A.P, Qn = A.Q, k = A.k;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int q0 = blockIdx.y * QG;
  const int nq = min(QG, A.NQ - q0);
  const MQSmem L = mq_smem(QG, k, GR::STRIDE, P);
  __half* sdt = reinterpret_cast<__half*>(mq_smem_raw + L.dt);
  float* s_top_d = reinterpret_cast<float*>(mq_smem_raw + L.top_d);
  float* s_hit_d = reinterpret_cast<float*>(mq_smem_raw + L.hit_d);
  long long* s_top_pos = reinterpret_cast<long long*>(mq_smem_raw + L.top_pos);
  long long* s_top_id = reinterpret_cast<long long*>(mq_smem_raw + L.top_id);
  long long* s_hit_pos = reinterpret_cast<long long*>(mq_smem_raw + L.hit_pos);
  long long* s_hit_id = reinterpret_cast<long long*>(mq_smem_raw + L.hit_id);
  unsigned long long* s_nh = reinterpret_cast<unsigned long long*>(mq_smem_raw + L.nh);
  int* s_lock = reinterpret_cast<int*>(mq_smem_raw + L.lock);
  unsigned* s_cnt = reinterpret_cast<unsigned*>(mq_smem_raw + L.cnt);
  unsigned char* wb = mq_smem_raw + L.warp0 + (size_t)w * L.per_warp;
  const int Pe = (P + 1) & ~1, Ppad = (P + 31) & ~31;
  float2* raw0 = reinterpret_cast<float2*>(wb);
  float2* raw1 = raw0 + Pe;
  size_t off = ((2 * (size_t)Pe * 8) + 15) & ~(size_t)15;
  float4* exs = reinterpret_cast<float4*>(wb + off);
  off += (((size_t)(Ppad / 2) * 16) + 15) & ~(size_t)15;
  float2* ens = reinterpret_cast<float2*>(wb + off);
  off += (((size_t)(Ppad / 2) * 8) + 15) & ~(size_t)15;
  float4* boxes = reinterpret_cast<float4*>(wb + off);
  off += 32 * 16;
  float* rowbuf = reinterpret_cast<float*>(wb + off);
  off += 32 * 4;
  uint64_t* bars = reinterpret_cast<uint64_t*>(wb + off);

  // stage the group's grids, init lists and counters
  {
    const uint4* src = reinterpret_cast<const uint4*>(dt0 + (size_t)q0 * GR::STRIDE);
    uint4* dst = reinterpret_cast<uint4*>(sdt);
    const int n16 = nq * GR::STRIDE * 2 / 16;
    for (int i = threadIdx.x; i < n16; i += MQ_T) dst[i] = src[i];
    const int npad = ((nq + 7) & ~7) * GR::STRIDE * 2 / 16;
    for (int i = n16 + threadIdx.x; i < npad; i += MQ_T) dst[i] = make_uint4(0u, 0u, 0u, 0u);
    const uint32_t* tsrc = reinterpret_cast<const uint32_t*>(tab0 + (size_t)q0 * (MQ_TAB_BYTES / 2));
    uint32_t* tdst = reinterpret_cast<uint32_t*>(mq_smem_raw + L.tab);
    for (int i = threadIdx.x; i < nq * (MQ_TAB_BYTES / 4); i += MQ_T) tdst[i] = tsrc[i];
    const int kk = k > 0 ? k : 1;
    for (int i = threadIdx.x; i < QG * kk; i += MQ_T) {
      s_top_d[i] = INFINITY; s_hit_d[i] = INFINITY;
      s_top_pos[i] = LLONG_MAX; s_hit_pos[i] = LLONG_MAX;
      s_top_id[i] = -1; s_hit_id[i] = -1;
    }
    for (int i = threadIdx.x; i < QG; i += MQ_T) { s_nh[i] = 0; s_lock[i] = 0; }
    for (int i = threadIdx.x; i < QG + 5; i += MQ_T) s_cnt[i] = 0;
  }
  __syncthreads();
  const uint32_t sdt_b = smem_u32(sdt);
  const uint32_t stab_b = smem_u32(mq_smem_raw + L.tab);
  const float lx = par0[0], ly = par0[1], ihx = par0[2], ihy = par0[3], cx = par0[4], cy = par0[5];
  const float ccx = par0[6], ccy = par0[7], iccx = par0[8], iccy = par0[9];
  const float lu = par0[10], ccu = par0[11], iccu = par0[12], lv = par0[13], ccv = par0[14], iccv = par0[15];
  const float ox = -lx * ihx, oy = -ly * ihy;
  const float lb_slack = c.lb_slack;
  const float invP = 1.f / (float)P;
  const bool expansion = (A.flags & LA_CH_EXPANSION) != 0;

  const int gw = blockIdx.x * MQ_W + w;
  const long long stride = (long long)gridDim.x * MQ_W;
  const long long first = A.pos_begin + gw;
  const long long count = first < A.pos_end ? (A.pos_end - first + stride - 1) / stride : 0;
  const bool use_tma = (P % 2) == 0;
  const uint32_t bytes = (uint32_t)P * 8u;
  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto rec_of = [&](long long pos) -> long long { return A.order ? A.order[pos] : pos; };
  if (use_tma && count > 0 && lane == 0) {
    mbar_expect_tx(&bars[0], bytes);
    tma_load_1d(raw0, A.db + (size_t)rec_of(first) * P * 2, bytes, &bars[0]);
  }
  uint32_t phase = 0;
  constexpr int UP = 8;  // points per lane (P <= 256)

  for (long long it = 0; it < count; ++it) {
    const int bi = (int)(it & 1);
    const long long pos = first + it * stride;
    const long long id = rec_of(pos);
    __syncwarp();
    const float2* cur;
    if (use_tma) {
      if (it + 1 < count && lane == 0) {
        fence_proxy_async();
        const long long nid = rec_of(pos + stride);
        mbar_expect_tx(&bars[bi ^ 1], bytes);
        tma_load_1d(bi ? raw0 : raw1, A.db + (size_t)nid * P * 2, bytes, &bars[bi ^ 1]);
      }
      mbar_wait(&bars[bi], (phase >> bi) & 1u);
      phase ^= (1u << bi);
      cur = bi ? raw1 : raw0;
    } else {
      const float2* src = reinterpret_cast<const float2*>(A.db) + (size_t)id * P;
      for (int j = lane; j < P; j += 32) raw0[j] = src[j];
      __syncwarp();
      cur = raw0;
    }
    if (id == A.exclude_id) continue;

    // ---- stage A, every query of the group: the column term from the
    // curve's bounding box and the query's gap tables,
    //   mean_q min_a |q - a| >= mean_q dist(q, box)
    //                        >= max(X, Y, (X + Y) / sqrt 2),
    //   X = Ax(lo.x) + Bx(hi.x) = mean_q max(lo.x - q.x, q.x - hi.x, 0), Y alike,
    // with the box rounded outward to the tables' grid lines
    float bx0 = INFINITY, by0 = INFINITY, bx1 = -INFINITY, by1 = -INFINITY;
    float bu0 = INFINITY, bv0 = INFINITY, bu1 = -INFINITY, bv1 = -INFINITY;
    for (int i = lane; i < P; i += 32) {
      const float2 a = cur[i];
      bx0 = fminf(bx0, a.x); by0 = fminf(by0, a.y); bx1 = fmaxf(bx1, a.x); by1 = fmaxf(by1, a.y);
      if (LA_MQ_DIAG) {
        const float u = a.x + a.y, v = a.x - a.y;
        bu0 = fminf(bu0, u); bv0 = fminf(bv0, v); bu1 = fmaxf(bu1, u); bv1 = fmaxf(bv1, v);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      bx0 = fminf(bx0, __shfl_xor_sync(FULL, bx0, o)); by0 = fminf(by0, __shfl_xor_sync(FULL, by0, o));
      bx1 = fmaxf(bx1, __shfl_xor_sync(FULL, bx1, o)); by1 = fmaxf(by1, __shfl_xor_sync(FULL, by1, o));
      if (LA_MQ_DIAG) {
        bu0 = fminf(bu0, __shfl_xor_sync(FULL, bu0, o)); bv0 = fminf(bv0, __shfl_xor_sync(FULL, bv0, o));
        bu1 = fmaxf(bu1, __shfl_xor_sync(FULL, bu1, o)); bv1 = fmaxf(bv1, __shfl_xor_sync(FULL, bv1, o));
      }
    }
    const int ilx = mq_line_lo(bx0, lx, ccx, iccx), ihx_ = mq_line_hi(bx1, lx, ccx, iccx);
    const int ily = mq_line_lo(by0, ly, ccy, iccy), ihy_ = mq_line_hi(by1, ly, ccy, iccy);
    // u, v of the curve's points carry fp32 rounding: widen by 1e-6
    const int ilu = mq_line_lo(bu0 - 1e-6f, lu, ccu, iccu), ihu = mq_line_hi(bu1 + 1e-6f, lu, ccu, iccu);
    const int ilv = mq_line_lo(bv0 - 1e-6f, lv, ccv, iccv), ihv = mq_line_hi(bv1 + 1e-6f, lv, ccv, iccv);
    // lane l: queries l and l + 32 of the group.  Projections on the unit
    // axes x, y and (1, +-1) / sqrt 2 each bound |q - a| from below:
    //   mean dist >= max(X, Y, (X + Y) / sqrt 2, max(U, V) / sqrt 2, (U + V) / 2)
    auto col_bound = [&](int qg) -> float {
      const uint32_t t = stab_b + (uint32_t)qg * MQ_TAB_BYTES;
      const float X = lds_half(t + 2u * ilx) + lds_half(t + 2u * (MQ_TAB_N + ihx_));
      const float Y = lds_half(t + 2u * (2 * MQ_TAB_N + ily)) + lds_half(t + 2u * (3 * MQ_TAB_N + ihy_));
      if (!LA_MQ_DIAG) return fmaxf(fmaxf(X, Y), (X + Y) * 0.70710670f);
      const float U = lds_half(t + 2u * (4 * MQ_TAB_N + ilu)) + lds_half(t + 2u * (5 * MQ_TAB_N + ihu));
      const float V = lds_half(t + 2u * (6 * MQ_TAB_N + ilv)) + lds_half(t + 2u * (7 * MQ_TAB_N + ihv));
      return fmaxf(fmaxf(fmaxf(X, Y), (X + Y) * 0.70710670f), fmaxf(fmaxf(U, V) * 0.70710670f, (U + V) * 0.49999997f));
    };
    const float clo = lane < nq ? col_bound(lane) : 0.f;
    const float chi = lane + 32 < nq ? col_bound(lane + 32) : 0.f;
    // running bounds: lane l holds thr of queries l, l + 32
    const float tlo = lane < nq ? __uint_as_float(__ldcg(c.thr + q0 + lane)) : INFINITY;
    const float thi = lane + 32 < nq ? __uint_as_float(__ldcg(c.thr + q0 + lane + 32)) : INFINITY;
    unsigned long long pass =
        (unsigned long long)__ballot_sync(FULL, lane < nq && !(fmaf(clo, 1.f - 1e-4f, -lb_slack) > fmaxf(tlo, A.threshold))) |
        ((unsigned long long)__ballot_sync(FULL, lane + 32 < nq &&
                                                     !(fmaf(chi, 1.f - 1e-4f, -lb_slack) > fmaxf(thi, A.threshold)))
         << 32);
    if (!pass) continue;
    if (lane == 0) atomicAdd(&s_cnt[0], (unsigned)__popcll(pass));
    // ---- stage B (row term on the common grid), computed for the queries
    // still alive: nearest vertex of each point once per curve
    int vi[UP];
    float ve[UP];
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      const int i = lane + 32 * u;
      vi[u] = 0;
      ve[u] = INFINITY;  // beyond P: contributes max(dt - inf, 0) = 0
      if (i < P) {
        const float2 a = cur[i];
        const unsigned ix = min(__float2uint_rn(fmaf(a.x, ihx, ox)), (unsigned)G0);
        const unsigned iy = min(__float2uint_rn(fmaf(a.y, ihy, oy)), (unsigned)G0);
        const float ex = a.x - __fmaf_rn((float)ix, cx, lx), ey = a.y - __fmaf_rn((float)iy, cy, ly);
        vi[u] = (int)(ix * GR::V + iy) * 2 + (int)sdt_b;
        ve[u] = sqrt_approx(fmaf(ey, ey, ex * ex));
      }
    }
    bool expanded = false;
    float ar2 = 0.f;
    const long long rpos = A.pos_map ? A.pos_map[pos] : pos + A.pos_base;
    while (pass) {
      const int qg = __ffsll((long long)pass) - 1;
      pass &= pass - 1;
      const int qi = q0 + qg;
      // thr as read at the start of this curve: an older (larger) value is
      // still an upper bound of the final k-th best
      const float t = fmaxf(__shfl_sync(FULL, qg < 32 ? tlo : thi, qg & 31), A.threshold);
      const float colb0 = __shfl_sync(FULL, qg < 32 ? clo : chi, qg & 31);
      float acc = 0.f;
      const uint32_t qoff = (uint32_t)qg * GR::STRIDE * 2u;
#pragma unroll
      for (int u = 0; u < UP; ++u) acc += fmaxf(lds_half((uint32_t)vi[u] + qoff) - ve[u], 0.f);
      const float row0 = warp_sum(acc) * invP;
      if (fmaf(row0 + colb0, 1.f - 1e-4f, -lb_slack) > t) continue;
      if (lane == 0) atomicAdd(&s_cnt[1], 1u);
      // stage 1: four-corner row bound on the query's own 64x64 grid
      const float* pp = c.lb_par + (size_t)qi * 8;
      const float rowb = fmaxf(row0, curve_row_bound(cur, P, c.lb_dt + (size_t)qi * (LB_DT_BYTES / sizeof(__half)),
                                                     pp[0], pp[1], pp[2], pp[3], pp[4], pp[5], lane));
      if (fmaf(rowb + colb0, 1.f - 1e-4f, -lb_slack) > t) continue;
      if (lane == 0) atomicAdd(&s_cnt[2], 1u);
      // stage 2: plus the column term from 10-point run boxes
      const float2* qsrc = reinterpret_cast<const float2*>(A.queries) + (size_t)qi * Qn;
      QueryRegs<QS> Q;
      load_query<QS>(Q, qsrc, Qn, lane);
      // column term from coarse boxes (10 of 20-point runs), then 20 of
      // 10-point runs
#ifndef LA_MQ_RUN1
#define LA_MQ_RUN1 20  // C5: 50 / 25 / 20 / 16 / none: 20.6 / 19.2 / 18.9 / 19.1 / 19.4 ms
#endif
#if LA_MQ_RUN1 > 0
      const float colb1 = fmaxf(colb0, curve_col_bound<QS, LA_MQ_RUN1>(Q, cur, P, Qn, boxes, lane));
      if (fmaf(rowb + colb1, 1.f - 1e-4f, -lb_slack) > t) continue;
#else
      const float colb1 = colb0;
#endif
      if (lane == 0) atomicAdd(&s_cnt[3], 1u);
      __syncwarp();
      const float colb = fmaxf(colb1, curve_col_bound<QS, 10>(Q, cur, P, Qn, boxes, lane));
      if (fmaf(rowb + colb, 1.f - 1e-4f, -lb_slack) > t) continue;
      if (lane == 0) atomicAdd(&s_cnt[4], 1u);
      if (!expanded) {
        ar2 = 0.f;
        for (int i = lane; i < Ppad / 2; i += 32) {
          float4 e4 = make_float4(-2.f * BIG, -2.f * BIG, -2.f * BIG, -2.f * BIG);
          float2 n2 = make_float2(FAR_N, FAR_N);
          if (2 * i < P) {
            const float2 p0 = cur[2 * i];
            const float x = p0.x - 0.5f, y = p0.y - 0.5f;
            e4.x = -2.f * x; e4.z = -2.f * y; n2.x = fmaf(y, y, x * x); ar2 = fmaxf(ar2, n2.x);
          }
          if (2 * i + 1 < P) {
            const float2 p1 = cur[2 * i + 1];
            const float x = p1.x - 0.5f, y = p1.y - 0.5f;
            e4.y = -2.f * x; e4.w = -2.f * y; n2.y = fmaf(y, y, x * x); ar2 = fmaxf(ar2, n2.y);
          }
          exs[i] = e4;
          ens[i] = n2;
        }
        ar2 = __uint_as_float(__reduce_max_sync(FULL, __float_as_uint(ar2)));
        __syncwarp();
        expanded = true;
      }
      float d;
      if (expansion) {
        const float delta = 20.f * U32 * fmaxf(ar2, Q.r2);
        float err = 0.f;
        d = curve_chamfer<QS, false>(Q, exs, ens, P, Qn, lane, delta, err, rowbuf);
        if (!(err <= A.fixup_below)) d = direct_chamfer<QS>(qsrc, Qn, exs, ens, P, lane, rowbuf);
      } else {
        float dummy;
        d = curve_chamfer<QS, true>(Q, exs, ens, P, Qn, lane, 0.f, dummy, rowbuf);
      }
      if (lane == 0) atomicAdd(&s_cnt[5 + qg], 1u);  // full evaluations of the query
      const size_t lb = (size_t)qg * k;
      if (d < A.threshold) {
        if (lane == 0) atomicAdd(&s_nh[qg], 1ull);
        if (rpos < *(volatile long long*)&s_hit_pos[lb + k - 1])
          mq_insert(s_hit_d + lb, s_hit_pos + lb, s_hit_id + lb, &s_lock[qg], k, lane, d, rpos, id + A.id_base, true);
      } else {
        const float kd = *(volatile float*)&s_top_d[lb + k - 1];
        const long long kp = *(volatile long long*)&s_top_pos[lb + k - 1];
        if (key_less(d, rpos, kd, kp))
          mq_insert(s_top_d + lb, s_top_pos + lb, s_top_id + lb, &s_lock[qg], k, lane, d, rpos, id + A.id_base,
                    false);
        if (d < __uint_as_float(__ldcg(c.thr + qi)))
          publish_kth(c.thr + qi, c.slots + (size_t)qi * 32, k, lane, d, id);
      }
    }
  }
  __syncthreads();
  // flush: list blockIdx.x of each query of the group
  for (int qg = w; qg < nq; qg += MQ_W) {
    const int qi = q0 + qg;
    const size_t base = ((size_t)qi * c.nwarps_total + blockIdx.x) * k;
    if (lane < k) {
      const size_t lb = (size_t)qg * k + lane;
      c.ws_top_d[base + lane] = s_top_d[lb];
      c.ws_top_pos[base + lane] = s_top_pos[lb];
      c.ws_top_id[base + lane] = s_top_id[lb];
      c.ws_hit_d[base + lane] = s_hit_d[lb];
      c.ws_hit_pos[base + lane] = s_hit_pos[lb];
      c.ws_hit_id[base + lane] = s_hit_id[lb];
    }
    if (lane == 0) {
      c.ws_nhit[(size_t)qi * c.nwarps_total + blockIdx.x] = (long long)s_nh[qg];
      if (A.n_full && s_cnt[5 + qg])
        atomicAdd(reinterpret_cast<unsigned long long*>(A.n_full + qi), (unsigned long long)s_cnt[5 + qg]);
    }
  }
  // counters: survivors of stages 0/1/2 and full evaluations (whole group)
  if (threadIdx.x == 0) {
    if (A.n_stage)
      for (int j = 0; j < 5; ++j)
        atomicAdd(reinterpret_cast<unsigned long long*>(A.n_stage + j), (unsigned long long)s_cnt[j]);
  }
}

// ------------------------------------------------------------ tensor-core path
// (LA_CH_TENSOR; even P <= 256, Q <= 256)  Squared distances of all point
// pairs come from tcgen05.mma.kind::tf32 as |a|^2 + |b|^2 - 2 a.b with a
// 3xTF32 split (x = x_hi + x_lo, x_hi = x with the 13 low mantissa bits
// cleared) packed into K = 16:
//   A row (point a):  [a_hx, a_hy, a_hx, a_hy, a_lx, a_ly, n_ah, n_al, 1, 1, 0...]
//   B row (point b):  [-2b_hx, -2b_hy, -2b_lx, -2b_ly, -2b_hx, -2b_hy, 1, 1, n_bh, n_bl, 0...]
// (coordinates centred at (0.5, 0.5), n = |.|^2 split the same way; only the
// a_lo.b_lo term, 2^-22 relative, is dropped).  Both directions are MMAs:
// query rows x curve columns gives the query-side row minima, curve rows x
// query columns the curve-side ones, each a thread-local minimum over a
// TMEM row after tcgen05.ld.  Rows whose minimum falls below TC_RECHECK
// (d < 0.007, where the expansion's cancellation could move sqrt(d^2) by
// more than ~1e-5) are recomputed with direct differences from the raw
// points.  One CTA = 8 warps, 256 TMEM columns (two CTAs share an SM: one
// CTA's MMA overlaps the other's epilogue); one elected thread issues TMA
// and MMA.  Operands are K-major in shared memory without swizzle: 8-row x
// 16-byte core matrices, K-adjacent ones 128 B apart, 8-row groups 512 B.
constexpr int TC_K = 16;
constexpr int TC_ROWB = TC_K * 4;           // bytes per operand row
constexpr int TC_OP = 256 * TC_ROWB;        // bytes per operand buffer (256 rows)
#ifndef TC_RECHECK_V
#define TC_RECHECK_V 1.0e-6f
#endif
constexpr float TC_RECHECK = TC_RECHECK_V;         // squared distance below which a row minimum is recomputed
constexpr float TC_FAR = 1.0e30f;           // |b|^2 of padding columns: never a minimum
constexpr size_t TC_SMEM = 8 * TC_OP + 4 * PMAX * sizeof(float2) + PMAX * sizeof(float2) + 1024 * sizeof(float) +
                           26 * sizeof(uint64_t) + 2 * sizeof(uint32_t) + 4 * 16 * sizeof(float) + 64;

__device__ __forceinline__ int tc_off(int r, int k) {
  return (r >> 3) * 512 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4;
}
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// operand rows for a point (centred coordinates x, y); pad rows: zeros (A) or far (B)
__device__ __forceinline__ void tc_rows(unsigned char* A, unsigned char* B, int r, bool real, float x, float y) {
  float ra[TC_K], rb[TC_K];
#pragma unroll
  for (int k = 0; k < TC_K; ++k) ra[k] = rb[k] = 0.f;
  if (real) {
    const float hx = tf32_hi(x), hy = tf32_hi(y), lx = x - hx, ly = y - hy;
    const float n = fmaf(y, y, x * x);
    const float nh = tf32_hi(n), nl = n - nh;
    ra[0] = hx; ra[1] = hy; ra[2] = hx; ra[3] = hy; ra[4] = lx; ra[5] = ly; ra[6] = nh; ra[7] = nl;
    ra[8] = 1.f; ra[9] = 1.f;
    rb[0] = -2.f * hx; rb[1] = -2.f * hy; rb[2] = -2.f * lx; rb[3] = -2.f * ly; rb[4] = -2.f * hx;
    rb[5] = -2.f * hy; rb[6] = 1.f; rb[7] = 1.f; rb[8] = nh; rb[9] = nl;
  } else {
    rb[8] = TC_FAR;
  }
  if (A) {
#pragma unroll
    for (int k = 0; k < TC_K; k += 4)
      *reinterpret_cast<float4*>(A + tc_off(r, k)) = make_float4(ra[k], ra[k + 1], ra[k + 2], ra[k + 3]);
  }
  if (B) {
#pragma unroll
    for (int k = 0; k < TC_K; k += 4)
      *reinterpret_cast<float4*>(B + tc_off(r, k)) = make_float4(rb[k], rb[k + 1], rb[k + 2], rb[k + 3]);
  }
}

__device__ __forceinline__ uint64_t tc_desc(uint32_t addr) {
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46);
}
__device__ __forceinline__ uint32_t tc_idesc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void tc_mma(uint32_t tmem, uint32_t a_addr, uint32_t b_addr, int n) {
  const uint32_t idesc = tc_idesc(n);
#pragma unroll
  for (int ks = 0; ks < TC_K / 8; ++ks) {
    const uint64_t ad = tc_desc(a_addr + ks * 256), bd = tc_desc(b_addr + ks * 256);
    const uint32_t acc = ks > 0;
    asm volatile(
        "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
  }
}
// tc_mma / tc_commit are called by a whole warp (warp-uniform arguments) and
// issued by one elected lane: from a lane-0 branch ptxas wraps each MMA in a
// uniformity loop that costs several times the MMA itself
// (tools/micro/umma_small.cu)
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// min over 8 consecutive TMEM columns of this thread's row
__device__ __forceinline__ float tc_min8(uint32_t taddr) {
  uint32_t v[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  float m = min3f(__uint_as_float(v[0]), __uint_as_float(v[1]), __uint_as_float(v[2]));
  m = min3f(m, __uint_as_float(v[3]), __uint_as_float(v[4]));
  m = min3f(m, __uint_as_float(v[5]), __uint_as_float(v[6]));
  return fminf(m, __uint_as_float(v[7]));
}

// min over columns [c0, c1) of this thread's TMEM row: 64-column chunks as
// two x32 loads behind one wait, 8-column tail chunks as x8 loads
#define LA_TC_LD32(v, addr)                                                                                   \
  asm volatile(                                                                                               \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"       \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"                            \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),      \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), \
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),           \
        "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),           \
        "=r"(v[30]), "=r"(v[31])                                                                              \
      : "r"(addr))
__device__ __forceinline__ float tc_rowmin(uint32_t tbase, int c0, int c1) {
  float m0 = INFINITY, m1 = INFINITY, m2 = INFINITY, m3 = INFINITY;  // independent chains
  int col = c0;
  for (; col + 32 <= c1;) {
    uint32_t a[32];
    LA_TC_LD32(a, tbase + (uint32_t)col);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      m0 = min3f(m0, __uint_as_float(a[j]), __uint_as_float(a[j + 1]));
      m1 = min3f(m1, __uint_as_float(a[j + 2]), __uint_as_float(a[j + 3]));
      m2 = min3f(m2, __uint_as_float(a[j + 4]), __uint_as_float(a[j + 5]));
      m3 = min3f(m3, __uint_as_float(a[j + 6]), __uint_as_float(a[j + 7]));
    }
    col += 32;
  }
  for (; col < c1; col += 8) m0 = fminf(m0, tc_min8(tbase + (uint32_t)col));
  return fminf(fminf(m0, m1), fminf(m2, m3));
}


// Warp-specialised pipeline, one CTA per SM (512 TMEM columns = two
// 256-column accumulator slots):
//   warp 8 (producer): TMA of raw curves and, from one elected lane, the
//     MMAs; tile g = TPC c + t (curve c; t < MT1: query-row tiles, else
//     curve-row tiles) goes into TMEM slot g & 1;
//   warps 0-7 (epilogue): build each curve's operands (double-buffered),
//     then per tile: warp w reads TMEM lanes 32 (w & 3).. for column half
//     (w >> 2), row minima; warps w and w + 4 meet on a named barrier,
//     warp w < 4 combines, rechecks small minima and accumulates.
// Hand-offs are mbarriers: raw_full[4] (TMA, two curves ahead), op_full[2] (operands built),
// op_empty[2] (last MMA of a curve done with its operands), tmem_full[2]
// (MMA committed), tmem_empty[2] (8 epilogue warps done reading), raw_empty[4]
// (epilogue done with a raw curve: TMA may refill it).
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

constexpr int TC_GROUP_WARPS = 12;         // per epilogue group: 4 TMEM lane quarters x 3 column parts
constexpr int TC_EPI_WARPS = 2 * TC_GROUP_WARPS;  // group 0 takes the even tiles (slot 0), group 1 the odd
constexpr int TC_PRODUCER = TC_EPI_WARPS;      // warp index of the TMA/MMA warp
constexpr int TC_SELECT = TC_EPI_WARPS + 1;    // warp index of the top-k warp
constexpr int TC_CTA = (TC_EPI_WARPS + 2) * 32;
constexpr int TC_RING = 4;                     // finished-curve ring (epilogue -> top-k warp)

#ifdef LA_TC_PROF
__device__ unsigned long long g_tc_prof[16];
#define TCP_T0() long long _tp = clock64()
#define TCP_ADD(i) do { long long _n = clock64(); atomicAdd(&g_tc_prof[i], (unsigned long long)(_n - _tp)); _tp = _n; } while (0)
#else
#define TCP_T0() do {} while (0)
#define TCP_ADD(i) do {} while (0)
#endif

__global__ void __launch_bounds__(TC_CTA, 1) chamfer_tc_kernel(const ScanCtx c) {
  extern __shared__ __align__(1024) unsigned char tsm[];
  unsigned char* qA = tsm;                 // query as A (rows = query points)
  unsigned char* qB = tsm + TC_OP;         // query as B
  unsigned char* cAb = tsm + 2 * TC_OP;    // curve as A, 3 buffers
  unsigned char* cBb = tsm + 5 * TC_OP;    // curve as B, 3 buffers
  auto raw = reinterpret_cast<float2(*)[PMAX]>(tsm + 8 * TC_OP);                          // [4][PMAX]
  float2* qc = reinterpret_cast<float2*>(tsm + 8 * TC_OP + 4 * PMAX * sizeof(float2));    // centred query
  float* part = reinterpret_cast<float*>(tsm + 8 * TC_OP + 5 * PMAX * sizeof(float2));    // [2][2][2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(part + 1024);
  uint64_t* raw_full = bars;        // [4]
  uint64_t* raw_empty = bars + 4;   // [4]
  uint64_t* op_full = bars + 8;     // [3]
  uint64_t* op_empty = bars + 11;   // [3]
  uint64_t* tm_full = bars + 14;    // [2]
  uint64_t* tm_empty = bars + 16;   // [2]
  uint64_t* ring_full = bars + 18;  // [TC_RING]
  uint64_t* ring_empty = bars + 22; // [TC_RING]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 26);
  float* red = reinterpret_cast<float*>(tmem_slot + 2);  // [TC_RING][2 groups][4 quarters][2] sums
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int qi = blockIdx.y;
  const la_chamfer_args& A = c.a;
  const int P = A.P, Qn = A.Q;
  const int N1 = (P + 15) & ~15, N2 = (Qn + 15) & ~15;
  const int MT1 = (Qn + 127) / 128, MT2 = (P + 127) / 128;
  const int TPC = MT1 + MT2;
  const float2* qsrc = reinterpret_cast<const float2*>(A.queries) + (size_t)qi * Qn;
  const long long first = A.pos_begin + blockIdx.x;  // scan positions are int64 (N may exceed 2^31)
  const int stride = (int)gridDim.x;
  const int count = first < A.pos_end ? (int)((A.pos_end - first + stride - 1) / stride) : 0;  // per CTA
  const uint32_t bytes = (uint32_t)P * 8u;
  auto rec_of = [&](long long pos) -> long long { return A.order ? A.order[pos] : pos; };

  for (int r = tid; r < 256; r += TC_CTA) {
    const bool real = r < Qn;
    float2 q = make_float2(0.f, 0.f);
    if (real) {
      q = qsrc[r];
      q.x -= 0.5f;
      q.y -= 0.5f;
      qc[r] = q;
    }
    tc_rows(r < 128 * MT1 ? qA : nullptr, r < N2 ? qB : nullptr, r, real, q.x, q.y);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) {
      mbar_init(&raw_full[i], 1);
      mbar_init(&raw_empty[i], TC_EPI_WARPS);
    }
    for (int i = 0; i < TC_RING; ++i) {
      mbar_init(&ring_full[i], 8);
      mbar_init(&ring_empty[i], 1);
    }
    for (int i = 0; i < 3; ++i) {
      mbar_init(&op_full[i], TC_EPI_WARPS);
      mbar_init(&op_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tm_full[i], 1);
      mbar_init(&tm_empty[i], TC_GROUP_WARPS);
    }
    fence_mbar_init();
  }
  fence_proxy_async();  // query operands -> async proxy
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == TC_SELECT) {
    // ------------------------------------------------ top-k warp
    WarpList top, hit;
    list_init(top);
    list_init(hit);
    long long nhit = 0;
    uint32_t rf = 0;
    for (int ci = 0; ci < count; ++ci) {
      const int rs = ci % TC_RING;
      mbar_wait(&ring_full[rs], (rf >> rs) & 1u);
      rf ^= 1u << rs;
      const float* rr = red + rs * 16;
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) {  // fixed order: group 0 quarters 0-3, then group 1
        s0 += rr[2 * k];
        s1 += rr[2 * k + 1];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&ring_empty[rs]);
      const float d = s0 / (float)Qn + s1 / (float)P;
      const long long pos = first + (long long)ci * stride;
      const long long id = rec_of(pos);
      if (id != A.exclude_id) {
        if (A.all_d && lane == 0) A.all_d[(size_t)qi * A.N + id] = d;
        const long long rpos = A.pos_map ? A.pos_map[pos] : pos + A.pos_base;
        consider(top, hit, nhit, c, lane, d, rpos, id + A.id_base);
      }
    }
    flush_lists(c, qi, blockIdx.x, lane, top, hit, nhit);
  } else if (warp == TC_PRODUCER) {
    // ------------------------------------------------ producer warp
    // raw curves are prefetched two ahead into four buffers (a buffer is
    // refilled once the epilogue released the curve it held, 4 curves back)
    {
      uint32_t re_ph = 0, of_ph = 0, te_ph = 0;
      auto tma = [&](int ci) {
        const int rb = ci & 3;
        if (ci >= 4) {
          mbar_wait(&raw_empty[rb], (re_ph >> rb) & 1u);
          re_ph ^= 1u << rb;
        }
        if (lane == 0) {
          mbar_expect_tx(&raw_full[rb], bytes);
          tma_load_1d(&raw[rb][0], A.db + (size_t)rec_of(first + (long long)ci * stride) * P * 2, bytes,
                      &raw_full[rb]);
        }
        __syncwarp();
      };
      if (count > 0) tma(0);
      if (count > 1) tma(1);
      int g = 0;
      for (int ci = 0; ci < count; ++ci) {
        if (ci + 2 < count) tma(ci + 2);
        const int b = ci % 3;
        TCP_T0();
        mbar_wait(&op_full[b], (of_ph >> b) & 1u);  // operands of curve ci built
        of_ph ^= 1u << b;
        TCP_ADD(0);
        tc_fence_after();
        for (int t = 0; t < TPC; ++t, ++g) {
          const int slot = g & 1;
          if (g >= 2) {
            TCP_T0();
            mbar_wait(&tm_empty[slot], (te_ph >> slot) & 1u);
            te_ph ^= 1u << slot;
            tc_fence_after();
            TCP_ADD(1);
          }
          const uint32_t d = tmem + (uint32_t)(slot * 256);
          if (t < MT1)
            tc_mma(d, smem_u32(qA) + t * 8192, smem_u32(cBb + b * TC_OP), N1);
          else
            tc_mma(d, smem_u32(cAb + b * TC_OP) + (t - MT1) * 8192, smem_u32(qB), N2);
          tc_commit(&tm_full[slot]);
        }
        tc_commit(&op_empty[b]);  // fires when all MMAs of curve ci are complete
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ epilogue warps
    uint32_t rf_ph = 0, oe_ph = 0, tf_ph = 0, re_ph = 0;
    const int grp = warp / TC_GROUP_WARPS, gw = warp % TC_GROUP_WARPS;
    const int quarter = gw & 3, half = gw >> 2;  // half = column part 0..2 (0: combiner warp)
    auto build = [&](int ci) {
      const int b = ci % 3, rb = ci & 3;
      mbar_wait(&raw_full[rb], (rf_ph >> rb) & 1u);
      rf_ph ^= 1u << rb;
      if (ci >= 3) {  // MMAs of curve ci - 3 done with operand buffer b
        mbar_wait(&op_empty[b], (oe_ph >> b) & 1u);
        oe_ph ^= 1u << b;
      }
      const float2* cur = &raw[rb][0];
      unsigned char* cA = cAb + b * TC_OP;
      unsigned char* cB = cBb + b * TC_OP;
      for (int r = tid; r < 256; r += TC_EPI_WARPS * 32) {
        const bool real = r < P;
        float2 p = make_float2(0.f, 0.f);
        if (real) {
          p = cur[r];
          p.x -= 0.5f;
          p.y -= 0.5f;
        }
        tc_rows(r < 128 * MT2 ? cA : nullptr, r < N1 ? cB : nullptr, r, real, p.x, p.y);
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&op_full[b]);
        if (half) mbar_arrive(&raw_empty[rb]);  // column-half warps never read raw curve ci again
      }
    };
    if (count > 0) build(0);
    int g = 0;
    float sum0 = 0.f, sum1 = 0.f;
    for (int ci = 0; ci < count; ++ci) {
      TCP_T0();
      if (ci + 1 < count) build(ci + 1);  // overlaps this curve's MMAs
      if (warp == 0 && lane == 0) TCP_ADD(2);
      const float2* cur = &raw[ci & 3][0];
      for (int t = 0; t < TPC; ++t, ++g) {
        if ((g & 1) != grp) continue;  // the other group's tile
        const int dir = t < MT1 ? 0 : 1, mt = dir == 0 ? t : t - MT1;
        const int NN = dir == 0 ? N1 : N2, rows = dir == 0 ? Qn : P;
        const int slot = g & 1;
#ifdef LA_TC_PROF
        long long _tp = clock64();
#endif
        mbar_wait(&tm_full[slot], (tf_ph >> slot) & 1u);
        tf_ph ^= 1u << slot;
        tc_fence_after();
        if (warp == 0 && lane == 0) TCP_ADD(3);
        const int ncol8 = NN >> 3, c0 = ((ncol8 * half) / 3) << 3, c1 = ((ncol8 * (half + 1)) / 3) << 3;
        const uint32_t tbase = tmem + (uint32_t)(slot * 256) + ((uint32_t)(quarter * 32) << 16);
        const float m = tc_rowmin(tbase, c0, c1);
        if (warp == 0 && lane == 0) TCP_ADD(4);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tm_empty[slot]);  // TMEM slot may be overwritten
        float* pp = part + (grp * 2 + ((g >> 1) & 1)) * 2 * 128;  // per group, double-buffered
        if (half) pp[(half - 1) * 128 + quarter * 32 + lane] = m;
        named_sync(1 + grp * 4 + quarter, 96);  // the 3 column-part warps of this lane quarter
        if (warp == 0 && lane == 0) TCP_ADD(5);
        if (!half) {
          const int row = mt * 128 + quarter * 32 + lane;
          const bool real = row < rows;
          const float mo = fminf(pp[quarter * 32 + lane], pp[128 + quarter * 32 + lane]);
          float mm = real ? fminf(m, mo) : INFINITY;
          unsigned need = __ballot_sync(FULL, real && mm < TC_RECHECK);
#ifdef LA_TC_PROF
          if (lane == 0) atomicAdd(&g_tc_prof[7], (unsigned long long)__popc(need));
          if (lane == 0) atomicAdd(&g_tc_prof[8], 1ull);
#endif
          while (__builtin_expect(need != 0u, 0)) {  // cancellation zone: direct differences, the warp sweeping the other side
            const int src = __ffs(need) - 1;
            need &= need - 1;
            const int rr = mt * 128 + quarter * 32 + src;
            const float2 pt = dir == 0 ? qc[rr] : make_float2(cur[rr].x - 0.5f, cur[rr].y - 0.5f);
            const int no = dir == 0 ? P : Qn;
            float e = INFINITY;
            for (int j = lane; j < no; j += 32) {
              const float2 o = dir == 0 ? make_float2(cur[j].x - 0.5f, cur[j].y - 0.5f) : qc[j];
              const float dx = pt.x - o.x, dy = pt.y - o.y;
              e = fminf(e, fmaf(dy, dy, dx * dx));
            }
            for (int o = 16; o > 0; o >>= 1) e = fminf(e, __shfl_xor_sync(FULL, e, o));
            if (lane == src) mm = e;
          }
          if (real) {  // MUFU square root (2^-22 relative): far inside the 1e-4 tolerance
            float r;
            asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(fmaxf(mm, 0.f)));
            if (dir == 0) sum0 += r;
            else sum1 += r;
          }
          if (warp == 0 && lane == 0) TCP_ADD(6);
        }
      }
      // curve ci complete: the combiner warps (0-3) hand their sums to the top-k warp
      if (!half) {
        const float s0 = warp_sum(sum0), s1 = warp_sum(sum1);
        const int rs = ci % TC_RING;
        if (ci >= TC_RING) {
          mbar_wait(&ring_empty[rs], (re_ph >> rs) & 1u);
          re_ph ^= 1u << rs;
        }
        if (lane == 0) {
          red[rs * 16 + (grp * 4 + quarter) * 2] = s0;
          red[rs * 16 + (grp * 4 + quarter) * 2 + 1] = s1;
          mbar_arrive(&ring_full[rs]);
          mbar_arrive(&raw_empty[ci & 3]);  // rechecks of curve ci are done
        }
      }
      sum0 = sum1 = 0.f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// ------------------------------------------------------------ generic path
// one CTA per (scan position, query): any P, Q; distances to a dense buffer
__global__ void __launch_bounds__(256) chamfer_generic_kernel(const la_chamfer_args A, float* dense) {
  extern __shared__ float2 gsm[];
  float2* pa = gsm;
  float2* pq = gsm + A.P;
  __shared__ float red[2][8];
  const int qi = blockIdx.y;
  const float2* qsrc = reinterpret_cast<const float2*>(A.queries) + (size_t)qi * A.Q;
  for (int i = threadIdx.x; i < A.Q; i += 256) pq[i] = qsrc[i];
  for (long long pos = A.pos_begin + blockIdx.x; pos < A.pos_end; pos += gridDim.x) {
    const long long id = A.order ? A.order[pos] : pos;
    const float2* src = reinterpret_cast<const float2*>(A.db) + (size_t)id * A.P;
    __syncthreads();
    for (int i = threadIdx.x; i < A.P; i += 256) pa[i] = src[i];
    __syncthreads();
    float rs = 0.0f, cs = 0.0f;
    for (int i = threadIdx.x; i < A.P; i += 256) {
      float m = INFINITY;
      for (int j = 0; j < A.Q; ++j) {
        const float dx = pa[i].x - pq[j].x, dy = pa[i].y - pq[j].y;
        m = fminf(m, fmaf(dy, dy, dx * dx));
      }
      rs += sqrtf(m);
    }
    for (int j = threadIdx.x; j < A.Q; j += 256) {
      float m = INFINITY;
      for (int i = 0; i < A.P; ++i) {
        const float dx = pa[i].x - pq[j].x, dy = pa[i].y - pq[j].y;
        m = fminf(m, fmaf(dy, dy, dx * dx));
      }
      cs += sqrtf(m);
    }
    rs = warp_sum(rs);
    cs = warp_sum(cs);
    if ((threadIdx.x & 31) == 0) {
      red[0][threadIdx.x >> 5] = rs;
      red[1][threadIdx.x >> 5] = cs;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      float r = 0.0f, q = 0.0f;
      for (int i = 0; i < 8; ++i) {
        r += red[0][i];
        q += red[1][i];
      }
      const float d = r / (float)A.P + q / (float)A.Q;
      dense[(size_t)qi * A.N + id] = d;
    }
  }
}

// selection over dense distances (generic path): same per-warp lists
__global__ void __launch_bounds__(CT) select_kernel(const ScanCtx c) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, qi = blockIdx.y;
  const la_chamfer_args& A = c.a;
  const int gw = blockIdx.x * CW + w;
  const long long stride = (long long)gridDim.x * CW;
  WarpList top, hit;
  list_init(top);
  list_init(hit);
  long long nhit = 0;
  for (long long pos = A.pos_begin + gw; pos < A.pos_end; pos += stride) {
    const long long id = A.order ? A.order[pos] : pos;
    if (id == A.exclude_id) continue;
    const float d = c.dense[(size_t)qi * A.N + id];
    const long long rpos = A.pos_map ? A.pos_map[pos] : pos + A.pos_base;
    consider(top, hit, nhit, c, lane, d, rpos, id + A.id_base);
  }
  flush_lists(c, qi, gw, lane, top, hit, nhit);
}

// merge per-warp lists: k rounds of CTA-wide argmin (one CTA per query)
__global__ void __launch_bounds__(1024) merge_kernel(const ScanCtx c) {
  const int qi = blockIdx.x;
  const la_chamfer_args& A = c.a;
  const int k = A.k;
  const long long n = (long long)c.nwarps_total * k;
  const size_t base = (size_t)qi * n;
  __shared__ float sd[32];
  __shared__ long long sp[32];
  __shared__ long long si[32];
  __shared__ long long sidx[32];
  __shared__ long long nh[32];
  // total hits
  long long h = 0;
  for (long long i = threadIdx.x; i < c.nwarps_total; i += 1024) h += c.ws_nhit[(size_t)qi * c.nwarps_total + i];
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(FULL, h, o);
  if ((threadIdx.x & 31) == 0) nh[threadIdx.x >> 5] = h;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int i = 0; i < 32; ++i) t += nh[i];
    if (A.n_hits) A.n_hits[qi] = t;
  }
  for (int pass = 0; pass < 2; ++pass) {
    float* D = pass == 0 ? c.ws_top_d : c.ws_hit_d;
    long long* Pp = pass == 0 ? c.ws_top_pos : c.ws_hit_pos;
    long long* I = pass == 0 ? c.ws_top_id : c.ws_hit_id;
    float* od = pass == 0 ? A.top_d : A.hit_d;
    int64_t* op = pass == 0 ? A.top_pos : A.hit_pos;
    int64_t* oi = pass == 0 ? A.top_id : A.hit_id;
    const bool by_pos = pass == 1;
    for (int r = 0; r < k; ++r) {
      float bd = INFINITY;
      long long bp = LLONG_MAX, bi = -1, bx = -1;
      for (long long i = threadIdx.x; i < n; i += 1024) {
        const long long p = Pp[base + i];
        if (p == LLONG_MAX) continue;  // empty or taken
        const float d = D[base + i];
        const bool better = by_pos ? (p < bp) : key_less(d, p, bd, bp);
        if (better) {
          bd = d; bp = p; bi = I[base + i]; bx = i;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const float od_ = __shfl_xor_sync(FULL, bd, o);
        const long long op_ = __shfl_xor_sync(FULL, bp, o);
        const long long oi_ = __shfl_xor_sync(FULL, bi, o);
        const long long ox_ = __shfl_xor_sync(FULL, bx, o);
        const bool better = by_pos ? (op_ < bp) : key_less(od_, op_, bd, bp);
        if (better) { bd = od_; bp = op_; bi = oi_; bx = ox_; }
      }
      if ((threadIdx.x & 31) == 0) {
        sd[threadIdx.x >> 5] = bd; sp[threadIdx.x >> 5] = bp;
        si[threadIdx.x >> 5] = bi; sidx[threadIdx.x >> 5] = bx;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        float d0 = sd[0]; long long p0 = sp[0], i0 = si[0], x0 = sidx[0];
        for (int j = 1; j < 32; ++j) {
          const bool better = by_pos ? (sp[j] < p0) : key_less(sd[j], sp[j], d0, p0);
          if (better) { d0 = sd[j]; p0 = sp[j]; i0 = si[j]; x0 = sidx[j]; }
        }
        if (od) od[(size_t)qi * k + r] = x0 >= 0 ? d0 : INFINITY;
        if (op) op[(size_t)qi * k + r] = x0 >= 0 ? p0 : -1;
        if (oi) oi[(size_t)qi * k + r] = x0 >= 0 ? i0 : -1;
        if (x0 >= 0) Pp[base + x0] = LLONG_MAX;  // consume
      }
      __syncthreads();
    }
  }
}


// ---- merge of per-shard lists gathered from every rank (dist.gather_merge):
// packed rows [world][NQ][6k + 1] int64 = top_d bits, top_id, top_pos,
// hit_d bits, hit_id, hit_pos (k each), n_hits.  Non-hits by (d, global scan
// position), hits by position (atlas.py:207-235 over the union of shards);
// entries with id < 0 are empty.  One CTA per query, rank selection.
__global__ void __launch_bounds__(256) shard_merge_kernel(const int64_t* __restrict__ g, int world, int NQ, int k,
                                                          float* top_d, int64_t* top_id, int64_t* top_pos,
                                                          float* hit_d, int64_t* hit_id, int64_t* hit_pos,
                                                          int64_t* n_hits) {
  const int qi = blockIdx.x;
  const int row = 6 * k + 1;
  const int n = world * k;
  __shared__ int nvalid[2];
  if (threadIdx.x < 2) nvalid[threadIdx.x] = 0;
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {  // 0: non-hits, 1: hits
    const int c0 = pass * 3 * k;
    float* od = pass ? hit_d : top_d;
    int64_t* oi = pass ? hit_id : top_id;
    int64_t* op = pass ? hit_pos : top_pos;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int64_t* r = g + ((size_t)(i / k) * NQ + qi) * row;
      const int e = i % k;
      const long long id = r[c0 + k + e];
      if (id < 0) continue;
      const float d = __int_as_float((int)(r[c0 + e] & 0xffffffffll));
      const long long pos = r[c0 + 2 * k + e];
      int rank = 0;
      for (int j = 0; j < n; ++j) {
        const int64_t* rj = g + ((size_t)(j / k) * NQ + qi) * row;
        const int ej = j % k;
        if (rj[c0 + k + ej] < 0) continue;
        const float dj = __int_as_float((int)(rj[c0 + ej] & 0xffffffffll));
        const long long pj = rj[c0 + 2 * k + ej];
        const bool less = pass ? (pj < pos || (pj == pos && j < i))
                               : (key_less(dj, pj, d, pos) || (dj == d && pj == pos && j < i));
        rank += less;
      }
      atomicAdd(&nvalid[pass], 1);
      if (rank < k) {
        od[(size_t)qi * k + rank] = d;
        oi[(size_t)qi * k + rank] = id;
        op[(size_t)qi * k + rank] = pos;
      }
    }
  }
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass)
    for (int r = nvalid[pass] + threadIdx.x; r < k; r += blockDim.x) {
      (pass ? hit_d : top_d)[(size_t)qi * k + r] = INFINITY;
      (pass ? hit_id : top_id)[(size_t)qi * k + r] = -1;
      (pass ? hit_pos : top_pos)[(size_t)qi * k + r] = -1;
    }
  if (threadIdx.x == 0 && n_hits) {
    long long h = 0;
    for (int w = 0; w < world; ++w) h += g[((size_t)w * NQ + qi) * row + 6 * k];
    n_hits[qi] = h;
  }
}

struct Plan {
  bool fast;
  int qs;
  int grid;        // CTAs per query (x)
  int nwarps;      // per query
  size_t ws_lists; // bytes of list area
  size_t ws_dense; // bytes of dense scratch (generic path without all_d)
  bool prune;      // exact row-bound pruning with a seed scan (fast path, top-k only)
  long long seed_end;
  int seed_grid;
  size_t ws_prune; // bytes of the pruning area
  bool index;      // indexed scan (cells given, one query): seed, bound step, scan of the survivors
  bool index_mq;   // the same for several queries (multi-query seed and bound step, per-query survivor lists)
  long long mq_seed_end;
  int iq_grid;     // CTAs per query of the survivors' scan
  size_t ws_index;
  // multi-query kernel (pruned, NQ >= 2)
  bool mq;
  int mq_g0;       // common grid cells per axis (32 or 64)
  int mq_qg;       // queries per group
  int mq_groups;
  int mq_grid;     // CTAs per group (= lists per query)
  size_t mq_smem;
};

// resident CTAs per SM of chamfer_scan_kernel<qs> (the register budget of
// LA_CH_MINB and ~90 KB of shared memory -- ten warps' curve double buffers,
// expanded curves and row buffers plus the 16.3 KB vertex + cell tables --
// allow 2), per device; racing threads compute and store the same value
// (relaxed atomics).  Unpruned scans reserve the tables too (unused).
int scan_occupancy(int qs) {
  static std::atomic<int> cache[64][9];
  if (qs < 1 || qs > 8) return 3;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 3;
  const int hit = cache[dev][qs].load(std::memory_order_relaxed);
  if (hit) return hit;
  const void* k = nullptr;
  switch (qs) {
    case 1: k = (const void*)chamfer_scan_kernel<1>; break;
    case 2: k = (const void*)chamfer_scan_kernel<2>; break;
    case 3: k = (const void*)chamfer_scan_kernel<3>; break;
    case 4: k = (const void*)chamfer_scan_kernel<4>; break;
    case 5: k = (const void*)chamfer_scan_kernel<5>; break;
    case 6: k = (const void*)chamfer_scan_kernel<6>; break;
    case 7: k = (const void*)chamfer_scan_kernel<7>; break;
    default: k = (const void*)chamfer_scan_kernel<8>; break;
  }
  int occ = 0;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SCAN_SMEM) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, CT, SCAN_SMEM) != cudaSuccess || occ < 1)
    occ = 3;
  cache[dev][qs].store(occ, std::memory_order_relaxed);
  return occ;
}

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

Plan make_plan(const la_chamfer_args* a) {
  Plan p{};
  const long long npos = a->pos_end - a->pos_begin;
  p.fast = a->P <= PMAX && a->Q <= 256 && a->Q >= 1;
  p.qs = (a->Q + 31) / 32;
  int sms = sm_count();
  if (sms <= 0) sms = 148;
  long long want = (npos + CW - 1) / CW;
  // one full wave of resident CTAs (a grid beyond it runs a second, mostly
  // idle wave); with several queries, CTAs per query so that the whole grid
  // fills whole waves
  const long long wave = (long long)sms * (p.fast ? scan_occupancy(p.qs) : 4);
  long long cap = 2 * wave;  // single query: two waves balance the tail best (measured 1/2/4/8: +2.4 % at 2)
  if (a->NQ > 1) {
    cap = (wave + a->NQ - 1) / a->NQ;
    double best = 0.0;
    for (int k = 1; k <= 32; ++k) {
      const long long gk = ((long long)k * wave + a->NQ - 1) / a->NQ;
      const long long tot = gk * a->NQ, waves = (tot + wave - 1) / wave;
      const double eff = (double)tot / (double)(waves * wave);
      if (eff > best + 1e-9) {
        best = eff;
        cap = gk;
      }
      if (eff >= 0.97 || gk >= want) break;
    }
  }
  if (cap < 1) cap = 1;
  long long g = want < cap ? want : cap;
  if (g < 1) g = 1;
  p.grid = (int)g;
  p.nwarps = p.grid * CW;
  const size_t per = (size_t)a->NQ * p.nwarps * (a->k > 0 ? a->k : 1);
  p.ws_lists = per * (2 * sizeof(float) + 4 * sizeof(long long)) + (size_t)a->NQ * p.nwarps * sizeof(long long);
  p.ws_dense = (!p.fast && !a->all_d) ? (size_t)a->NQ * a->N * sizeof(float) : 0;
  p.prune = p.fast && a->k > 0 && !a->all_d && !(a->flags & (LA_CH_TENSOR | LA_CH_NO_PRUNE)) &&
            npos >= PRUNE_MIN_POS;
  if (p.prune) {
    // optional seed scan (LA_CH_SEED_SCAN): the exact k-th of a 1/128
    // prefix published before the main scan; off by default (the slot
    // minima converge within the first wave and measured faster)
    p.index = a->cells != nullptr && a->NQ == 1 && !(a->flags & LA_CH_NO_INDEX);
    const long long seed_div = p.index ? LA_CH_INDEX_SEED_DIV : (a->flags & LA_CH_SEED_SCAN) ? 128 : 0;
    long long sn = seed_div > 0 ? npos / seed_div : 0;
    if (seed_div > 0 && sn < 64LL * a->k) sn = 64LL * a->k;
    if (sn > npos) sn = npos;
    p.seed_end = a->pos_begin + sn;
    long long sg = (sn + 8LL * CW - 1) / (8LL * CW);
    if (sg > p.grid) sg = p.grid;
    if (sg < 1) sg = 1;
    p.seed_grid = (int)sg;
    p.ws_prune = (size_t)a->NQ * (LB_DT_BYTES + 8 * sizeof(float) + 33 * sizeof(unsigned)) + 16 +
                 (size_t)a->NQ * a->k * 2 * (sizeof(float) + 2 * sizeof(long long)) + 256;
    if (p.index) {
      // cell table, the survivors' records and reported positions, their count
      p.ws_index = align_up((size_t)IDX_TAB * sizeof(unsigned short)) +
                   2 * align_up((size_t)npos * sizeof(long long)) + 256 + align_up((CD_CELLS + 1) * sizeof(unsigned));
      if (a->coarse && a->fine)
        p.ws_index += 2 * align_up((size_t)npos * sizeof(long long)) + align_up((CD2_CELLS / 4 + 1) * sizeof(unsigned));
    }
    p.mq = a->NQ >= 2 && !(a->flags & LA_CH_NO_MQ) && (a->P % 2) == 0;
    if (p.mq) {
      p.mq_g0 = (a->flags & LA_CH_MQ_FINE) ? 64 : 32;
      const int stride = p.mq_g0 == 64 ? MQGrid<64>::STRIDE : MQGrid<32>::STRIDE;
      // largest group whose shared memory fits one CTA per SM, then groups
      // of equal size
      const size_t cap = 227 * 1024 - 1024;
      int qg = MQ_MAXG;
      while (qg > 1 && mq_smem(qg, a->k, stride, a->P).total > cap) --qg;
      p.mq_groups = (a->NQ + qg - 1) / qg;
      p.mq_qg = (a->NQ + p.mq_groups - 1) / p.mq_groups;
      p.mq_smem = mq_smem(p.mq_qg, a->k, stride, a->P).total;
      long long gx = ((long long)sms + p.mq_groups - 1) / p.mq_groups;  // one wave of 1 CTA per SM
      const long long wantx = (npos + MQ_W - 1) / MQ_W;
      if (gx > wantx) gx = wantx;
      if (gx < 1) gx = 1;
      p.mq_grid = (int)gx;
      if (p.mq_grid > p.nwarps) {  // lists per query: the workspace holds max(nwarps, mq_grid)
        p.nwarps = p.mq_grid;
        const size_t per2 = (size_t)a->NQ * p.nwarps * (a->k > 0 ? a->k : 1);
        p.ws_lists = per2 * (2 * sizeof(float) + 4 * sizeof(long long)) + (size_t)a->NQ * p.nwarps * sizeof(long long);
      }
      p.ws_prune += (size_t)a->NQ * (stride * sizeof(__half) + MQ_TAB_BYTES) + 16 * sizeof(float) + 256;
      // indexed: multi-query kernel over a seed prefix, bound step for every
      // (query, curve), then each query's survivors with the single-query
      // kernel (lists of up to npos entries per query)
      p.index_mq = a->cells != nullptr && (a->flags & LA_CH_INDEX_MQ) && !(a->flags & LA_CH_NO_INDEX) && a->P <= 256 &&
                   (long long)a->NQ * npos <= (1ll << 28);
      if (p.index_mq) {
        long long sn = npos / LA_CH_INDEX_MQ_SEED_DIV;
        if (sn < 4096) sn = 4096;
        if (sn > npos) sn = npos;
        p.mq_seed_end = a->pos_begin + sn;
        long long gq = ((long long)sms * scan_occupancy(p.qs) + a->NQ - 1) / a->NQ;  // one wave over all queries
        if (gq < 1) gq = 1;
        if (gq > p.nwarps) gq = p.nwarps;
        p.iq_grid = (int)gq;
        p.ws_index = align_up((size_t)a->NQ * IDX_TAB * sizeof(unsigned short)) +
                     2 * align_up((size_t)a->NQ * npos * sizeof(long long)) + align_up((size_t)a->NQ * 8) + 256 +
                     align_up((size_t)a->NQ * (CD_CELLS / 4 + 1) * sizeof(unsigned));
      }
    }
  }
  return p;
}

}  // namespace
}  // namespace la

using namespace la;

extern "C" {

int la_merge_shard_lists(const int64_t* gathered, int32_t world, int32_t NQ, int32_t k, float* top_d,
                         int64_t* top_id, int64_t* top_pos, float* hit_d, int64_t* hit_id, int64_t* hit_pos,
                         int64_t* n_hits, void* stream) {
  if (!gathered || world < 1 || NQ < 1 || k < 1 || k > LA_MAX_TOPK || !top_d || !top_id || !top_pos || !hit_d ||
      !hit_id || !hit_pos)
    return fail(LA_EINVAL, "la_merge_shard_lists: bad args");
  if (NQ > 2147483647 || (long long)world * k > (1 << 20)) return fail(LA_ERANGE, "la_merge_shard_lists: too large");
  shard_merge_kernel<<<NQ, 256, 0, static_cast<cudaStream_t>(stream)>>>(gathered, world, NQ, k, top_d, top_id,
                                                                       top_pos, hit_d, hit_id, hit_pos, n_hits);
  return cuda_status("la_merge_shard_lists");
}

size_t la_chamfer_workspace(const la_chamfer_args* a) {
  if (!a) return 0;
  const Plan p = make_plan(a);
  return align_up(p.ws_lists) + align_up(p.ws_dense) + align_up(p.ws_prune) + align_up(p.ws_index) + 1024;
}

int la_chamfer_index(const float* db, int64_t N, int32_t P, uint16_t* cells, uint8_t* coarse, uint8_t* fine,
                     void* stream) {
  if (N < 0 || P < 1 || !db || !cells) return fail(LA_EINVAL, "la_chamfer_index: bad args");
  if (N == 0) return 0;
  if (coarse || fine) {
    int sm = sm_count();
    if (sm <= 0) sm = 148;
    long long gc = (N + 7) / 8;
    if (gc > (long long)sm * 8) gc = (long long)sm * 8;
    if (coarse)
      index_coarse_kernel<CDG><<<(unsigned)gc, 256, 0, static_cast<cudaStream_t>(stream)>>>(
          reinterpret_cast<const float2*>(db), N, P, coarse);
    if (fine)
      index_coarse_kernel<CD2G><<<(unsigned)gc, 256, 0, static_cast<cudaStream_t>(stream)>>>(
          reinterpret_cast<const float2*>(db), N, P, fine);
  }
  const long long n = (long long)N * idx_row(P);
  int sms = sm_count();
  if (sms <= 0) sms = 148;
  long long g = (n + 255) / 256;
  if (g > (long long)sms * 16) g = (long long)sms * 16;
  index_kernel<<<(unsigned)g, 256, 0, static_cast<cudaStream_t>(stream)>>>(reinterpret_cast<const float2*>(db), N, P,
                                                                           cells);
  return cuda_status("la_chamfer_index");
}

int la_chamfer_topk(const la_chamfer_args* a, void* stream) {
  if (!a) return fail(LA_EINVAL, "la_chamfer_topk: null args");
  if (a->N < 0 || a->P < 1 || a->Q < 1 || a->NQ < 1 || !a->db || !a->queries)
    return fail(LA_EINVAL, "la_chamfer_topk: bad sizes/buffers");
  if (a->k < 0 || a->k > LA_MAX_TOPK) return fail(LA_ERANGE, "la_chamfer_topk: k=%d beyond %d", a->k, LA_MAX_TOPK);
  if (a->pos_begin < 0 || a->pos_end > a->N || a->pos_begin > a->pos_end)
    return fail(LA_EINVAL, "la_chamfer_topk: bad scan range");
  if (a->k > 0 && (!a->top_d || !a->top_id || !a->top_pos || !a->hit_d || !a->hit_id || !a->hit_pos))
    return fail(LA_EINVAL, "la_chamfer_topk: k > 0 needs top_* and hit_* outputs");
  if (a->k == 0 && !a->all_d) return fail(LA_EINVAL, "la_chamfer_topk: nothing to output");
  if (a->NQ > 65535) return fail(LA_ERANGE, "la_chamfer_topk: NQ too large");
  const Plan p = make_plan(a);
  if (!a->ws || a->ws_bytes < la_chamfer_workspace(a)) return fail(LA_EWS, "la_chamfer_topk: workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ScanCtx c{};
  c.a = *a;
  c.nwarps_total = p.nwarps;
  unsigned char* w = static_cast<unsigned char*>(a->ws);
  const size_t per = (size_t)a->NQ * p.nwarps * (a->k > 0 ? a->k : 1);
  c.ws_top_pos = reinterpret_cast<long long*>(w); w += per * sizeof(long long);
  c.ws_top_id = reinterpret_cast<long long*>(w); w += per * sizeof(long long);
  c.ws_hit_pos = reinterpret_cast<long long*>(w); w += per * sizeof(long long);
  c.ws_hit_id = reinterpret_cast<long long*>(w); w += per * sizeof(long long);
  c.ws_nhit = reinterpret_cast<long long*>(w); w += (size_t)a->NQ * p.nwarps * sizeof(long long);
  c.ws_top_d = reinterpret_cast<float*>(w); w += per * sizeof(float);
  c.ws_hit_d = reinterpret_cast<float*>(w); w += per * sizeof(float);
  w = static_cast<unsigned char*>(a->ws) + align_up(p.ws_lists);
  c.dense = a->all_d ? a->all_d : reinterpret_cast<float*>(w);
  const dim3 grid(p.grid, a->NQ);
  if (p.fast && (a->flags & LA_CH_TENSOR) && (a->P % 2) == 0) {
    // one list per CTA: one CTA per SM (512 TMEM columns), grid split over the queries
    int sms = sm_count();
    long long want = a->pos_end - a->pos_begin;
    long long g = (long long)sms;
    if (a->NQ > 1) {
      // CTAs per query so that g x NQ fills whole waves of one CTA per SM
      double best = 0.0;
      for (int k = 1; k <= 32; ++k) {
        const long long gk = ((long long)k * sms + a->NQ - 1) / a->NQ;
        if (gk > p.nwarps || gk > want) break;
        const long long tot = gk * a->NQ, waves = (tot + sms - 1) / sms;
        const double eff = (double)tot / (double)(waves * sms);
        if (eff > best + 1e-9) {
          best = eff;
          g = gk;
        }
        if (eff >= 0.97) break;
      }
      if (best == 0.0) g = ((long long)sms + a->NQ - 1) / a->NQ;
    }
    if (g > want) g = want;
    if (g < 1) g = 1;
    if (g > p.nwarps) g = p.nwarps;  // list workspace is sized for p.nwarps lists per query
    ScanCtx ct = c;
    ct.nwarps_total = (int)g;
    cudaFuncSetAttribute(chamfer_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TC_SMEM);
    chamfer_tc_kernel<<<dim3((unsigned)g, a->NQ), TC_CTA, TC_SMEM, s>>>(ct);
    if (a->k > 0) merge_kernel<<<a->NQ, 1024, 0, s>>>(ct);
    return cuda_status("la_chamfer_topk (tensor)");
  }
  if (p.fast) {
    auto scan = [&](const ScanCtx& cc, dim3 g) -> int {
      switch (p.qs) {
#define LA_CASE(QSV)                                                                                   \
  case QSV:                                                                                            \
    cudaFuncSetAttribute(chamfer_scan_kernel<QSV>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                         (int)SCAN_SMEM);                                                             \
    chamfer_scan_kernel<QSV><<<g, CT, SCAN_SMEM, s>>>(cc);                                            \
    return 0;
        LA_CASE(1) LA_CASE(2) LA_CASE(3) LA_CASE(4) LA_CASE(5) LA_CASE(6) LA_CASE(7) LA_CASE(8)
#undef LA_CASE
        default: return fail(LA_ERANGE, "la_chamfer_topk: Q=%d", a->Q);
      }
    };
    if (p.prune) {
      unsigned char* pw = static_cast<unsigned char*>(a->ws) + align_up(p.ws_lists) + align_up(p.ws_dense);
      __half* dt = reinterpret_cast<__half*>(pw); pw += (size_t)a->NQ * LB_DT_BYTES;
      float* par = reinterpret_cast<float*>(pw); pw += (size_t)a->NQ * 8 * sizeof(float);
      unsigned* thr = reinterpret_cast<unsigned*>(pw); pw += (size_t)a->NQ * sizeof(unsigned);
      unsigned* slots = reinterpret_cast<unsigned*>(pw); pw += (size_t)a->NQ * 32 * sizeof(unsigned);
      pw = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(pw) + 15) & ~(uintptr_t)15);
      const size_t nk = (size_t)a->NQ * a->k;
      int64_t* sp = reinterpret_cast<int64_t*>(pw);  // top_id, top_pos, hit_id, hit_pos
      float* sd = reinterpret_cast<float*>(sp + 4 * nk); // top_d, hit_d
      lb_grid_kernel<<<dim3((LBV * LBV + 255) / 256, a->NQ), 256, 0, s>>>(a->queries, a->Q, dt, par);
      c.slots = slots;
      c.lb_dt = dt;
      c.lb_par = par;
      c.thr = thr;
      c.lb_slack = 4e-6f + ((a->flags & LA_CH_EXPANSION) ? a->fixup_below : 0.f);
      if (p.index) {
        // seed: the pruned scan over the prefix, only for its running bound
        // (k-th smallest of the slot minima: an upper bound of the final
        // k-th best; its lists are not needed -- the bound step looks at
        // every position again)
        const long long npos = a->pos_end - a->pos_begin;
        thr_init_kernel<<<1, 32, 0, s>>>(nullptr, a->k, a->NQ, thr, slots);
        unsigned char* iw = static_cast<unsigned char*>(a->ws) + align_up(p.ws_lists) + align_up(p.ws_dense) +
                            align_up(p.ws_prune);
        unsigned short* table = reinterpret_cast<unsigned short*>(iw); iw += align_up((size_t)IDX_TAB * 2);
        int64_t* order2 = reinterpret_cast<int64_t*>(iw); iw += align_up((size_t)npos * sizeof(long long));
        int64_t* pmap2 = reinterpret_cast<int64_t*>(iw); iw += align_up((size_t)npos * sizeof(long long));
        long long* cnt = reinterpret_cast<long long*>(iw); iw += 256;
        unsigned* qlist = reinterpret_cast<unsigned*>(iw); iw += align_up((CD_CELLS + 1) * sizeof(unsigned));
        int sms = sm_count();
        if (sms <= 0) sms = 148;
        index_table_kernel<<<dim3((IDX_TAB + 255) / 256, 1), 256, 0, s>>>(a->queries, a->Q, table);
        if (a->coarse) index_qlist_kernel<CDG><<<1, 256, 0, s>>>(a->queries, a->Q, qlist);
        // The seed prefix (1/64 of the positions) is itself scanned through
        // the bound step when it is long enough: a plain pruned scan of its
        // first 1/16 gives a first bound, the bound step over the prefix
        // lists the curves that bound leaves, and their scan leaves the
        // seed's running bound -- the same bound the plain scan of the whole
        // prefix would reach (its k-th best comes from the same curves), for
        // a fraction of the point streaming.
        const long long sn = p.seed_end - a->pos_begin;
        const long long sn0 = sn >= 65536 ? sn / 16 : sn;
        ScanCtx sc = c;
        sc.prune = 1;
        sc.a.pos_end = a->pos_begin + sn0;
        sc.a.n_hits = nullptr;
        sc.a.n_full = nullptr;
        sc.nwarps_total = p.seed_grid;
        if (int e = scan(sc, dim3(p.seed_grid, 1))) return e;
        if (sn0 < sn) {
          cudaMemsetAsync(cnt, 0, sizeof(long long), s);
          long long bs = (sn + IB_T - 1) / IB_T;
          if (bs > (long long)sms * (2048 / IB_T)) bs = (long long)sms * (2048 / IB_T);
          index_bound_kernel<<<(unsigned)bs, IB_T, 0, s>>>(a->cells, a->P, a->order, a->pos_map, a->pos_begin,
                                                           a->pos_base, sn, table, thr, a->threshold, c.lb_slack,
                                                           order2, pmap2, reinterpret_cast<unsigned long long*>(cnt),
                                                           a->coarse, qlist, a->Q);
          ScanCtx sb = sc;
          sb.a.order = order2;
          sb.a.pos_map = pmap2;
          sb.a.pos_begin = 0;
          sb.a.pos_end = sn;
          sb.pos_count = cnt;
          if (int e = scan(sb, dim3(p.seed_grid, 1))) return e;
        }
        // bound step against the seed's bound; survivors appended to (order2,
        // pos_map2), counted on the device; then the pruned scan over them
        cudaMemsetAsync(cnt, 0, 3 * sizeof(long long), s);
        long long bg = (npos + IB_T - 1) / IB_T;
        if (bg > (long long)sms * (2048 / IB_T)) bg = (long long)sms * (2048 / IB_T);
        index_bound_kernel<<<(unsigned)bg, IB_T, 0, s>>>(a->cells, a->P, a->order, a->pos_map, a->pos_begin,
                                                         a->pos_base, npos, table, thr, a->threshold, c.lb_slack,
                                                         order2, pmap2, reinterpret_cast<unsigned long long*>(cnt),
                                                         a->coarse, qlist, a->Q);
        if (a->n_stage) index_count_kernel<<<1, 1, 0, s>>>(cnt, a->n_stage);
        if (a->coarse && a->fine) {
          // second level over the survivors: the 32 x 32 tables
          int64_t* order3 = reinterpret_cast<int64_t*>(iw); iw += align_up((size_t)npos * sizeof(long long));
          int64_t* pmap3 = reinterpret_cast<int64_t*>(iw); iw += align_up((size_t)npos * sizeof(long long));
          unsigned* qw2 = reinterpret_cast<unsigned*>(iw); iw += align_up((CD2_CELLS / 4 + 1) * sizeof(unsigned));
          long long* cnt2 = cnt + 1;
          index_qlist_kernel<CD2G><<<1, 256, 0, s>>>(a->queries, a->Q, qw2);
          index_bound2_kernel<<<(unsigned)((long long)sms * (2048 / IB_T)), IB_T, 0, s>>>(
              a->cells, a->P, a->fine, cnt, order2, pmap2, table, qw2, a->Q, thr, a->threshold, c.lb_slack, order3,
              pmap3, reinterpret_cast<unsigned long long*>(cnt2), npos);
          index_close_kernel<<<sms * 2, 256, 0, s>>>(order3, pmap3, reinterpret_cast<unsigned long long*>(cnt2), npos);
          index_close_count_kernel<<<1, 1, 0, s>>>(reinterpret_cast<unsigned long long*>(cnt2));
          if (a->n_stage) index_count_kernel<<<1, 1, 0, s>>>(cnt2, a->n_stage + 1);
          order2 = order3;
          pmap2 = pmap3;
          cnt = cnt2;
        }
        c.a.order = order2;
        c.a.pos_map = pmap2;
        c.a.pos_begin = 0;
        c.a.pos_end = npos;
        c.pos_count = cnt;
        c.prune = 1;
      } else {
        // optional seed: plain scan of a prefix, merged; its k-th best starts thr
        float* seed_kth = nullptr;
        if (p.seed_end > a->pos_begin) {
          ScanCtx sc = c;
          sc.a.pos_end = p.seed_end;
          sc.a.n_hits = nullptr;
          sc.a.n_full = nullptr;
          sc.a.top_id = sp; sc.a.top_pos = sp + nk; sc.a.hit_id = sp + 2 * nk; sc.a.hit_pos = sp + 3 * nk;
          sc.a.top_d = sd; sc.a.hit_d = sd + nk;
          sc.nwarps_total = p.seed_grid;  // one list per CTA (cta_flush_lists)
          if (int e = scan(sc, dim3(p.seed_grid, a->NQ))) return e;
          merge_kernel<<<a->NQ, 1024, 0, s>>>(sc);
          seed_kth = sd;
        }
        thr_init_kernel<<<(a->NQ + 255) / 256, 256, 0, s>>>(seed_kth, a->k, a->NQ, thr, slots);
        c.prune = 1;
      }
      if (p.mq) {
        // common-grid distance tables of every query, then one launch over
        // (CTAs, query groups)
        pw = reinterpret_cast<unsigned char*>(sd + 2 * nk);
        pw = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(pw) + 255) & ~(uintptr_t)255);
        const int stride = p.mq_g0 == 64 ? MQGrid<64>::STRIDE : MQGrid<32>::STRIDE;
        __half* dt0 = reinterpret_cast<__half*>(pw); pw += (size_t)a->NQ * stride * sizeof(__half);
        __half* tab0 = reinterpret_cast<__half*>(pw); pw += (size_t)a->NQ * MQ_TAB_BYTES;
        float* par0 = reinterpret_cast<float*>(pw);
        mq_box_kernel<<<1, 1024, 0, s>>>(a->queries, (long long)a->NQ * a->Q, p.mq_g0, par0);
        const int nv = (p.mq_g0 + 1) * (p.mq_g0 + 1);
        mq_dt_kernel<<<dim3((nv + 255) / 256, a->NQ), 256, 0, s>>>(a->queries, a->Q, p.mq_g0, stride, par0, dt0);
        mq_tab_kernel<<<a->NQ, 160, 0, s>>>(a->queries, a->Q, par0, tab0);
        c.nwarps_total = p.mq_grid;  // lists per query written by the kernel (and merged)
        const dim3 g(p.mq_grid, p.mq_groups);
        auto launch_mq = [&](const ScanCtx& cc) -> int {
          cudaError_t ce = cudaSuccess;
          switch (p.qs * 100 + p.mq_g0) {
#define LA_MQ(QSV, G)                                                                                  \
  case QSV * 100 + G:                                                                                  \
    ce = cudaFuncSetAttribute(chamfer_mq_kernel<QSV, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                              (int)p.mq_smem);                                                         \
    chamfer_mq_kernel<QSV, G><<<g, MQ_T, p.mq_smem, s>>>(cc, p.mq_qg, dt0, tab0, par0);                \
    break;
            LA_MQ(1, 32) LA_MQ(2, 32) LA_MQ(3, 32) LA_MQ(4, 32) LA_MQ(5, 32) LA_MQ(6, 32) LA_MQ(7, 32) LA_MQ(8, 32)
            LA_MQ(1, 64) LA_MQ(2, 64) LA_MQ(3, 64) LA_MQ(4, 64) LA_MQ(5, 64) LA_MQ(6, 64) LA_MQ(7, 64) LA_MQ(8, 64)
#undef LA_MQ
            default: return fail(LA_ERANGE, "la_chamfer_topk: Q=%d", a->Q);
          }
          if (ce != cudaSuccess) return fail((int)ce, "la_chamfer_topk: mq smem attr: %s", cudaGetErrorString(ce));
          return 0;
        };
        if (p.index_mq) {
          // seed: the multi-query kernel over a prefix, for every query's
          // running bound; bound step for every (query, curve) on the cell
          // rows; each query's survivors with the single-query kernel
          const long long npos = a->pos_end - a->pos_begin;
          ScanCtx sc = c;
          sc.a.pos_end = p.mq_seed_end;
          sc.a.n_hits = nullptr;
          sc.a.n_full = nullptr;
          sc.a.n_stage = nullptr;
          if (int e = launch_mq(sc)) return e;
          unsigned char* iw = static_cast<unsigned char*>(a->ws) + align_up(p.ws_lists) + align_up(p.ws_dense) +
                              align_up(p.ws_prune);
          unsigned short* tables = reinterpret_cast<unsigned short*>(iw);
          iw += align_up((size_t)a->NQ * IDX_TAB * sizeof(unsigned short));
          int64_t* order2 = reinterpret_cast<int64_t*>(iw); iw += align_up((size_t)a->NQ * npos * sizeof(long long));
          int64_t* pmap2 = reinterpret_cast<int64_t*>(iw); iw += align_up((size_t)a->NQ * npos * sizeof(long long));
          long long* cnt = reinterpret_cast<long long*>(iw);
          int sms = sm_count();
          if (sms <= 0) sms = 148;
          cudaMemsetAsync(cnt, 0, (size_t)a->NQ * sizeof(long long), s);
          index_table_kernel<<<dim3((IDX_TAB + 255) / 256, a->NQ), 256, 0, s>>>(a->queries, a->Q, tables);
          cudaError_t ce = cudaFuncSetAttribute(index_bound_mq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)IBM_SMEM);
          if (ce != cudaSuccess) return fail((int)ce, "la_chamfer_topk: bound smem attr: %s", cudaGetErrorString(ce));
          const int ngroups = (a->NQ + IBM_QG - 1) / IBM_QG;
          long long bx = ((npos + 1) / 2 + IBM_T / 32 - 1) / (IBM_T / 32);
          if (bx > sms) bx = sms;
          unsigned* qwm = reinterpret_cast<unsigned*>(reinterpret_cast<unsigned char*>(cnt) + align_up((size_t)a->NQ * 8));
          if (a->coarse) index_qlist_kernel<CDG><<<a->NQ, 256, 0, s>>>(a->queries, a->Q, qwm);
          index_bound_mq_kernel<<<dim3((unsigned)bx, ngroups), IBM_T, IBM_SMEM, s>>>(
              a->cells, a->P, a->order, a->pos_map, a->pos_begin, a->pos_base, npos, a->NQ, tables, thr, a->threshold,
              c.lb_slack, npos, order2, pmap2, reinterpret_cast<unsigned long long*>(cnt), a->coarse, qwm, a->Q);
          if (a->n_stage) index_count_mq_kernel<<<1, 1, 0, s>>>(cnt, a->NQ, a->n_stage);
          ScanCtx c2 = c;
          c2.a.order = order2;
          c2.a.pos_map = pmap2;
          c2.a.pos_begin = 0;
          c2.a.pos_end = npos;
          c2.pos_count = cnt;
          c2.list_stride = npos;
          c2.nwarps_total = p.iq_grid;  // one list per CTA (cta_flush_lists)
          if (int e = scan(c2, dim3(p.iq_grid, a->NQ))) return e;
          if (a->k > 0) merge_kernel<<<a->NQ, 1024, 0, s>>>(c2);
          return cuda_status("la_chamfer_topk (indexed multi-query)");
        }
        if (int e = launch_mq(c)) return e;
        if (a->k > 0) merge_kernel<<<a->NQ, 1024, 0, s>>>(c);
        return cuda_status("la_chamfer_topk (multi-query)");
      }
    }
    if (int e = scan(c, grid)) return e;
    c.nwarps_total = p.grid;  // one list per CTA (cta_flush_lists)
  } else {
    const size_t smem = sizeof(float2) * ((size_t)a->P + a->Q);
    if (smem > 200 * 1024) return fail(LA_ERANGE, "la_chamfer_topk: P+Q too large for the generic path");
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(chamfer_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long npos = a->pos_end - a->pos_begin;
    int sms = sm_count();
    long long gx = npos < (long long)sms * 8 ? npos : (long long)sms * 8;
    if (gx < 1) gx = 1;
    chamfer_generic_kernel<<<dim3((unsigned)gx, a->NQ), 256, smem, s>>>(*a, c.dense);
    if (a->k > 0) select_kernel<<<grid, CT, 0, s>>>(c);
  }
  if (a->k > 0) merge_kernel<<<a->NQ, 1024, 0, s>>>(c);
  return cuda_status("la_chamfer_topk");
}

}  // extern "C"

#ifdef LA_TC_PROF
extern "C" int la_tc_prof_read(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, la::g_tc_prof, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(la::g_tc_prof, z, sizeof(z));
  }
  return 0;
}
#endif
