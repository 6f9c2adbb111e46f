// Farthest-pair path normalisation fused with is_circle (sm_100a).
//
// Reference semantics: linkatlas curves.py
//   _farthest_pair    curves.py:22-30  exact O(P^2) argmax of cdist, the
//                                      lexicographically smallest pair on ties
//   normalize         curves.py:45-71  rotate the pair to +x, unit diameter,
//                                      bbox centred at (0.5, 0.5), half-turn
//                                      choice by first-point angle, then y-mass
//   is_circle         curves.py:95-101 population variance of the radius about
//                                      (0.5, 0.5) strictly below 5e-4
//
// Mapping: one CTA per curve; the curve is staged in shared memory.  The
// O(P^2) search uses the circulant pairing (i, i+k mod P), k = 1..P/2, so
// every thread runs the same trip count (no triangular imbalance) and smem
// reads are consecutive across the warp.  Each thread keeps its best pair and
// the runner-up value; the CTA reduction yields the farthest pair plus the
// best competing distance, which drives the frame-stability flag.  The
// O(P) frame transform and the variance run in f64.
#include "common.cuh"
#include <climits>
#include <type_traits>

namespace la {
namespace {

constexpr int NT = 256;
constexpr int MAXP = 2048;

struct Best {
  double v1;      // best value (squared distance)
  long long k1;   // its pair key i*P + j (i < j); smaller wins ties
  double v2;      // best value among other pairs
};

__device__ __forceinline__ void consider(Best& b, double v, long long key) {
  if (v > b.v1 || (v == b.v1 && key < b.k1)) {
    b.v2 = fmax(b.v2, b.v1);
    b.v1 = v;
    b.k1 = key;
  } else {
    b.v2 = fmax(b.v2, v);
  }
}

__device__ __forceinline__ Best merge(Best a, Best b) {
  // combine two disjoint candidate sets
  Best r;
  if (b.v1 > a.v1 || (b.v1 == a.v1 && b.k1 < a.k1)) {
    r.v1 = b.v1; r.k1 = b.k1; r.v2 = fmax(b.v2, a.v1);
  } else {
    r.v1 = a.v1; r.k1 = a.k1; r.v2 = fmax(a.v2, b.v1);
  }
  return r;
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = threadIdx.x < NT / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if (threadIdx.x == 0) red[0] = s;
  }
  __syncthreads();
  return red[0];
}

// numpy's pairwise summation (the inner loop of np.add.reduce on a
// contiguous float64 run): < 8 terms sequential, <= 128 terms eight strided
// accumulators combined ((0+1)+(2+3))+((4+5)+(6+7)) plus the tail, longer
// runs split at n/2 rounded down to a multiple of 8.  Used by the circle
// variance so is_circle sees numpy's exact np.var.
template <class F>
__device__ double np_pairwise(const F& f, int lo, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = dadd(r, f(lo + i));
    return r;
  }
  if (n <= 128) {
    double a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = f(lo + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = dadd(a[j], f(lo + i + j));
    double r = dadd(dadd(dadd(a[0], a[1]), dadd(a[2], a[3])), dadd(dadd(a[4], a[5]), dadd(a[6], a[7])));
    for (; i < n; ++i) r = dadd(r, f(lo + i));
    return r;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return dadd(np_pairwise(f, lo, n2), np_pairwise(f, lo + n2, n - n2));
}

// np.var(hypot(x - .5, y - .5)) (curves.py:99-100) in numpy's summation
// order, by a whole CTA: the radii and squared deviations are computed in
// parallel into buf (P doubles of shared memory), the two pairwise sums are
// thread-serial (cheap adds).  Every thread calls it; all get the variance.
template <class G>
__device__ double np_circle_var(const G& pt, int P, double* buf, double* bc) {
  for (int k = threadIdx.x; k < P; k += blockDim.x) {
    const double2 q = pt(k);
    buf[k] = np_hypot(dsub(q.x, 0.5), dsub(q.y, 0.5));
  }
  __syncthreads();
  if (threadIdx.x == 0) bc[0] = ddiv(np_pairwise([&](int k) { return buf[k]; }, 0, P), (double)P);
  __syncthreads();
  const double mean = bc[0];
  for (int k = threadIdx.x; k < P; k += blockDim.x) {
    const double x = dsub(buf[k], mean);
    buf[k] = dmul(x, x);
  }
  __syncthreads();
  if (threadIdx.x == 0) bc[0] = ddiv(np_pairwise([&](int k) { return buf[k]; }, 0, P), (double)P);
  __syncthreads();
  const double var = bc[0];
  __syncthreads();
  return var;
}

__device__ __forceinline__ double block_min(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double s = threadIdx.x < NT / 32 ? red[threadIdx.x] : INFINITY;
    for (int o = 16; o > 0; o >>= 1) s = fmin(s, __shfl_xor_sync(FULL, s, o));
    if (threadIdx.x == 0) red[0] = s;
  }
  __syncthreads();
  return red[0];
}

template <typename Tin>
__device__ __forceinline__ double2 load_pt(const void* base, size_t idx) {
  if constexpr (sizeof(Tin) == 8) {
    const double2* p = static_cast<const double2*>(base);
    return p[idx];
  } else {
    const float2 f = static_cast<const float2*>(base)[idx];
    return make_double2(f.x, f.y);
  }
}

// Value compared in the pair search.  f64 input: cdist's squared sum
// (xi-xj)^2 + (yi-yj)^2 without FMA contraction; the square root is taken
// only for pairs within rounding of the maximum (sqrt is monotone, so the
// cdist argmax is among them; a second pass resolves pairs whose distinct
// squared sums round to the same cdist value, lexicographically as
// np.argmax does).  f32 input: the fp32 squared distance (near-ties are
// flagged unstable).
template <typename Tin, typename V2>
__device__ __forceinline__ double pair_value(const V2 pj, const V2 pi) {
  if constexpr (sizeof(Tin) == 8) {
    const double dx = dsub(pj.x, pi.x), dy = dsub(pj.y, pi.y);
    return dadd(dmul(dx, dx), dmul(dy, dy));
  } else {
    const float dx = pj.x - pi.x, dy = pj.y - pi.y;
    return (double)fmaf(dy, dy, dx * dx);
  }
}

// pair search in the input precision (Tin), everything after in f64
template <typename Tin>
__global__ void __launch_bounds__(NT) normalize_kernel(const la_norm_args p) {
  extern __shared__ __align__(16) unsigned char smraw[];
  using V2 = typename std::conditional<sizeof(Tin) == 8, double2, float2>::type;
  V2* pts = reinterpret_cast<V2*>(smraw);                                    // 2P entries (doubled)
  double2* e = reinterpret_cast<double2*>(smraw + sizeof(V2) * 2 * p.P);    // P f64 outputs
  __shared__ double red[32];
  __shared__ long long redk[32];
  __shared__ double red2[32];
  const int P = p.P;
  const int tid = threadIdx.x;

  for (long long m = blockIdx.x; m < p.M; m += gridDim.x) {
    const long long row = p.src_row ? p.src_row[m] : m;
    const Tin* src = static_cast<const Tin*>(p.paths) + (size_t)row * P * 2;
    __syncthreads();
    for (int k = tid; k < P; k += NT) {
      V2 v;
      v.x = src[2 * k];
      v.y = src[2 * k + 1];
      pts[k] = v;
      pts[k + P] = v;
    }
    __syncthreads();

    // ---- farthest pair (curves.py:22-30)
    Best b{-1.0, 0x7fffffffffffffffll, -1.0};
    const int half = P / 2;
    for (int i = tid; i < P; i += NT) {
      const V2 pi = pts[i];
      const int kmax = (P & 1) ? half : half - 1;
      for (int k = 1; k <= kmax; ++k) {
        const int j = i + k - (i + k >= P ? P : 0);
        const long long key = (i < j) ? (long long)i * P + j : (long long)j * P + i;
        consider(b, pair_value<Tin>(pts[i + k], pi), key);
      }
      if (!(P & 1) && i < half) consider(b, pair_value<Tin>(pts[i + half], pi), (long long)i * P + (i + half));
    }
    // warp then CTA reduction of (v1, k1, v2)
    for (int o = 16; o > 0; o >>= 1) {
      Best q;
      q.v1 = __shfl_xor_sync(FULL, b.v1, o);
      q.k1 = __shfl_xor_sync(FULL, b.k1, o);
      q.v2 = __shfl_xor_sync(FULL, b.v2, o);
      b = merge(b, q);
    }
    if ((tid & 31) == 0) {
      red[tid >> 5] = b.v1;
      redk[tid >> 5] = b.k1;
      red2[tid >> 5] = b.v2;
    }
    __syncthreads();
    if (tid < 32) {
      Best q{-1.0, 0x7fffffffffffffffll, -1.0};
      if (tid < NT / 32) q = Best{red[tid], redk[tid], red2[tid]};
      for (int o = 16; o > 0; o >>= 1) {
        Best r;
        r.v1 = __shfl_xor_sync(FULL, q.v1, o);
        r.k1 = __shfl_xor_sync(FULL, q.k1, o);
        r.v2 = __shfl_xor_sync(FULL, q.v2, o);
        q = merge(q, r);
      }
      if (tid == 0) {
        red[0] = q.v1;
        redk[0] = q.k1;
        red2[0] = q.v2;
      }
    }
    __syncthreads();
    const double vmax = red[0];
    long long key = redk[0];
    const double vsecond = red2[0];
    __syncthreads();
    if constexpr (sizeof(Tin) == 8) {
      // another pair within rounding of the maximum squared sum may reach
      // the same cdist value with a smaller key: compare square roots there
      const double thr = vmax - vmax * 0x1p-48;
      if (vsecond >= thr) {
        const double dmax = __dsqrt_rn(vmax);
        long long kbest = key;
        for (int i = tid; i < P; i += NT) {
          for (int j = i + 1; j < P; ++j) {
            const double v = pair_value<Tin>(pts[j], pts[i]);
            if (v >= thr && __dsqrt_rn(v) == dmax) {
              const long long k = (long long)i * P + j;
              if (k < kbest) kbest = k;
            }
          }
        }
        for (int o = 16; o > 0; o >>= 1) kbest = min(kbest, __shfl_xor_sync(FULL, kbest, o));
        if ((tid & 31) == 0) redk[tid >> 5] = kbest;
        __syncthreads();
        if (tid == 0) {
          long long kk = redk[0];
          for (int w = 1; w < NT / 32; ++w) kk = min(kk, redk[w]);
          redk[0] = kk;
        }
        __syncthreads();
        key = redk[0];
        __syncthreads();
      }
    }
    const int pi_ = (int)(key / P), pj_ = (int)(key % P);

    // exact diameter in f64 (cdist: sqrt of the summed squared differences)
    const double2 Pi = load_pt<Tin>(src, pi_), Pj = load_pt<Tin>(src, pj_);
    const double vx = dsub(Pj.x, Pi.x), vy = dsub(Pj.y, Pi.y);
    const double d = __dsqrt_rn(dadd(dmul(vx, vx), dmul(vy, vy)));
    if (!(d > 0.0) || vmax <= 0.0) {
      if (tid == 0) {
        p.status[m] = 1;
        if (p.pair) { p.pair[2 * m] = 0; p.pair[2 * m + 1] = 0; }
        if (p.diameter) p.diameter[m] = 0.0;
        if (p.unstable) p.unstable[m] = 1;
        if (p.is_circle) p.is_circle[m] = 0;
        if (p.circle_var) p.circle_var[m] = 0.0;
      }
      continue;
    }
    const double c = ddiv(vx, d), s = ddiv(vy, d);
    // base = ((P - P_i) @ rot.T) / d, rot = [[c, s], [-s, c]].  numpy hands
    // the (T,2)@(2,2) product to OpenBLAS dgemm, whose FMA kernels
    // accumulate k = 0 then k = 1: fma(w, rot[col][1], u * rot[col][0])
    // (0 mismatches in 6000 products against numpy here)
    double lox = INFINITY, loy = INFINITY, hix = -INFINITY, hiy = -INFINITY;
    for (int k = tid; k < P; k += NT) {
      const double2 q = load_pt<Tin>(src, k);
      const double u = dsub(q.x, Pi.x), w = dsub(q.y, Pi.y);
      const double bx = ddiv(__fma_rn(w, s, dmul(u, c)), d);
      const double by = ddiv(__fma_rn(w, c, dmul(u, -s)), d);
      e[k] = make_double2(bx, by);
      lox = fmin(lox, bx); hix = fmax(hix, bx);
      loy = fmin(loy, by); hiy = fmax(hiy, by);
    }
    lox = block_min(lox, red);
    loy = block_min(loy, red);
    hix = -block_min(-hix, red);
    hiy = -block_min(-hiy, red);
    if (p.bbox) {
      double ilx = INFINITY, ily = INFINITY, ihx = -INFINITY, ihy = -INFINITY;
      for (int k = tid; k < P; k += NT) {
        const double2 q = load_pt<Tin>(src, k);
        ilx = fmin(ilx, q.x); ihx = fmax(ihx, q.x);
        ily = fmin(ily, q.y); ihy = fmax(ihy, q.y);
      }
      ilx = block_min(ilx, red);
      ily = block_min(ily, red);
      ihx = -block_min(-ihx, red);
      ihy = -block_min(-ihy, red);
      if (tid == 0) {
        p.bbox[4 * m] = ilx; p.bbox[4 * m + 1] = ily;
        p.bbox[4 * m + 2] = ihx; p.bbox[4 * m + 3] = ihy;
      }
    }
    const double mx = ddiv(dadd(lox, hix), 2.0), my = ddiv(dadd(loy, hiy), 2.0);
    // e = base - mid; cand_a = e + 0.5, cand_b = (-e) + 0.5 (bbox of -base is
    // the negated bbox, so its centre is exactly -mid)
    for (int k = tid; k < P; k += NT) {
      const double2 q = e[k];
      e[k] = make_double2(dsub(q.x, mx), dsub(q.y, my));
    }
    __syncthreads();
    // half-turn choice (curves.py:63-71)
    bool use_a;
    {
      const double ax = dsub(dadd(e[0].x, 0.5), 0.5), ay = dsub(dadd(e[0].y, 0.5), 0.5);
      const double bx = dsub(dadd(-e[0].x, 0.5), 0.5), by = dsub(dadd(-e[0].y, 0.5), 0.5);
      double aa = atan2(ay, ax), ab = atan2(by, bx);
      const double two_pi = 6.283185307179586;
      if (aa < 0.0) aa = dadd(aa, two_pi);
      if (ab < 0.0) ab = dadd(ab, two_pi);
      if (fabs(dsub(aa, ab)) <= 1e-12) {
        double ma = 0.0, mb = 0.0;
        for (int k = tid; k < P; k += NT) {
          ma += fmax(dsub(dadd(e[k].y, 0.5), 0.5), 0.0);
          mb += fmax(dsub(dadd(-e[k].y, 0.5), 0.5), 0.0);
        }
        ma = block_sum(ma, red);
        mb = block_sum(mb, red);
        use_a = ma >= mb;
      } else {
        use_a = aa < ab;
      }
    }
    // write + circle statistics
    for (int k = tid; k < P; k += NT) {
      const double2 q = e[k];
      const double ox = use_a ? dadd(q.x, 0.5) : dadd(-q.x, 0.5);
      const double oy = use_a ? dadd(q.y, 0.5) : dadd(-q.y, 0.5);
      e[k] = make_double2(ox, oy);
      if (p.out_f64) {
        reinterpret_cast<double2*>(p.out)[(size_t)m * P + k] = make_double2(ox, oy);
      } else {
        reinterpret_cast<float2*>(p.out)[(size_t)m * P + k] = make_float2((float)ox, (float)oy);
      }
    }
    __syncthreads();
    double var = 0.0;
    if (p.is_circle || p.circle_var)  // pts is free after the pair search: reuse it for the radii
      var = np_circle_var([&](int k) { return e[k]; }, P, reinterpret_cast<double*>(pts), red);
    if (tid == 0) {
      p.status[m] = 0;
      if (p.pair) { p.pair[2 * m] = pi_; p.pair[2 * m + 1] = pj_; }
      if (p.diameter) p.diameter[m] = d;
      if (p.is_circle) p.is_circle[m] = var < 5e-4 ? 1 : 0;
      if (p.circle_var) p.circle_var[m] = var;
      if (p.unstable) {
        const double lim = vmax * (1.0 - p.rel_tol) * (1.0 - p.rel_tol);  // squared values
        const bool tie = vsecond > lim;
        const bool flip = fabs(dsub(e[0].y, 0.5)) < p.y_tol;
        p.unstable[m] = (tie || flip) ? 1 : 0;
      }
    }
  }
}

template <typename Tin>
__global__ void __launch_bounds__(NT) circle_kernel(const void* paths, int64_t M, int32_t P, double* var_out,
                                                    uint8_t* flag) {
  __shared__ double red[32];
  for (long long m = blockIdx.x; m < M; m += gridDim.x) {
    const Tin* src = static_cast<const Tin*>(paths) + (size_t)m * P * 2;
    extern __shared__ double cbuf[];
    const double var =
        np_circle_var([&](int k) { return make_double2((double)src[2 * k], (double)src[2 * k + 1]); }, P, cbuf, red);
    if (threadIdx.x == 0) {
      if (var_out) var_out[m] = var;
      if (flag) flag[m] = var < 5e-4 ? 1 : 0;
    }
  }
}

// ---------------------------------------------------------------------------
// fp32 batch path: one WARP per curve (P <= 256), two passes over the full
// P x P distance matrix with register blocking — each lane holds up to 8
// rows (points l, l+32, ...) packed in f32x2 pairs and every column point is
// a shared-memory broadcast, so a column costs one LDS for 8 pair distances.
//   pass 1: M = max d^2 (FMNMX3 chains, REDUX.MAX on the float bits); each
//           column's warp maximum is kept in shared memory
//   pass 2: only the columns whose maximum reaches M (1 - rel)^2: pairs
//           i < j with d^2 >= M (1 - rel)^2 -> near-max count (frame
//           stability) and the lexicographically smallest pair with d^2 == M
// then the f64 frame transform / bbox / half-turn rule / variance with warp
// shuffles only (no CTA barriers).
#ifndef LA_NW_WARPS
#define LA_NW_WARPS 8
#endif
constexpr int NW_WARPS = LA_NW_WARPS;
constexpr int NW_PMAX = 256;

__device__ __forceinline__ double warp_min_d(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// maxThreads only: ptxas then settles at 79 registers (3 CTAs per SM); an
// explicit minBlocks of 1 gives 114 (2 CTAs, 10 % slower), 3 or 4 cap it
// tighter and are slower too (measured, round 1 session 2)
#ifndef LA_NW_MINB
#define LA_NW_MINB 3  // 3 CTAs per SM: 200k curves 1.63 (no bound) / 1.53 / 1.73 (4) ms
#endif
__global__ void __launch_bounds__(NW_WARPS * 32, LA_NW_MINB) normalize_warp_kernel(const la_norm_args p) {
  __shared__ __align__(16) float2 pts[NW_WARPS][NW_PMAX];
  // (-2x', -2y', |p'|^2, m): p' centred at point 0; m = pass-1 maximum of
  // column j (and of its partner column: one reduction per column pair)
  __shared__ __align__(16) float4 cen[NW_WARPS][NW_PMAX];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int P = p.P;
  const int R2 = (P + 63) / 64;  // packed row pairs per lane (<= 4)
  for (long long m = (long long)blockIdx.x * NW_WARPS + w; m < p.M; m += (long long)gridDim.x * NW_WARPS) {
    const long long row = p.src_row ? p.src_row[m] : m;
    const float2* src = static_cast<const float2*>(p.paths) + (size_t)row * P;
    __syncwarp();
    const float2 o = src[0];
    for (int k = lane; k < P; k += 32) {
      const float2 v = src[k];
      pts[w][k] = v;
      const float x = v.x - o.x, y = v.y - o.y;
      cen[w][k] = make_float4(-2.f * x, -2.f * y, fmaf(y, y, x * x), 0.f);  // -2 p' exact
    }
    __syncwarp();
    // rows l + 64q and l + 64q + 32 packed as f32x2; padding rows duplicate
    // point 0 (cannot raise the max; masked in pass 2)
    float2 xr[4], yr[4], nr[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i0 = lane + 64 * q, i1 = i0 + 32;
      const float4 a = cen[w][(q < R2 && i0 < P) ? i0 : 0], b = cen[w][(q < R2 && i1 < P) ? i1 : 0];
      xr[q] = make_float2(-0.5f * a.x, -0.5f * b.x);  // exact
      yr[q] = make_float2(-0.5f * a.y, -0.5f * b.y);
      nr[q] = make_float2(a.z, b.z);
    }
    // d^2(i, j) = (|p_i|^2 - 2 p_i.p_j) + |p_j|^2 in the expansion form: two
    // FFMA2 per row pair, the column's |p_j|^2 added once.  Both passes use
    // the identical expression, so the pass-1 maximum is reproduced exactly.
    // Pairs i < j only: row pair q holds rows >= 64q.
    float M = -INFINITY;
    // column j needs row pairs q < ceil(j / 64): walk the columns in segments
    // with a compile-time pair count (predicated-off groups would still issue)
    // column top = max over the lane's rows; (max t) + z == max(t + z)
    // because rounding is monotonic
    auto col_top = [&](auto NQc, int j) -> float {
      constexpr int NQ = decltype(NQc)::value;
      const float4 c = cen[w][j];
      const float2 m2x = make_float2(c.x, c.x), m2y = make_float2(c.y, c.y);
      float cm = -INFINITY;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float2 t = __ffma2_rn(yr[q], m2y, __ffma2_rn(xr[q], m2x, nr[q]));
        cm = fmaxf(fmaxf(cm, t.x), t.y);
      }
      return cm + c.z;
    };
    auto pass1 = [&](auto NQc, int j0, int j1) {
      int j = j0;
#pragma unroll 1
      for (; j + 1 < j1; j += 2) {
        const float t0 = col_top(NQc, j), t1 = col_top(NQc, j + 1);
        const float tt = fmaxf(t0, t1);
        M = fmaxf(M, tt);
        const float cw = __int_as_float(__reduce_max_sync(FULL, __float_as_int(tt)));
        if (lane == 0) {
          cen[w][j].w = cw;
          cen[w][j + 1].w = cw;
        }
      }
      if (j < j1) {
        const float tt = col_top(NQc, j);
        M = fmaxf(M, tt);
        const float cw = __int_as_float(__reduce_max_sync(FULL, __float_as_int(tt)));
        if (lane == 0) cen[w][j].w = cw;
      }
    };
    pass1(std::integral_constant<int, 1>{}, 1, min(P, 65));
    if (R2 >= 2) pass1(std::integral_constant<int, 2>{}, 65, min(P, 129));
    if (R2 >= 3) pass1(std::integral_constant<int, 3>{}, 129, min(P, 193));
    if (R2 >= 4) pass1(std::integral_constant<int, 4>{}, 193, P);
    M = __int_as_float(__reduce_max_sync(FULL, __float_as_int(M)));  // M >= 0 in practice
    const float thr = (float)((double)M * (1.0 - p.rel_tol) * (1.0 - p.rel_tol));
    // pass 2: (a) the lexicographically smallest pair with d^2 == M (only
    // columns whose maximum reaches M are inspected) and (b) whether a
    // second pair lies within the near-tie band — counting stops as soon as
    // the warp has seen two (near-circles would otherwise inspect every
    // column).
    int cnt = 0, key = INT_MAX;
    bool two = false;
    // one column of pass 2 (NQ row pairs)
    auto col2 = [&](auto NQc, int j) {
      constexpr int NQ = decltype(NQc)::value;
      {
        const float4 c = cen[w][j];
        const float2 m2x = make_float2(c.x, c.x), m2y = make_float2(c.y, c.y);
        float2 tv[NQ];
        float cm = -INFINITY;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          tv[q] = __ffma2_rn(yr[q], m2y, __ffma2_rn(xr[q], m2x, nr[q]));
          cm = fmaxf(fmaxf(cm, tv[q].x), tv[q].y);
        }
        const float top = cm + c.z;
        if (top >= M) {
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const int i0 = lane + 64 * q, i1 = i0 + 32;
            if (i0 < j && i0 < P && tv[q].x + c.z == M) key = min(key, i0 * P + j);
            if (i1 < j && i1 < P && tv[q].y + c.z == M) key = min(key, i1 * P + j);
          }
        }
        const bool near = !two && top >= thr;
        if (__any_sync(FULL, near)) {
          if (near) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
              const int i0 = lane + 64 * q, i1 = i0 + 32;
              cnt += (i0 < j && i0 < P && tv[q].x + c.z >= thr) ? 1 : 0;
              cnt += (i1 < j && i1 < P && tv[q].y + c.z >= thr) ? 1 : 0;
            }
          }
          two = __reduce_add_sync(FULL, cnt) >= 2;
        }
      }
    };
    // candidate columns: warp maximum >= thr (every column holding a pair
    // with d^2 == M or in the near band), visited in ascending order
    __syncwarp();
    for (int j0 = 0; j0 < P; j0 += 32) {
      const int jl = j0 + lane;
      unsigned cand = __ballot_sync(FULL, jl >= 1 && jl < P && cen[w][jl].w >= thr);
      while (cand) {
        const int j = j0 + __ffs(cand) - 1;
        cand &= cand - 1;
        if (j < 65) col2(std::integral_constant<int, 1>{}, j);
        else if (j < 129) col2(std::integral_constant<int, 2>{}, j);
        else if (j < 193) col2(std::integral_constant<int, 3>{}, j);
        else col2(std::integral_constant<int, 4>{}, j);
      }
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
    key = __reduce_min_sync(FULL, key);
    const int pi_ = key == INT_MAX ? 0 : key / P, pj_ = key == INT_MAX ? 0 : key % P;
    // ---- f64 frame (curves.py:56-71)
    const double2 Pi = make_double2(pts[w][pi_].x, pts[w][pi_].y);
    const double2 Pj = make_double2(pts[w][pj_].x, pts[w][pj_].y);
    const double vx = Pj.x - Pi.x, vy = Pj.y - Pi.y;
    const double d = sqrt(vx * vx + vy * vy);
    if (!(d > 0.0) || !(M > 0.f)) {
      if (lane == 0) {
        p.status[m] = 1;
        if (p.pair) { p.pair[2 * m] = 0; p.pair[2 * m + 1] = 0; }
        if (p.diameter) p.diameter[m] = 0.0;
        if (p.unstable) p.unstable[m] = 1;
        if (p.is_circle) p.is_circle[m] = 0;
        if (p.circle_var) p.circle_var[m] = 0.0;
      }
      continue;
    }
    const double id = 1.0 / d;
    const double c = vx * id, sn = vy * id;
    auto base = [&](int k) -> double2 {
      const double u = (double)pts[w][k].x - Pi.x, v = (double)pts[w][k].y - Pi.y;
      return make_double2((u * c + v * sn) * id, (u * -sn + v * c) * id);
    };
    double lox = INFINITY, loy = INFINITY, hix = -INFINITY, hiy = -INFINITY;
    double ilx = INFINITY, ily = INFINITY, ihx = -INFINITY, ihy = -INFINITY;
    // frame coordinates computed once, cached in the (now free) cen storage;
    // the radii of the variance pass go to the pts storage afterwards
    double2* bc = reinterpret_cast<double2*>(&cen[w][0]);
    double* rk = reinterpret_cast<double*>(&pts[w][0]);
    __syncwarp();  // every lane is done with cen (pass 2)
    for (int k = lane; k < P; k += 32) {
      const double2 b = base(k);
      bc[k] = b;
      lox = fmin(lox, b.x); hix = fmax(hix, b.x);
      loy = fmin(loy, b.y); hiy = fmax(hiy, b.y);
      if (p.bbox) {
        ilx = fmin(ilx, (double)pts[w][k].x); ihx = fmax(ihx, (double)pts[w][k].x);
        ily = fmin(ily, (double)pts[w][k].y); ihy = fmax(ihy, (double)pts[w][k].y);
      }
    }
    lox = warp_min_d(lox); loy = warp_min_d(loy);
    hix = warp_max_d(hix); hiy = warp_max_d(hiy);
    const double mx = (lox + hix) * 0.5, my = (loy + hiy) * 0.5;
    bool use_a;
    __syncwarp();
    {
      const double2 b0 = bc[0];
      const double ex = b0.x - mx, ey = b0.y - my;
      const double ax = (ex + 0.5) - 0.5, ay = (ey + 0.5) - 0.5;
      const double bx = (-ex + 0.5) - 0.5, by = (-ey + 0.5) - 0.5;
      // clear half-planes decide without atan2: ay >= 1e-6 puts aa strictly
      // inside (0, pi) and by <= -1e-6 puts ab inside (pi, 2 pi), so
      // aa < ab and |aa - ab| > 1e-12 (and symmetrically); the first point
      // within 1e-6 of the flip line takes the reference's atan2 path
      double aa = 0.0, ab = 0.0;
      if (ay >= 1e-6 && by <= -1e-6) {
        aa = 0.0;
        ab = 4.0;
      } else if (ay <= -1e-6 && by >= 1e-6) {
        aa = 4.0;
        ab = 0.0;
      } else {
        aa = atan2(ay, ax);
        ab = atan2(by, bx);
        if (aa < 0.0) aa += 6.283185307179586;
        if (ab < 0.0) ab += 6.283185307179586;
      }
      if (fabs(aa - ab) <= 1e-12) {
        double ma = 0.0, mb = 0.0;
        for (int k = lane; k < P; k += 32) {
          const double e = bc[k].y - my;
          ma += fmax((e + 0.5) - 0.5, 0.0);
          mb += fmax((-e + 0.5) - 0.5, 0.0);
        }
        use_a = warp_sum_d(ma) >= warp_sum_d(mb);
      } else {
        use_a = aa < ab;
      }
    }
    double rsum = 0.0;
    double y0 = 0.0;
    for (int k = lane; k < P; k += 32) {
      const double2 b = bc[k];
      const double ex = b.x - mx, ey = b.y - my;
      const double ox = use_a ? ex + 0.5 : -ex + 0.5;
      const double oy = use_a ? ey + 0.5 : -ey + 0.5;
      if (k == 0) y0 = oy;
      if (p.out_f64) reinterpret_cast<double2*>(p.out)[(size_t)m * P + k] = make_double2(ox, oy);
      else reinterpret_cast<float2*>(p.out)[(size_t)m * P + k] = make_float2((float)ox, (float)oy);
      const double r = sqrt((ox - 0.5) * (ox - 0.5) + (oy - 0.5) * (oy - 0.5));
      rk[k] = r;  // pts[w][k] is not read after the first frame pass
      rsum += r;
    }
    y0 = __shfl_sync(FULL, y0, 0);
    double var = 0.0;
    if (p.is_circle || p.circle_var) {
      const double mean = warp_sum_d(rsum) / (double)P;
      double acc = 0.0;
      for (int k = lane; k < P; k += 32) {  // each lane reads back its own radii
        const double dr = rk[k] - mean;
        acc += dr * dr;
      }
      var = warp_sum_d(acc) / (double)P;
    }
    if (p.bbox) {
      ilx = warp_min_d(ilx); ily = warp_min_d(ily);
      ihx = warp_max_d(ihx); ihy = warp_max_d(ihy);
    }
    if (lane == 0) {
      p.status[m] = 0;
      if (p.pair) { p.pair[2 * m] = pi_; p.pair[2 * m + 1] = pj_; }
      if (p.diameter) p.diameter[m] = d;
      if (p.is_circle) p.is_circle[m] = var < 5e-4 ? 1 : 0;
      if (p.circle_var) p.circle_var[m] = var;
      if (p.unstable) p.unstable[m] = (cnt > 1 || fabs(y0 - 0.5) < p.y_tol) ? 1 : 0;
      if (p.bbox) {
        p.bbox[4 * m] = ilx; p.bbox[4 * m + 1] = ily;
        p.bbox[4 * m + 2] = ihx; p.bbox[4 * m + 3] = ihy;
      }
    }
  }
}

}  // namespace
}  // namespace la

using namespace la;

extern "C" int la_circle_stats(const void* paths, int32_t in_f64, int64_t M, int32_t P, double* var,
                               uint8_t* flag, void* stream) {
  if (!paths || M < 0 || P < 1 || (!var && !flag)) return fail(LA_EINVAL, "la_circle_stats: bad args");
  if (M == 0) return 0;
  const int sms = sm_count();
  long long grid = M < (long long)sms * 8 ? M : (long long)sms * 8;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t smem = sizeof(double) * (size_t)P;
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(circle_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(circle_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  if (in_f64) circle_kernel<double><<<(unsigned)grid, NT, smem, s>>>(paths, M, P, var, flag);
  else circle_kernel<float><<<(unsigned)grid, NT, smem, s>>>(paths, M, P, var, flag);
  return cuda_status("la_circle_stats");
}

extern "C" int la_normalize(const la_norm_args* a, void* stream) {
  if (!a) return fail(LA_EINVAL, "la_normalize: null args");
  if (a->M < 0 || a->P < 2) return fail(LA_EINVAL, "la_normalize: need P >= 2 (got %d)", a->P);
  if (a->P > MAXP) return fail(LA_ERANGE, "la_normalize: P=%d exceeds %d", a->P, MAXP);
  if (!a->paths || !a->out || !a->status) return fail(LA_EINVAL, "la_normalize: null buffer");
  if (a->M == 0) return 0;
  const int sms = sm_count();
  if (sms <= 0) return fail(LA_EINVAL, "la_normalize: no device");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t in_sz = a->in_f64 ? sizeof(double2) : sizeof(float2);
  const size_t smem = in_sz * 2 * a->P + sizeof(double2) * a->P;
  long long grid = a->M;
  const long long cap = (long long)sms * 8;
  if (grid > cap) grid = cap;
  if (a->in_f64) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(normalize_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    normalize_kernel<double><<<(unsigned)grid, NT, smem, s>>>(*a);
  } else if (a->P <= NW_PMAX) {
    long long g2 = (a->M + NW_WARPS - 1) / NW_WARPS;
    const long long cap2 = (long long)sms * 8;
    if (g2 > cap2) g2 = cap2;
    normalize_warp_kernel<<<(unsigned)g2, NW_WARPS * 32, 0, s>>>(*a);
  } else {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(normalize_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    normalize_kernel<float><<<(unsigned)grid, NT, smem, s>>>(*a);
  }
  return cuda_status("la_normalize");
}
