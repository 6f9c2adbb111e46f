// Batched dyad-solver replay and validity screen (sm_100a).
//
// Reference semantics: linkatlas solver.py
//   plan_geometry   solver.py:105-120 (batch form 189-201)
//   dyad_solve      solver.py:123-139
//   simulate_batch  solver.py:172-239  (first_t / first_joint rule 226-231)
//   check_feasible  solver.py:242-249 and find_valid_variant generator.py:241-283
//
// Mapping.  One warp owns one candidate (so the compiled plan, its step
// geometry and all control flow are warp-uniform); its 32 lanes evaluate 32
// crank angles at once — angles are independent (each t reads only same-t
// values, solver.py:159-165).  Joint positions of the lane's angle live in a
// per-warp shared-memory column pos[joint][lane] (dynamic joint indices
// without local-memory spills; conflict-free).
//
// Precision.  Screen angles are evaluated in fp32 with a first-order bound
// on each joint's fp32 position error, kept next to the position (input
// rounding, per-dyad rounding, amplification |x|(1+|x|/d)/h of the parents'
// error by flat dyads).  A dyad whose margin
// min(ra+rb-d, d-|ra-rb|) is within tau + 3 E(parents) of a lock makes the
// lane's angle ambiguous; ambiguous lanes below the round's first certain
// lock are replayed in f64.  f64 rounds (replays, path writes, the all-f64
// mode) come in two instantiations: EXACT mirrors numpy's operation order
// with IEEE ops and glibc's hypot (bit-identical to simulate_batch), fast
// uses DFMA and Newton-refined MUFU reciprocal square roots (a few ulp).
// Lock flags then match the f64 reference (0 mismatches on 4M 5-20 joint
// candidates against the exact mode) and coordinates stay within 1e-4 of
// the bounding-box diagonal (SURVEY.md §7 hard part (a)).
//
// Angle order.  With T % 4 == 0 the T/4 "coarse" angles t = 4i are screened
// first (they are bit-identical to the T_low = T/4 sweep of the two-fidelity
// gate, SURVEY probe P5).  A coarse lock fixes validity; the exact first
// locking angle is then searched among the fine angles below it in ascending
// order, stopping at the first 32-angle round with a lock.  Survivors sweep
// the remaining angles (screen) or all T angles in natural order writing
// coalesced float2 paths (simulate).
#include "common.cuh"
#include "sim_common.cuh"
#include <atomic>
#include <mutex>
#include <type_traits>

namespace la {
int launch_screen_lane(const la_sim_args& a, cudaStream_t s);  // screen.cu
namespace {

constexpr int NJ = LA_MAX_JOINTS;
constexpr int NS = LA_MAX_STEPS;
#ifndef LA_SIM_WARPS
#define LA_SIM_WARPS 8
#endif
constexpr int SIM_WARPS = LA_SIM_WARPS;
constexpr int SIM_THREADS = SIM_WARPS * 32;
#ifndef LA_SIM_CHUNK
#define LA_SIM_CHUNK 32  // most candidates per work chunk
#endif
#ifndef LA_SIM_TICKETS
#define LA_SIM_TICKETS 8  // chunks per warp a launch aims for
#endif
#ifndef LA_SIM_MINB
#define LA_SIM_MINB 4  // resident CTAs per SM the register allocation targets
#endif

// Per-warp shared memory: step records + initial pose, followed by a joint
// position column block pos[joint][lane] sized for the batch's largest n.
// The block is viewed as float2 (fp32 screen rounds) or double2 (f64 rounds).
struct __align__(16) StepRec {
  float sp;              // ra + rb           (fp32 margin test)
  float df;              // |ra - rb|
  float c2;              // ra^2 - rb^2
  float ra2;             // branch sign * ra^2 (|ra2| = ra^2)
  uint32_t pmask;        // 8-byte slots: fp16 error offsets of the parents (a | b << 16)
  uint32_t a_off;        // byte offset of joint a's float2 column
  uint32_t b_off;
  uint32_t t_off;
};

struct __align__(16) StepRec64 {
  uint32_t idx;          // target | a << 8 | b << 16
  uint32_t _u;
  double br;             // branch sign
  // exact mode: hi, lo, ra^2, rb^2; fast mode: hi^2, lo^2 (-1 if lo <= 0),
  // ra^2, (ra^2 - rb^2) / 2
  double hi;             // (ra + rb) + LOCK_EPS   (solver.py:213, same rounding)
  double lo;             // |ra - rb| - LOCK_EPS
  double ra2;            // ra * ra
  double rb2;            // rb * rb
};

struct __align__(16) WarpHead {
  StepRec st[NS];
  StepRec64 st64[NS];
  double2 p0[NJ];        // f64 initial pose
  int8_t tg[NS];
  int8_t nstatic;
  int8_t statics[NJ + 1];  // joints that never move (fixed + pivot)
};

struct Warp {
  WarpHead* h;
  unsigned char* cols;   // pos block: slot (joint j, lane) at (j * 32 + lane) * slot bytes
  int lane;
  int slot;              // 8 (fp32 x, y) or 16 (fp32 x, y, e, - / f64 x, y)
  int ecol_off;          // 8-byte slots: byte offset of the fp16 error array [joint][lane]
  __device__ __forceinline__ float2& p32(int j) const {
    return *reinterpret_cast<float2*>(cols + (size_t)(j * 32 + lane) * slot);
  }
  __device__ __forceinline__ double2& p64(int j) const {
    return reinterpret_cast<double2*>(cols)[j * 32 + lane];
  }
};

struct SimCtx {
  int n, ns;
  double r1;
  float tau;
  float r1f;
  float2 p0f;
};

// f64 dyad replay of one angle (solver.py:205-231).
//
// Exact mode (LA_SIM_EXACT64): numpy's operation order with IEEE
// round-to-nearest operations only (no contraction):
//   d = hypot(dx, dy)                          (glibc algorithm, np_hypot)
//   lock: d < eps | d > (ra+rb)+eps | d < |ra-rb|-eps   (LOCK_EPS 1e-9)
//   x = ((d*d + ra*ra) - rb*rb) / (2*d);  h = sqrt(max(ra*ra - x*x, 0))
//   ux = dx/d, uy = dy/d
//   p = ((pa.x + x*ux) - (br*h)*uy,  (pa.y + x*uy) + (br*h)*ux)
// so positions and lock decisions are bit-identical to simulate_batch.
// Fast mode: DFMA throughout, u = x / d and (h / d)^2 from one refined MUFU
// reciprocal of d^2, h / d from one refined reciprocal square root (a few
// ulp from numpy; the lock decision, taken on d^2 against the squared
// thresholds, can differ only for margins within ~1e-15).
template <bool EXACT, typename Get, typename Put>
__device__ __forceinline__ int dyads_f64(const WarpHead& H, const SimCtx& C, Get get, Put put,
                                         double* margin = nullptr) {
  const double eps = 1e-9;
#pragma unroll 1
  for (int s = 0; s < C.ns; ++s) {
    const StepRec64& g = H.st64[s];
    const uint4 w0 = *reinterpret_cast<const uint4*>(&g);  // idx, _, br
    const int t = w0.x & 0xff, a = (w0.x >> 8) & 0xff, b = w0.x >> 16;
    const double br = __hiloint2double((int)w0.w, (int)w0.z);
    const double2 pa = get(a), pb = get(b);
    const double2 hl = *reinterpret_cast<const double2*>(&g.hi);
    const double2 rr = *reinterpret_cast<const double2*>(&g.ra2);
    const double dx = dsub(pb.x, pa.x);
    const double dy = dsub(pb.y, pa.y);
    if (EXACT) {
      const double d = np_hypot(dx, dy);
      const bool lock = !(d >= eps) | (d > hl.x) | (d < hl.y);
      if (lock) return s;
      const double x = __ddiv_rn(dsub(dadd(dmul(d, d), rr.x), rr.y), dmul(2.0, d));
      const double h = __dsqrt_rn(fmax(dsub(rr.x, dmul(x, x)), 0.0));
      const double ux = __ddiv_rn(dx, d), uy = __ddiv_rn(dy, d);
      const double bh = dmul(br, h);
      put(t, make_double2(dsub(dadd(pa.x, dmul(x, ux)), dmul(bh, uy)),
                          dadd(dadd(pa.y, dmul(x, uy)), dmul(bh, ux))));
    } else if (margin) {
      // triage pass of the exact mode (records as in exact mode): the
      // distance of every lock test from its threshold
      const double d2 = fma(dy, dy, dx * dx);
      const double inv = rsqrt_f64(d2);
      const double d = d2 * inv;
      *margin = fmin(*margin, fmin(fabs(d - eps), fmin(fabs(hl.x - d), fabs(d - hl.y))));
      const bool lock = !(d >= eps) | (d > hl.x) | (d < hl.y);
      if (lock) return s;
      const double x = fma(d, d, rr.x - rr.y) * (0.5 * inv);
      const double h2 = fma(-x, x, rr.x);
      const double h2c = fmax(h2, 1e-300);
      const double hh = h2c * rsqrt_f64(h2c);
      const double h = h2 > 0.0 ? hh : 0.0;
      const double xi = x * inv;
      const double hb = br * h * inv;
      put(t, make_double2(fma(-hb, dy, fma(xi, dx, pa.x)), fma(hb, dx, fma(xi, dy, pa.y))));
    } else {
      // fast records: hl = (hi^2, lo^2 or -1 when lo <= 0), rr = (ra^2,
      // (ra^2 - rb^2) / 2).  With r = 1 / d^2:
      //   x / d = 1/2 + (ra^2 - rb^2) r / 2 = u,   (h / d)^2 = ra^2 r - u^2
      // so one reciprocal and one square root per dyad, and the lock tests
      // compare d^2 with the squared thresholds (same decisions up to the
      // rounding of a square, ~1e-16 relative)
      const double d2 = fma(dy, dy, dx * dx);
      const bool lock = !(d2 >= eps * eps) | (d2 > hl.x) | (d2 < hl.y);
      if (lock) return s;
      const double r = rcp_f64(d2);
      const double u = fma(rr.y, r, 0.5);
      const double w = fma(-u, u, rr.x * r);
      const double wc = fmax(w, 1e-300);
      const double vv = wc * rsqrt_f64(wc);
      const double hb = br * (w > 0.0 ? vv : 0.0);
      put(t, make_double2(fma(-hb, dy, fma(u, dx, pa.x)), fma(hb, dx, fma(u, dy, pa.y))));
    }
  }
  return -1;
}

__device__ __forceinline__ double2 crank_tip(const WarpHead& H, const SimCtx& C, double ct, double st) {
  return make_double2(dadd(H.p0[0].x, dmul(C.r1, ct)), dadd(H.p0[0].y, dmul(C.r1, st)));
}

// rare path of the fp32 screen: the whole angle again in f64, positions in
// a lane-private array; rounded results go back to the fp32 column
// Exact mode triages: a fast f64 pass first; only when one of its lock
// tests comes within kExactTriage of its threshold (fast and exact f64
// differ by a few ulp, amplified at most ~1e8-fold below that margin) is
// the angle redone in the exact arithmetic.  The lock decision is therefore
// the exact one, at fast-pass cost for almost every replay.

template <bool EXACT>
__device__ __noinline__ int replay_f64_local(const Warp& W, const SimCtx& C, double ct, double st) {
  double2 q[NJ];
  const WarpHead& H = *W.h;
#pragma unroll 1
  for (int k = 0; k < H.nstatic; ++k) {
    const int j = H.statics[k];
    q[j] = H.p0[j];
  }
  q[1] = crank_tip(H, C, ct, st);
  // only the lock decision leaves the replay: the next angle recomputes
  // every moving joint, so nothing is written back to the fp32 columns
  auto get = [&](int j) { return q[j]; };
  auto put = [&](int j, double2 v) { q[j] = v; };
  if (EXACT) {
    double margin = INFINITY;
    const int lk = dyads_f64<false>(H, C, get, put, &margin);
    if (margin > kExactTriage) return lk;
  }
  return dyads_f64<EXACT>(H, C, get, put);
}

// fp32 angle evaluation with f64 fix-up.  A lane whose dyad margin
// M = min(ra + rb - d, d - |ra - rb|) (unit-box lengths) has |M| < tau at or
// before its first lock (or is NaN) is ambiguous.  Angles increase with the
// lane index in every round, so only ambiguous lanes BELOW the round's first
// certain lock can change the round's outcome; those are replayed in f64
// (the others cannot lower the first locking angle).  Every lock decision
// that reaches the result is therefore clear of fp32 error or f64-exact.
struct Ctr {
  unsigned int fix_lanes = 0, replay_rounds = 0, lane_angles = 0, lane_dyads = 0;
};

// COUNT: maintain the diagnostic counters (la_sim_args.counters); the
// uninstrumented instantiation keeps ~10 registers free (fewer spills, 4-5 %
// faster screen)
template <bool EXACT, bool COUNT, bool ERR4>
__device__ __forceinline__ int solve32(const Warp& W, const SimCtx& C, const double* __restrict__ cs,
                                       const float2* __restrict__ cs32, int t, bool active, Ctr& ctr) {
  const WarpHead& H = *W.h;
  int lk = -1;
  bool fix = false;
  if (active) {
    const float2 c = cs32[t];
    const float tau = C.tau;
    const uint32_t col = smem_u32(W.cols) + (uint32_t)W.lane * (uint32_t)W.slot;
    sts_f2(col + 32u * (uint32_t)W.slot, make_float2(fmaf(C.r1f, c.x, C.p0f.x), fmaf(C.r1f, c.y, C.p0f.y)));
    // step records walked by shared address; the lock step is recovered
    // from the address when a lane leaves the loop
    const uint32_t rec0 = smem_u32(&H.st[0]), rec_end = rec0 + (uint32_t)C.ns * (uint32_t)sizeof(StepRec);
    uint32_t rec = rec0;
    unsigned fixw = 0u;
    if (ERR4) {
      // each joint's 16-byte slot holds its fp32 position and a first-order
      // bound e on that position's error: static joints and the crank tip
      // start at kErr0 (inputs rounded to fp32); a dyad's target gets
      //   e_t = max(kappa, 1) max(e_a, e_b) + kErrStep
      // (its parents' error amplified by the dyad, plus its own rounding)
#pragma unroll 1
      for (; rec != rec_end; rec += (uint32_t)sizeof(StepRec)) {
        const float4 g0 = lds_f4(rec);
        const uint4 g1 = lds_u4(rec + 16u);
        const float4 pa = lds_f4(col + g1.y);
        const float4 pb = lds_f4(col + g1.z);
        const float dx = pb.x - pa.x, dy = pb.y - pa.y;
        const float d2 = fmaf(dy, dy, dx * dx);
        const float inv = rsqrt_approx(d2);
        const float d = d2 * inv;
        const float m = fminf(g0.x - d, d - g0.y);
        const float ep = fmaxf(pa.z, pb.z);
        // the margin moves by at most 2 ep (d from two parents) + rounding
        flag_below(fixw, fabsf(m), fmaf(kMarginK, ep, tau));  // NaN -> f64 decides
        if (m < 0.0f) {
          lk = (int)((rec - rec0) / (uint32_t)sizeof(StepRec));
          break;
        }
        const float x = (d2 + g0.z) * (0.5f * inv);
        const float h = sqrt_approx(fmaxf(fmaf(-x, x, fabsf(g0.w)), 0.0f));
        // amplification of parent errors by an ill-conditioned (flat) dyad:
        // dh/dd = -(x/h)(1 - x/d), so |dh| <= |x| (1 + |x|/d) / h * |dd|;
        // well-conditioned dyads move their target about as far as their
        // parents moved (kappa ~ 1).  h -> 0 makes the bound infinite, so
        // every later dependent step of this angle goes to the f64 replay.
        const float ax = fabsf(x);
        const float num = ax * fmaf(ax, inv, 1.0f);
        const float e = fmaf(fmaxf(num * rcp_approx(h), 1.0f), ep, kErrStep);
        const float xi = x * inv;
        const float hb = copysignf(h, g0.w) * inv;
        // (the slot's fourth word is never read)
        sts_f4(col + g1.w,
               make_float4(fmaf(-hb, dy, fmaf(xi, dx, pa.x)), fmaf(hb, dx, fmaf(xi, dy, pa.y)), e, e));
      }
    } else {
      // large mechanisms (8-byte slots keep three CTAs per SM): the same
      // per-joint bound, stored as fp16 (rounded up; kErr0 and small bounds
      // are subnormal halves, resolution 6e-8) in
      // a [joint][lane] array after the position columns
      const uint32_t ecol = smem_u32(W.cols) + (uint32_t)W.ecol_off + (uint32_t)W.lane * 2u;
#pragma unroll 1
      for (; rec != rec_end; rec += (uint32_t)sizeof(StepRec)) {
        const float4 g0 = lds_f4(rec);
        const uint4 g1 = lds_u4(rec + 16u);
        const float2 pa = lds_f2(col + g1.y);
        const float2 pb = lds_f2(col + g1.z);
        const float dx = pb.x - pa.x, dy = pb.y - pa.y;
        const float d2 = fmaf(dy, dy, dx * dx);
        const float inv = rsqrt_approx(d2);
        const float d = d2 * inv;
        const float m = fminf(g0.x - d, d - g0.y);
        // pmask holds the parents' error offsets (a | b << 16)
        const float ep = fmaxf(lds_h16(ecol + (g1.x & 0xffffu)), lds_h16(ecol + (g1.x >> 16)));
        flag_below(fixw, fabsf(m), fmaf(kMarginK, ep, tau));  // NaN -> f64 decides
        if (m < 0.0f) {
          lk = (int)((rec - rec0) / (uint32_t)sizeof(StepRec));
          break;
        }
        const float x = (d2 + g0.z) * (0.5f * inv);
        const float h = sqrt_approx(fmaxf(fmaf(-x, x, fabsf(g0.w)), 0.0f));
        const float ax = fabsf(x);
        const float num = ax * fmaf(ax, inv, 1.0f);
        const float e = fmaf(fmaxf(num * rcp_approx(h), 1.0f), ep, kErrStep);
        const float xi = x * inv;
        const float hb = copysignf(h, g0.w) * inv;
        sts_f2(col + g1.w, make_float2(fmaf(-hb, dy, fmaf(xi, dx, pa.x)), fmaf(hb, dx, fmaf(xi, dy, pa.y))));
        sts_h16(ecol + (g1.w >> 2), e);
      }
    }
    fix = fixw != 0u;
    const int s = (int)((rec - rec0) / (uint32_t)sizeof(StepRec));
  if (COUNT) {
      ++ctr.lane_angles;
      ctr.lane_dyads += (unsigned)(s < C.ns ? s + 1 : C.ns);
    }
  }
  const unsigned certain = __ballot_sync(FULL, active && lk >= 0 && !fix);
  const unsigned below = certain ? ((1u << (__ffs(certain) - 1)) - 1u) : FULL;
  const unsigned need = __ballot_sync(FULL, active && fix) & below;
  if (need) {
    if ((need >> W.lane) & 1u) {
      lk = replay_f64_local<EXACT>(W, C, cs[2 * t], cs[2 * t + 1]);
      if (COUNT) ++ctr.fix_lanes;
    }
    if (COUNT && W.lane == 0) ++ctr.replay_rounds;
  } else if (active && fix) {
    lk = -1;  // above a certain lock: irrelevant to this round's outcome
  }
  return lk;
}

// f64 angle evaluation with positions in the warp's double2 column
template <bool EXACT>
__device__ __forceinline__ int solve64(const Warp& W, const SimCtx& C, const double* __restrict__ cs, int t,
                                       bool active) {
  if (!active) return -1;
  const WarpHead& H = *W.h;
  // 32-bit shared addresses: column j of this lane at base + j * 512
  const uint32_t base = smem_u32(W.cols) + (uint32_t)W.lane * 16u;
  sts_d2(base + 512u, crank_tip(H, C, cs[2 * t], cs[2 * t + 1]));
  return dyads_f64<EXACT>(H, C, [&](int j) { return lds_d2(base + ((uint32_t)j << 9)); },
                          [&](int j, double2 v) { sts_d2(base + ((uint32_t)j << 9), v); });
}

__device__ __forceinline__ void fill_static32(const Warp& W) {
  const WarpHead& H = *W.h;
  if (W.slot == 16) {
    float4* slot = reinterpret_cast<float4*>(W.cols) + W.lane;
#pragma unroll 1
    for (int k = 0; k < H.nstatic; ++k) {
      const int j = H.statics[k];
      slot[j * 32] = make_float4((float)H.p0[j].x, (float)H.p0[j].y, kErr0, 0.f);
    }
    slot[32] = make_float4(0.f, 0.f, kErr0, 0.f);  // crank tip: error of its inputs
  } else {
    const uint32_t ecol = smem_u32(W.cols) + (uint32_t)W.ecol_off + (uint32_t)W.lane * 2u;
#pragma unroll 1
    for (int k = 0; k < H.nstatic; ++k) {
      const int j = H.statics[k];
      W.p32(j) = make_float2((float)H.p0[j].x, (float)H.p0[j].y);
      sts_h16(ecol + 64u * j, kErr0);
    }
    sts_h16(ecol + 64u, kErr0);  // crank tip
  }
}

__device__ __forceinline__ void fill_static64(const Warp& W) {
  const WarpHead& H = *W.h;
#pragma unroll 1
  for (int k = 0; k < H.nstatic; ++k) {
    const int j = H.statics[k];
    W.p64(j) = H.p0[j];
  }
}

// first locking lane of a round -> (angle index within the round's list, step)
struct RoundLock {
  int src;
  int step;
};

__device__ __forceinline__ RoundLock round_lock(bool active, int lk) {
  const unsigned bal = __ballot_sync(FULL, active && lk >= 0);
  if (!bal) return RoundLock{-1, -1};
  const int src = __ffs(bal) - 1;
  return RoundLock{src, __shfl_sync(FULL, lk, src)};
}


// bytes per (joint, lane) slot: double2 for f64 rounds; fp32 screens use
// (x, y, e, -) with per-joint error bounds (ERR4) or (x, y) with the taint
// model (large mechanisms, where 16-byte slots would cost occupancy)
template <bool WRITE, bool SCREEN64, bool ERR4>
__host__ __device__ constexpr size_t col_bytes() {
  return (WRITE || SCREEN64 || ERR4) ? 16 : 8;
}
// per (joint, lane) bytes of the column block: slots + the fp16 error array
// of 8-byte-slot screens
template <bool WRITE, bool SCREEN64, bool ERR4>
__host__ __device__ constexpr size_t col_block_bytes() {
  return col_bytes<WRITE, SCREEN64, ERR4>() == 8 ? 10 : 16;
}

template <bool WRITE, bool SCREEN64, bool WONLY, bool EXACT, bool COUNT, bool ERR4>
__global__ void __launch_bounds__(SIM_THREADS, LA_SIM_MINB) sim_kernel(const la_sim_args p, int njmax, int chunk_items,
                                                                    unsigned* queue) {
  extern __shared__ __align__(16) unsigned char sim_smem_raw[];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int T = p.T;
  // fp32 copy of the crank table for the screen rounds (f64 stays global)
  float2* cs32 = reinterpret_cast<float2*>(sim_smem_raw);
  const size_t cs_bytes = ((size_t)T * sizeof(float2) + 15) & ~(size_t)15;
  for (int t = threadIdx.x; t < T; t += SIM_THREADS)
    cs32[t] = make_float2((float)p.crank_cs[2 * t], (float)p.crank_cs[2 * t + 1]);
  __syncthreads();
  constexpr uint32_t SLOT = (uint32_t)col_bytes<WRITE, SCREEN64, ERR4>();
  const size_t per_warp = (sizeof(WarpHead) + (size_t)njmax * 32 * col_block_bytes<WRITE, SCREEN64, ERR4>() + 15) &
                          ~(size_t)15;
  Warp W;
  W.h = reinterpret_cast<WarpHead*>(sim_smem_raw + cs_bytes + per_warp * w);
  W.cols = sim_smem_raw + cs_bytes + per_warp * w + sizeof(WarpHead);
  W.lane = lane;
  W.slot = (int)SLOT;
  W.ecol_off = njmax * 32 * (int)SLOT;
  WarpHead& H = *W.h;
  const long long nwarps = (long long)gridDim.x * SIM_WARPS;
  const bool coarse = !WONLY && !(p.flags & LA_SIM_NO_COARSE) && (T % 4 == 0) && T >= 8;
  const bool gate_only = (p.flags & LA_SIM_GATE_ONLY) != 0;
  const bool defer = !WRITE && (p.flags & LA_SIM_DEFER) != 0;
  const bool scatter = (p.flags & LA_SIM_SCATTER) != 0;
  Ctr ctr;
  unsigned long long n_angles = 0, n_dyads = 0, n_cand = 0;

  long long nitems = p.cand ? p.n_cand : p.B;
  if (p.cand_count) {
    const long long c = *p.cand_count;
    nitems = c < nitems ? c : nitems;
  }
  // Work assignment: chunks of CH consecutive candidates.  The first chunk
  // of every warp is static (chunk = global warp index); with a work queue
  // (queue != nullptr: a zeroed counter, one-wave persistent grid) every
  // further chunk is the next ticket, so warps stay busy until the batch is
  // drained whatever their candidates cost; the last warp to leave zeroes
  // the counters again.  Without a queue the chunks are dealt round-robin.
  // What depends only on the plan (step indices, column offsets, static
  // joints) is decoded once per run of candidates sharing a plan (generator
  // batches hold each topology's candidates together).
  const int CH = chunk_items;
  const unsigned nchunks = (unsigned)((nitems + CH - 1) / CH);  // la_simulate bounds the item count
  int g_cur = -1;
  bool bad_plan = false;
  uint32_t tab = 0u;  // this lane's step: target | a << 8 | b << 16
  SimCtx C;
  C.n = 0;
  C.ns = 0;
  C.tau = p.fixup_tau;
  unsigned chunk = blockIdx.x * SIM_WARPS + w;
  while (chunk < nchunks) {
  // the next ticket is taken now by lane 0 and broadcast after this chunk,
  // so the atomic's round trip runs under the chunk's work
  unsigned next = chunk + (unsigned)nwarps;
  if (queue && lane == 0) next = (unsigned)nwarps + atomicAdd(queue, 1u);
  // (la_simulate bounds the item count by 2^31)
  const unsigned item_end = min(chunk * (unsigned)CH + (unsigned)CH, (unsigned)nitems);
#pragma unroll 1
  for (unsigned item = chunk * (unsigned)CH; item < item_end; ++item) {
    const long long b = p.cand ? p.cand[item] : item;
    const int g = p.topo ? p.topo[b] : 0;
    const double* P0 = p.pos0 + (size_t)b * p.pos_stride * 2;
    __syncwarp();  // every lane is past the previous candidate
    if (lane < njmax) H.p0[lane] = make_double2(P0[2 * lane], P0[2 * lane + 1]);
    if (g != g_cur) {
      // plan-dependent state, kept across candidates of the same plan
      g_cur = g;
      const la_plan* pl = p.plans + g;
      C.n = pl->n;
      C.ns = pl->nsteps;
      const uint32_t fixed = pl->fixed_mask | 1u;  // joint 0 is static (solver.py:183)
      bad_plan = C.n > njmax || C.n < 2 || C.ns > NS || C.ns < 0;
      if (!bad_plan) {
        if (lane < C.ns) {
          const uint32_t it_ = (uint8_t)pl->step[lane][0], ia_ = (uint8_t)pl->step[lane][1],
                         ib_ = (uint8_t)pl->step[lane][2];
          tab = it_ | (ia_ << 8) | (ib_ << 16);
          H.tg[lane] = (int8_t)it_;
          H.st64[lane].idx = tab;
          // 8-byte slots: the parents' fp16 error offsets (a | b << 16); the
          // 16-byte-slot screens keep their bound inside the slot; then the
          // column offsets: slot (joint, lane) at (j * 32 + lane) * SLOT
          *reinterpret_cast<uint4*>(&H.st[lane].pmask) =
              make_uint4(SLOT == 8 ? ((uint32_t)ia_ * 64u) | ((uint32_t)ib_ * 64u << 16) : 0u,
                         (uint32_t)ia_ * 32u * SLOT, (uint32_t)ib_ * 32u * SLOT, (uint32_t)it_ * 32u * SLOT);
        }
        // static joints (1 is the crank tip even if typed Fixed)
        const bool is_static = lane < C.n && lane != 1 && ((fixed >> lane) & 1u);
        const unsigned bal = __ballot_sync(FULL, is_static);
        if (is_static) H.statics[__popc(bal & ((1u << lane) - 1u))] = (int8_t)lane;
        if (lane == 0) H.nstatic = (int8_t)__popc(bal);
      }
    }
    __syncwarp();
    if (bad_plan) {
      // plan does not fit the launch (n > pos_stride): flag only
      if (lane == 0) {
        if (p.first_t) p.first_t[item] = -1;
        if (p.first_joint) p.first_joint[item] = -2;
      }
      continue;
    }
    if (lane < C.ns) {
      // plan_geometry (solver.py:105-120), f64
      const double2 pa = H.p0[(tab >> 8) & 0xffu], pb = H.p0[tab >> 16], pt = H.p0[tab & 0xffu];
      const double ax = dsub(pt.x, pa.x), ay = dsub(pt.y, pa.y);
      const double bx = dsub(pt.x, pb.x), by = dsub(pt.y, pb.y);
      // np.hypot bit for bit (glibc algorithm, common.cuh) in exact mode;
      // otherwise a Newton-refined sqrt of the sum (an ulp or two)
      double ra, rb;
      if (EXACT) {
        ra = np_hypot(ax, ay);
        rb = np_hypot(bx, by);
      } else {
        const double a2 = dadd(dmul(ax, ax), dmul(ay, ay)), b2 = dadd(dmul(bx, bx), dmul(by, by));
        ra = a2 > 0.0 ? dmul(a2, rsqrt_f64(a2)) : 0.0;
        rb = b2 > 0.0 ? dmul(b2, rsqrt_f64(b2)) : 0.0;
      }
      const double cross = dsub(dmul(dsub(pb.x, pa.x), dsub(pt.y, pa.y)),
                                dmul(dsub(pb.y, pa.y), dsub(pt.x, pa.x)));
      const double br = cross >= 0.0 ? 1.0 : -1.0;
      StepRec64& r64 = H.st64[lane];  // idx stays (plan-dependent)
      r64.br = br;
      const double hi = dadd(dadd(ra, rb), 1e-9), lo = dsub(fabs(dsub(ra, rb)), 1e-9);
      if (EXACT) {
        *reinterpret_cast<double2*>(&r64.hi) = make_double2(hi, lo);
        *reinterpret_cast<double2*>(&r64.ra2) = make_double2(dmul(ra, ra), dmul(rb, rb));
      } else {
        // fast records (dyads_f64): squared thresholds, ra^2 and (ra^2 - rb^2) / 2
        *reinterpret_cast<double2*>(&r64.hi) = make_double2(hi * hi, lo > 0.0 ? lo * lo : -1.0);
        *reinterpret_cast<double2*>(&r64.ra2) = make_double2(ra * ra, 0.5 * (ra * ra - rb * rb));
      }
      *reinterpret_cast<float4*>(&H.st[lane].sp) =
          make_float4((float)(ra + rb), (float)fabs(ra - rb), (float)(ra * ra - rb * rb),
                      br < 0.0 ? -((float)ra * (float)ra) : (float)ra * (float)ra);
    }
    {
      // crank radius as np.hypot wherever paths are written or f64 is exact
      // (solver.py:180): with the host's crank table the crank tip row is
      // then rebuilt bit for bit; fp32 screens take a Newton-refined root
      const double dx = dsub(H.p0[1].x, H.p0[0].x), dy = dsub(H.p0[1].y, H.p0[0].y);
      if (EXACT || WRITE) {
        C.r1 = np_hypot(dx, dy);
      } else {
        const double r2 = dadd(dmul(dx, dx), dmul(dy, dy));
        C.r1 = r2 > 0.0 ? dmul(r2, rsqrt_f64(r2)) : 0.0;
      }
      C.r1f = (float)C.r1;
      C.p0f = make_float2((float)H.p0[0].x, (float)H.p0[0].y);
    }
    __syncwarp();
    if (SCREEN64 || WONLY) fill_static64(W);
    else fill_static32(W);
    __syncwarp();

    auto screen = [&](int t, bool act) -> int {
      if (SCREEN64 || WONLY) return solve64<EXACT>(W, C, p.crank_cs, t, act);
      return solve32<EXACT, COUNT, ERR4>(W, C, p.crank_cs, cs32, t, act, ctr);
    };

    int first_t = T, first_j = -1, low_t = -1, low_j = -1;
    bool locked = false;
    int rounds = 0;
    if (coarse) {
      const int Tc = T / 4;
#pragma unroll 1
      for (int r = 0; r * 32 < Tc; ++r) {
        const int i = r * 32 + lane;
        const bool act = i < Tc;
        const int lk = screen(4 * i, act);
        ++rounds;
        const RoundLock L = round_lock(act, lk);
        if (L.src >= 0) {
          low_t = r * 32 + L.src;
          low_j = H.tg[L.step];
          locked = true;
          break;
        }
      }
      if (locked) {
        first_t = 4 * low_t;
        first_j = low_j;
        if (!gate_only) {
          // exact first lock: fine angles below the coarse lock, ascending
          const int nf = 3 * low_t;
#pragma unroll 1
          for (int r = 0; r * 32 < nf; ++r) {
            const int i = r * 32 + lane;
            const bool act = i < nf;
            const int lk = screen(fine_angle(i), act);
            ++rounds;
            const RoundLock L = round_lock(act, lk);
            if (L.src >= 0) {
              first_t = fine_angle(r * 32 + L.src);
              first_j = H.tg[L.step];
              break;
            }
          }
        }
      }
    }
    if (!locked && defer) {
      first_t = LA_PENDING;  // coarse survivor: decided by a later f64 pass
      first_j = -1;
    } else if (!locked) {
      if (WRITE) {
        // all T angles in natural order, f64, coalesced float2 stores
        if (!SCREEN64 && !WONLY) {
          __syncwarp();
          fill_static64(W);
        }
        const long long row = p.traj_row ? p.traj_row[item] : item * (long long)p.traj_stride;
        const bool out64 = (p.flags & LA_SIM_TRAJ_F64) != 0;
        float2* out = reinterpret_cast<float2*>(p.traj) + (size_t)row * T;
        double2* out_d = reinterpret_cast<double2*>(p.traj) + (size_t)row * T;
        // split rows (traj2): dyad targets to traj, the static joints and the
        // crank tip (closed-form in the inputs, solver.py:183-187) to traj2,
        // each in ascending joint order
        const bool split = p.traj2 != nullptr;
        uint32_t tmask = 0u;
        float2* out2 = nullptr;
        if (split) {
#pragma unroll 1
          for (int s = 0; s < C.ns; ++s) tmask |= 1u << H.tg[s];
          out2 = reinterpret_cast<float2*>(p.traj2) + (size_t)p.traj_row2[item] * T;
        }
#pragma unroll 1
        for (int r = 0; r * 32 < T; ++r) {
          const int t = r * 32 + lane;
          const bool act = t < T;
          const int lk = solve64<EXACT>(W, C, p.crank_cs, t, act);
          ++rounds;
          const RoundLock L = round_lock(act, lk);
          if (L.src >= 0) {
            first_t = r * 32 + L.src;
            first_j = H.tg[L.step];
            break;
          }
          if (act) {
            // row j of this candidate at out + j * T: one pointer step per
            // joint, columns read by 32-bit shared address
            uint32_t a = smem_u32(W.cols) + (uint32_t)lane * 16u;
            if (out64) {
              double2* o = out_d + t;
#pragma unroll 1
              for (int j = 0; j < C.n; ++j, a += 512u, o += T) __stcs(o, lds_d2(a));
            } else if (split) {
              float2* o = out + t;
              float2* o2 = out2 + t;
#pragma unroll 1
              for (int j = 0; j < C.n; ++j, a += 512u) {
                const double2 v = lds_d2(a);
                const bool tj = (tmask >> j) & 1u;
                st_cs(tj ? o : o2, make_float2((float)v.x, (float)v.y));
                if (tj) o += T;
                else o2 += T;
              }
            } else {
              float2* o = out + t;
#pragma unroll 2
              for (int j = 0; j < C.n; ++j, a += 512u, o += T) {
                const double2 v = lds_d2(a);
                st_cs(o, make_float2((float)v.x, (float)v.y));
              }
            }
          }
        }
      } else {
        const int nf = coarse ? 3 * (T / 4) : T;
#pragma unroll 1
        for (int r = 0; r * 32 < nf; ++r) {
          const int i = r * 32 + lane;
          const bool act = i < nf;
          const int t = coarse ? fine_angle(i) : i;
          const int lk = screen(t, act);
          ++rounds;
          const RoundLock L = round_lock(act, lk);
          if (L.src >= 0) {
            const int is = r * 32 + L.src;
            first_t = coarse ? fine_angle(is) : is;
            first_j = H.tg[L.step];
            break;
          }
        }
      }
    }
    if (lane == 0) {
      const long long o = scatter && p.cand ? p.cand[item] : item;
      if (p.first_t) p.first_t[o] = first_t;
      if (p.first_joint) p.first_joint[o] = first_j;
      if (p.low_t) p.low_t[o] = low_t;
      if (p.low_joint) p.low_joint[o] = low_j;
    }
    if (COUNT) {
      n_angles += 32ull * rounds;
      n_dyads += 32ull * rounds * (unsigned long long)C.ns;
      ++n_cand;
    }
  }
  chunk = queue ? __shfl_sync(FULL, next, 0) : next;
  }
  if (queue && lane == 0) {
    // leave the counters zeroed for the next launch that gets this slot
    __threadfence();
    if (atomicAdd(queue + 1, 1u) == (unsigned)nwarps - 1u) {
      queue[0] = 0u;
      queue[1] = 0u;
    }
  }
  if (COUNT && p.counters) {
    unsigned long long f = ctr.fix_lanes, la = ctr.lane_angles, ld = ctr.lane_dyads;
    const unsigned long long rr = ctr.replay_rounds;
    for (int o = 16; o > 0; o >>= 1) {
      f += __shfl_xor_sync(FULL, f, o);
      la += __shfl_xor_sync(FULL, la, o);
      ld += __shfl_xor_sync(FULL, ld, o);
    }
    if (lane == 0) {
      atomicAdd(p.counters + 0, f);
      atomicAdd(p.counters + 1, n_angles);
      atomicAdd(p.counters + 2, n_dyads);
      atomicAdd(p.counters + 3, n_cand);
      atomicAdd(p.counters + 4, rr);
      atomicAdd(p.counters + 5, la);
      atomicAdd(p.counters + 6, ld);
    }
  }
}

__global__ void geometry_kernel(const double* __restrict__ pos0, const int32_t* __restrict__ topo,
                                const la_plan* __restrict__ plans, int64_t B, int32_t pos_stride,
                                double* r_a, double* r_b, double* branch) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * NS) return;
  const long long b = i / NS;
  const int s = (int)(i % NS);
  const la_plan* pl = plans + (topo ? topo[b] : 0);
  double ra = 0.0, rb = 0.0, br = 0.0;
  if (s < pl->nsteps) {
    const double* P = pos0 + (size_t)b * pos_stride * 2;
    const int t = pl->step[s][0], a = pl->step[s][1], c = pl->step[s][2];
    const double ax = P[2 * a], ay = P[2 * a + 1], bx = P[2 * c], by = P[2 * c + 1];
    const double tx = P[2 * t], ty = P[2 * t + 1];
    ra = np_hypot(dsub(tx, ax), dsub(ty, ay));
    rb = np_hypot(dsub(tx, bx), dsub(ty, by));
    const double cross = dsub(dmul(dsub(bx, ax), dsub(ty, ay)), dmul(dsub(by, ay), dsub(tx, ax)));
    br = cross >= 0.0 ? 1.0 : -1.0;
  }
  r_a[i] = ra;
  r_b[i] = rb;
  branch[i] = br;
}

__global__ void dyad_kernel(const double* __restrict__ pa, const double* __restrict__ pb,
                            const double* __restrict__ ra_, const double* __restrict__ rb_,
                            const double* __restrict__ br_, int64_t n, double* out, int32_t* ok) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double dx = dsub(pb[2 * i], pa[2 * i]);
  const double dy = dsub(pb[2 * i + 1], pa[2 * i + 1]);
  const double d = np_hypot(dx, dy);
  const double ra = ra_[i], rb = rb_[i];
  const double eps = 1e-9;
  if (d < eps || d > dadd(dadd(ra, rb), eps) || d < dsub(fabs(dsub(ra, rb)), eps)) {
    ok[i] = 0;
    out[2 * i] = __longlong_as_double(0x7ff8000000000000ll);
    out[2 * i + 1] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  const double x = ddiv(dsub(dadd(dmul(d, d), dmul(ra, ra)), dmul(rb, rb)), dmul(2.0, d));
  const double h = __dsqrt_rn(fmax(dsub(dmul(ra, ra), dmul(x, x)), 0.0));
  const double ux = ddiv(dx, d), uy = ddiv(dy, d);
  const double bh = dmul(br_[i], h);
  // dyad_solve (solver.py:139): p_a + x*u - branch*h*u_perp, evaluated as
  // (pa + x*ux) - (branch*h)*uy  /  (pa + x*uy) + (branch*h)*ux
  out[2 * i] = dsub(dadd(pa[2 * i], dmul(x, ux)), dmul(bh, uy));
  out[2 * i + 1] = dadd(dadd(pa[2 * i + 1], dmul(x, uy)), dmul(bh, ux));
  ok[i] = 1;
}

// ---------------------------------------------------------------- compaction
constexpr int CP_THREADS = 1024;  // one tile = 1024 candidates

// ---- compaction with dense row offsets: selected item i (first_t == T)
// gets idx = i and row_off = sum of its predecessors' joint counts, so a
// write pass with traj_row = row_off stores paths without padding rows
__device__ __forceinline__ int item_rows(const int32_t* topo, const la_plan* plans, long long i) {
  return plans[topo ? topo[i] : 0].n;
}
// split rows: dyad targets (nsteps rows) / the other joints (static + crank)
__device__ __forceinline__ int2 item_rows2(const int32_t* topo, const la_plan* plans, long long i) {
  const la_plan& p = plans[topo ? topo[i] : 0];
  return make_int2(p.nsteps, p.n - p.nsteps);
}

// ---- single-pass ordered selection (decoupled look-back).  Tile t of
// CP_THREADS consecutive items is taken in ticket order (so every
// predecessor tile is held by a running CTA); its selected count and row
// sums are block-scanned, published as an aggregate, and the tile's
// exclusive prefix is gathered from its predecessors' published values --
// aggregates, back to the nearest inclusive prefix -- by one warp, 32 tiles
// per step.  One launch replaces count + single-CTA scan + scatter.
//   MODE 0: ids only; 1: rows = plan n; 2: rows = plan nsteps (dyad
//   targets), rows2 = n - nsteps (static joints + crank tip)
// Tile word: flag (2 bits: 0 empty, 1 aggregate, 2 inclusive) | count (31)
// | rows (31); rows2 lives in agg2 / inc2, written before the word.
constexpr unsigned long long LB_AGG = 1ull << 62, LB_INC = 2ull << 62;

template <int MODE>
__global__ void __launch_bounds__(CP_THREADS) select_kernel(const int32_t* __restrict__ first_t, int64_t B,
                                                            int32_t value, const int32_t* __restrict__ topo,
                                                            const la_plan* __restrict__ plans,
                                                            unsigned long long* st, long long* agg2, long long* inc2,
                                                            unsigned* ticket, long long ntiles, int64_t* idx,
                                                            int64_t* row, int64_t* row2, int64_t* count,
                                                            int64_t* total, int64_t* total2) {
  __shared__ unsigned s_tile;
  __shared__ int wc[CP_THREADS / 32], wr[CP_THREADS / 32], wr2[CP_THREADS / 32];
  __shared__ long long s_ex[3];
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const long long tile = s_tile;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long i = tile * CP_THREADS + threadIdx.x;
  const bool v = i < B && first_t[i] == value;
  int r = 0, r2 = 0;
  if (v && MODE == 1) r = item_rows(topo, plans, i);
  if (v && MODE == 2) {
    const int2 q = item_rows2(topo, plans, i);
    r = q.x;
    r2 = q.y;
  }
  const unsigned bal = __ballot_sync(FULL, v);
  int x = r, x2 = r2;  // inclusive warp scans of the row counts
  if (MODE > 0) {
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, x, o), y2 = __shfl_up_sync(FULL, x2, o);
      if (lane >= o) {
        x += y;
        x2 += y2;
      }
    }
  }
  if (lane == 31) {
    wc[w] = __popc(bal);
    wr[w] = x;
    wr2[w] = x2;
  }
  __syncthreads();
  if (w == 0) {
    // exclusive scan of the warp totals, tile totals in lane 31
    const int c = wc[lane], sr = wr[lane], sr2 = wr2[lane];
    int xc = c, xs = sr, xs2 = sr2;
    for (int o = 1; o < 32; o <<= 1) {
      const int yc = __shfl_up_sync(FULL, xc, o), ys = __shfl_up_sync(FULL, xs, o),
                ys2 = __shfl_up_sync(FULL, xs2, o);
      if (lane >= o) {
        xc += yc;
        xs += ys;
        xs2 += ys2;
      }
    }
    wc[lane] = xc - c;
    wr[lane] = xs - sr;
    wr2[lane] = xs2 - sr2;
    const long long tc = __shfl_sync(FULL, xc, 31), tr = __shfl_sync(FULL, xs, 31), tr2 = __shfl_sync(FULL, xs2, 31);
    if (lane == 0) {
      agg2[tile] = tr2;
      __threadfence();
      atomicExch(st + tile, LB_AGG | ((unsigned long long)tc << 31) | (unsigned long long)tr);
    }
    // look-back
    long long ec = 0, er = 0, er2 = 0;
    for (long long j = tile - 1; j >= 0;) {
      const long long k = j - lane;
      unsigned long long wv = LB_INC;  // k < 0: an inclusive zero
      if (k >= 0) wv = *reinterpret_cast<volatile unsigned long long*>(st + k);
      const unsigned long long flag = wv & (3ull << 62);
      const unsigned inc = __ballot_sync(FULL, flag == LB_INC);
      const int lim = inc ? __ffs(inc) - 1 : 31;  // lanes 0..lim are needed
      const unsigned need = lim == 31 ? FULL : ((2u << lim) - 1u);
      if (__ballot_sync(FULL, flag == 0ull) & need) continue;  // a predecessor has not published yet
      long long c = 0, rr = 0, rr2 = 0;
      if (lane <= lim && k >= 0) {
        c = (long long)((wv >> 31) & 0x7fffffffull);
        rr = (long long)(wv & 0x7fffffffull);
        __threadfence();
        rr2 = flag == LB_INC ? *reinterpret_cast<volatile long long*>(inc2 + k)
                             : *reinterpret_cast<volatile long long*>(agg2 + k);
      }
      for (int o = 16; o > 0; o >>= 1) {
        c += __shfl_xor_sync(FULL, c, o);
        rr += __shfl_xor_sync(FULL, rr, o);
        rr2 += __shfl_xor_sync(FULL, rr2, o);
      }
      ec += c;
      er += rr;
      er2 += rr2;
      if (inc) break;
      j -= 32;
    }
    if (lane == 0) {
      inc2[tile] = er2 + tr2;
      __threadfence();
      atomicExch(st + tile, LB_INC | ((unsigned long long)(ec + tc) << 31) | (unsigned long long)(er + tr));
      s_ex[0] = ec;
      s_ex[1] = er;
      s_ex[2] = er2;
      if (tile == ntiles - 1) {
        *count = ec + tc;
        if (total) *total = er + tr;
        if (total2) *total2 = er2 + tr2;
      }
    }
  }
  __syncthreads();
  if (v) {
    const long long pos = s_ex[0] + wc[w] + __popc(bal & ((1u << lane) - 1u));
    idx[pos] = i;
    if (MODE > 0) row[pos] = s_ex[1] + wr[w] + (x - r);
    if (MODE == 2) row2[pos] = s_ex[2] + wr2[w] + (x2 - r2);
  }
}

}  // namespace
}  // namespace la

using namespace la;

// Work-queue counters of la_simulate's persistent launches: per device one
// zeroed array of (ticket, done) pairs.  A launch takes the next pair of a
// ring (its kernel leaves the pair zeroed, and the ring is far longer than
// any number of launches in flight); a launch recorded into a CUDA graph
// takes a pair of its own that is never handed out again (a graph may be
// replayed at any time); when those run out, or the array cannot be
// allocated, the launch falls back to the static round-robin schedule.
namespace {
constexpr unsigned Q_RING = 1u << 15, Q_CAPTURED = 1u << 15;
struct QueuePool {
  std::atomic<unsigned*> base{nullptr};
  std::atomic<unsigned> ring{0}, captured{0};
};
unsigned* take_queue(cudaStream_t s) {
  static QueuePool pools[64];
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  QueuePool& P = pools[dev];
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  unsigned* base = P.base.load(std::memory_order_acquire);
  if (!base) {
    if (cap != cudaStreamCaptureStatusNone) return nullptr;  // no allocation while a graph is being recorded
    std::lock_guard<std::mutex> lock(mu);
    base = P.base.load(std::memory_order_acquire);
    if (!base) {
      const size_t bytes = (size_t)(Q_RING + Q_CAPTURED) * 2 * sizeof(unsigned);
      if (cudaMalloc(&base, bytes) != cudaSuccess || cudaMemset(base, 0, bytes) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
      }
      P.base.store(base, std::memory_order_release);
    }
  }
  if (cap != cudaStreamCaptureStatusNone) {
    const unsigned c = P.captured.fetch_add(1, std::memory_order_relaxed);
    return c < Q_CAPTURED ? base + 2 * (size_t)(Q_RING + c) : nullptr;
  }
  return base + 2 * (size_t)(P.ring.fetch_add(1, std::memory_order_relaxed) % Q_RING);
}
}  // namespace

extern "C" {

int la_simulate(const la_sim_args* a, void* stream) {
  if (!a) return fail(LA_EINVAL, "la_simulate: null args");
  if (a->B < 0 || a->G < 1 || a->T < 1 || a->T > 1000000)
    return fail(LA_EINVAL, "la_simulate: bad sizes B=%lld G=%d T=%d", (long long)a->B, a->G, a->T);
  if (a->pos_stride < 2 || a->pos_stride > 4096) return fail(LA_EINVAL, "la_simulate: bad pos_stride");
  if (!a->pos0 || !a->plans || !a->crank_cs) return fail(LA_EINVAL, "la_simulate: null buffer");
  if (!a->cand && (!a->first_t || !a->first_joint)) return fail(LA_EINVAL, "la_simulate: null outputs");
  if (a->cand_count && !a->cand) return fail(LA_EINVAL, "la_simulate: cand_count without cand");
  if (a->cand && a->n_cand < 0) return fail(LA_EINVAL, "la_simulate: bad n_cand");
  const bool write = (a->flags & LA_SIM_WRITE_TRAJ) != 0;
  if (write && !a->traj) return fail(LA_EINVAL, "la_simulate: WRITE_TRAJ without traj");
  const long long items = a->cand ? a->n_cand : a->B;
  if (a->B == 0 || items == 0) return 0;
  if (items >= (1ll << 31)) return fail(LA_ERANGE, "la_simulate: more than 2^31 candidates in one launch");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool f64 = (a->flags & LA_SIM_FP64) != 0;
  const int njmax = a->pos_stride < NJ ? a->pos_stride : NJ;
  if (a->T > 2048) return fail(LA_ERANGE, "la_simulate: T=%d beyond 2048", a->T);
  // fp32 screens of small mechanisms keep a per-joint error bound in
  // 16-byte slots; from 13 joints on the 8-byte taint-model slots keep three
  // CTAs per SM resident (measured C3, 20 joints: 19.4 vs 21.8 ms)
  const bool err4 = njmax <= 12;
  const size_t colb = (write || f64 || err4) ? 16 : 10;  // 8-byte slots + fp16 error
  static_assert(col_block_bytes<false, false, false>() == 10 && col_block_bytes<true, false, true>() == 16,
                "launch and kernel column layouts");
  if ((a->flags & LA_SIM_SCATTER) && !a->cand) return fail(LA_EINVAL, "la_simulate: SCATTER needs cand");
  const size_t cs_bytes = ((size_t)a->T * sizeof(float2) + 15) & ~(size_t)15;
  const size_t smem = cs_bytes + ((sizeof(WarpHead) + (size_t)njmax * 32 * colb + 15) & ~(size_t)15) * SIM_WARPS;
  const bool wonly = (a->flags & LA_SIM_WRITE_ONLY) != 0;
  if (wonly && !write) return fail(LA_EINVAL, "la_simulate: WRITE_ONLY needs WRITE_TRAJ");
  const bool exact = (a->flags & LA_SIM_EXACT64) != 0;
  if (!write && !f64 && (a->flags & LA_SIM_LANE_SCREEN)) return launch_screen_lane(*a, s);
  using KernT = void (*)(const la_sim_args, int, int, unsigned*);
  auto pick = [&](auto cnt) -> KernT {
    constexpr bool C = decltype(cnt)::value;
    // ERR4 only matters where the fp32 screen runs (not WONLY / FP64)
    if (exact) {
      if (wonly) return sim_kernel<true, false, true, true, C, false>;
      if (f64) return write ? sim_kernel<true, true, false, true, C, false> : sim_kernel<false, true, false, true, C, false>;
      if (write) return sim_kernel<true, false, false, true, C, true>;  // 16-byte slots: room for e
      return err4 ? sim_kernel<false, false, false, true, C, true> : sim_kernel<false, false, false, true, C, false>;
    }
    if (wonly) return sim_kernel<true, false, true, false, C, false>;
    if (f64) return write ? sim_kernel<true, true, false, false, C, false> : sim_kernel<false, true, false, false, C, false>;
    if (write) return sim_kernel<true, false, false, false, C, true>;
    return err4 ? sim_kernel<false, false, false, false, C, true> : sim_kernel<false, false, false, false, C, false>;
  };
  const KernT kern = a->counters ? pick(std::true_type{}) : pick(std::false_type{});
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return fail((int)e, "la_simulate: smem attr: %s", cudaGetErrorString(e));
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, SIM_THREADS, smem);
  if (e != cudaSuccess) return fail((int)e, "la_simulate: occupancy: %s", cudaGetErrorString(e));
  const int sms = sm_count();
  if (sms <= 0) return fail(LA_EINVAL, "la_simulate: no device");
  // Persistent one-wave grid fed by a work queue (tickets of CH candidates:
  // candidates differ widely in cost -- early lock vs all T angles -- and
  // the queue keeps every warp busy until the batch is drained).  A ticket
  // covers more candidates in larger batches (about LA_SIM_TICKETS tickets
  // per resident warp), so consecutive candidates share their plan's decode
  // and the ticket counter stays cold.  Without a queue: four waves of resident CTAs, chunks dealt
  // round-robin (measured 1/2/4/8/16 waves: C2 step 0.310 / 0.298 / 0.290 /
  // 0.298 / 0.310 ms).
#ifdef LA_SIM_FORCE_STATIC
  unsigned* queue = nullptr;
#else
  // (the write-only pass keeps the round-robin deal: its candidates cost
  // about the same, measured 0.123 ms static vs 0.127 ms queued on C2)
  unsigned* queue = ((a->flags & LA_SIM_STATIC_GRID) || wonly) ? nullptr : take_queue(s);
#endif
  const long long resident = (long long)sms * (occ > 0 ? occ : 1);
  long long per = items / (resident * SIM_WARPS * LA_SIM_TICKETS);
  const int chunk = (per < 1 || wonly) ? 1 : per > LA_SIM_CHUNK ? LA_SIM_CHUNK : (int)per;
  const long long want = ((items + chunk - 1) / chunk + SIM_WARPS - 1) / SIM_WARPS;
  long long grid = queue ? resident : resident * 4;
  if (grid > want) grid = want;
  const la_sim_args p = *a;
  kern<<<(unsigned)grid, SIM_THREADS, smem, s>>>(p, njmax, chunk, queue);
  return cuda_status("la_simulate");
}

int la_plan_geometry(const double* pos0, const int32_t* topo, const la_plan* plans, int64_t B,
                     int32_t G, int32_t pos_stride, double* r_a, double* r_b, double* branch,
                     void* stream) {
  if (B < 0 || G < 1 || !pos0 || !plans || !r_a || !r_b || !branch)
    return fail(LA_EINVAL, "la_plan_geometry: bad args");
  if (B == 0) return 0;
  const long long n = B * NS;
  geometry_kernel<<<(unsigned)((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      pos0, topo, plans, B, pos_stride, r_a, r_b, branch);
  return cuda_status("la_plan_geometry");
}

int la_dyad_solve(const double* pa, const double* pb, const double* r_a, const double* r_b,
                  const double* branch, int64_t n, double* out, int32_t* ok, void* stream) {
  if (n < 0 || !pa || !pb || !r_a || !r_b || !branch || !out || !ok)
    return fail(LA_EINVAL, "la_dyad_solve: bad args");
  if (n == 0) return 0;
  dyad_kernel<<<(unsigned)((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      pa, pb, r_a, r_b, branch, n, out, ok);
  return cuda_status("la_dyad_solve");
}

// look-back selection workspace: a ticket, then per tile the published
// word and the aggregate / inclusive rows2 (zeroed by a memset per call)
static size_t select_ws(int64_t B) {
  const long long tiles = (B + CP_THREADS - 1) / CP_THREADS;
  return 16 + (size_t)(tiles > 0 ? tiles : 1) * 3 * sizeof(long long);
}

static int select_launch(int mode, const int32_t* first_t, int64_t B, int32_t value, const int32_t* topo,
                         const la_plan* plans, int64_t* idx, int64_t* row, int64_t* row2, int64_t* count,
                         int64_t* total, int64_t* total2, void* ws, cudaStream_t s) {
  const long long tiles = (B + CP_THREADS - 1) / CP_THREADS;
  unsigned char* w = static_cast<unsigned char*>(ws);
  unsigned* ticket = reinterpret_cast<unsigned*>(w);
  unsigned long long* st = reinterpret_cast<unsigned long long*>(w + 16);
  long long* agg2 = reinterpret_cast<long long*>(st + tiles);
  long long* inc2 = agg2 + tiles;
  cudaMemsetAsync(ws, 0, 16 + (size_t)tiles * sizeof(unsigned long long), s);
  switch (mode) {
    case 0:
      select_kernel<0><<<(unsigned)tiles, CP_THREADS, 0, s>>>(first_t, B, value, topo, plans, st, agg2, inc2, ticket,
                                                              tiles, idx, row, row2, count, total, total2);
      break;
    case 1:
      select_kernel<1><<<(unsigned)tiles, CP_THREADS, 0, s>>>(first_t, B, value, topo, plans, st, agg2, inc2, ticket,
                                                              tiles, idx, row, row2, count, total, total2);
      break;
    default:
      select_kernel<2><<<(unsigned)tiles, CP_THREADS, 0, s>>>(first_t, B, value, topo, plans, st, agg2, inc2, ticket,
                                                              tiles, idx, row, row2, count, total, total2);
  }
  return 0;
}

size_t la_compact_workspace(int64_t B) { return select_ws(B); }

size_t la_compact_rows_workspace(int64_t B) { return select_ws(B); }

int la_compact_rows(const int32_t* first_t, int64_t B, int32_t T, const int32_t* topo, const la_plan* plans,
                    int64_t* idx, int64_t* row_off, int64_t* count, int64_t* row_total, void* ws, size_t ws_bytes,
                    void* stream) {
  if (B < 0 || B >= (1ll << 31) / LA_MAX_JOINTS || !first_t || !plans || !idx || !row_off || !count || !row_total)
    return fail(LA_EINVAL, "la_compact_rows: bad args");
  if (ws_bytes < la_compact_rows_workspace(B) || !ws) return fail(LA_EWS, "la_compact_rows: workspace");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (B == 0) {
    cudaMemsetAsync(count, 0, sizeof(int64_t), s);
    cudaMemsetAsync(row_total, 0, sizeof(int64_t), s);
    return cuda_status("la_compact_rows");
  }
  select_launch(1, first_t, B, T, topo, plans, idx, row_off, nullptr, count, row_total, nullptr, ws, s);
  return cuda_status("la_compact_rows");
}

size_t la_compact_rows_split_workspace(int64_t B) { return select_ws(B); }

int la_compact_rows_split(const int32_t* first_t, int64_t B, int32_t T, const int32_t* topo, const la_plan* plans,
                          int64_t* idx, int64_t* target_row, int64_t* other_row, int64_t* count,
                          int64_t* target_total, int64_t* other_total, void* ws, size_t ws_bytes, void* stream) {
  if (B < 0 || B >= (1ll << 31) / LA_MAX_JOINTS || !first_t || !plans || !idx || !target_row || !other_row ||
      !count || !target_total || !other_total)
    return fail(LA_EINVAL, "la_compact_rows_split: bad args");
  if (ws_bytes < la_compact_rows_split_workspace(B) || !ws) return fail(LA_EWS, "la_compact_rows_split: workspace");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (B == 0) {
    cudaMemsetAsync(count, 0, sizeof(int64_t), s);
    cudaMemsetAsync(target_total, 0, sizeof(int64_t), s);
    cudaMemsetAsync(other_total, 0, sizeof(int64_t), s);
    return cuda_status("la_compact_rows_split");
  }
  select_launch(2, first_t, B, T, topo, plans, idx, target_row, other_row, count, target_total, other_total, ws, s);
  return cuda_status("la_compact_rows_split");
}

int la_compact_valid(const int32_t* first_t, int64_t B, int32_t T, int64_t* valid_idx,
                     int64_t* valid_count, void* ws, size_t ws_bytes, void* stream) {
  if (B < 0 || B >= (1ll << 31) || !first_t || !valid_idx || !valid_count)
    return fail(LA_EINVAL, "la_compact_valid: bad args");
  if (ws_bytes < la_compact_workspace(B) || !ws) return fail(LA_EWS, "la_compact_valid: workspace");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (B == 0) {
    cudaMemsetAsync(valid_count, 0, sizeof(int64_t), s);
    return cuda_status("la_compact_valid");
  }
  select_launch(0, first_t, B, T, nullptr, nullptr, valid_idx, nullptr, nullptr, valid_count, nullptr, nullptr, ws, s);
  return cuda_status("la_compact_valid");
}

}  // extern "C"
