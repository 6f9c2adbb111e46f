// Lane-per-candidate validity screen (sm_100a).
//
// Reference semantics: linkatlas solver.py
//   plan_geometry   solver.py:105-120 (batch form 189-201)
//   dyad_solve      solver.py:123-139, batch step 205-231 (lock rule, first_t /
//                   first_joint: earliest angle, then earliest plan step)
//   check_feasible  solver.py:242-249, find_valid_variant generator.py:263-283
//                   (T_low = T/4 sweep inside T; negatives keep the T_low step)
//
// Mapping.  Each LANE owns one candidate and walks its crank angles in the
// coarse-first order (t = 0, 4, 8, ... until the first lock; then the fine
// angles below that lock in ascending order; a coarse survivor either stops
// (LA_SIM_DEFER: its paths come from the write pass) or sweeps the fine
// angles).  Angles are independent (each t reads only same-t values,
// solver.py:159-165), so the lane stops exactly at its first lock: no angle
// beyond it is evaluated, and the per-candidate plan geometry is computed by
// 32 lanes at once.  A lane that finishes takes the next candidate of its
// warp's chunk (chunks of 32 consecutive work items, striding over the grid);
// refills are batched (>= refill_min free lanes) so the divergent f64
// prologue runs for several lanes at once.
//
// Per-warp shared memory, [row][lane] so every access is conflict-free:
//   col[j][lane]  float4 (x, y, e, -): fp32 joint position at the lane's
//                 current angle and a first-order bound e on its fp32 error
//   geo[s][lane]  float2 (r_a, +-r_b): fp32 step radii, sign = branch
//   idx[s][lane]  uint32 a | b << 8 | target << 16
//
// Precision.  The error bound of a dyad's target is
//   e_t = max(kappa, 1) * max(e_a, e_b) + kErrStep,  kappa = |x|(1+|x|/d)/h
// (amplification of the parents' error by a flat dyad; static joints and the
// crank tip start at kErr0).  A dyad whose margin min(ra+rb-d, d-|ra-rb|) is
// within tau + 3 max(e_a, e_b) of a lock, or NaN, makes the angle ambiguous:
// the lane parks on it ("blocked") and the warp replays the parked angles of
// all blocked lanes together in f64 once replay_min lanes are parked (or no
// unparked lane is left).  The f64 replay is exact-mode triaged as in sim.cu
// (fast pass; numpy's operation order when a lock test is within 1e-7).
#include "common.cuh"
#include "sim_common.cuh"

namespace la {
namespace {

constexpr int NJ = LA_MAX_JOINTS;
constexpr int SC_WARPS = 4;
constexpr int SC_THREADS = SC_WARPS * 32;
constexpr int kChunk = 32;  // work items per warp chunk

enum : int { PH_COARSE = 0, PH_BELOW = 1, PH_SWEEP = 2, PH_NATURAL = 3 };

__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// |p - q| in f64: glibc hypot bit for bit (exact mode) or a Newton-refined
// square root of the sum (an ulp or two)
template <bool EXACT>
__device__ __forceinline__ double dist64(double2 p, double2 q) {
  const double dx = dsub(p.x, q.x), dy = dsub(p.y, q.y);
  if (EXACT) return np_hypot(dx, dy);
  const double s = dadd(dmul(dx, dx), dmul(dy, dy));
  return s > 0.0 ? dmul(s, rsqrt_f64(s)) : 0.0;
}

__device__ __forceinline__ double2 ld_pose(const double* P0, int j) {
  return *reinterpret_cast<const double2*>(P0 + 2 * j);
}

// plan_geometry of one step (solver.py:105-120): r_a, r_b, branch
template <bool EXACT>
__device__ __forceinline__ void step_geometry(const double* P0, int t, int a, int b, double& ra, double& rb,
                                              double& br) {
  const double2 pa = ld_pose(P0, a), pb = ld_pose(P0, b), pt = ld_pose(P0, t);
  ra = dist64<EXACT>(pt, pa);
  rb = dist64<EXACT>(pt, pb);
  const double cross = dsub(dmul(dsub(pb.x, pa.x), dsub(pt.y, pa.y)), dmul(dsub(pb.y, pa.y), dsub(pt.x, pa.x)));
  br = cross >= 0.0 ? 1.0 : -1.0;
}

// one f64 evaluation of angle (ct, st) for a lane, positions in a
// lane-private array (rare path).  FAST: DFMA + Newton rsqrt, with the
// smallest distance of any lock test from its threshold in *margin;
// otherwise numpy's operation order (bit-identical lock decisions).
template <bool EXACT, bool FAST>
__device__ __forceinline__ int replay_pass(const double* P0, const la_plan* pl, int ns, double2* q, double* margin) {
  const double eps = 1e-9;
#pragma unroll 1
  for (int s = 0; s < ns; ++s) {
    const int t = (uint8_t)pl->step[s][0], a = (uint8_t)pl->step[s][1], b = (uint8_t)pl->step[s][2];
    double ra, rb, br;
    step_geometry<EXACT>(P0, t, a, b, ra, rb, br);
    const double hi = dadd(dadd(ra, rb), eps), lo = dsub(fabs(dsub(ra, rb)), eps);
    const double ra2 = dmul(ra, ra), rb2 = dmul(rb, rb);
    const double2 pa = q[a], pb = q[b];
    const double dx = dsub(pb.x, pa.x), dy = dsub(pb.y, pa.y);
    if (!FAST) {
      const double d = np_hypot(dx, dy);
      if (!(d >= eps) | (d > hi) | (d < lo)) return s;
      const double x = __ddiv_rn(dsub(dadd(dmul(d, d), ra2), rb2), dmul(2.0, d));
      const double h = __dsqrt_rn(fmax(dsub(ra2, dmul(x, x)), 0.0));
      const double ux = __ddiv_rn(dx, d), uy = __ddiv_rn(dy, d);
      const double bh = dmul(br, h);
      q[t] = make_double2(dsub(dadd(pa.x, dmul(x, ux)), dmul(bh, uy)), dadd(dadd(pa.y, dmul(x, uy)), dmul(bh, ux)));
    } else {
      const double d2 = fma(dy, dy, dx * dx);
      const double inv = rsqrt_f64(d2);
      const double d = d2 * inv;
      *margin = fmin(*margin, fmin(fabs(d - eps), fmin(fabs(hi - d), fabs(d - lo))));
      if (!(d >= eps) | (d > hi) | (d < lo)) return s;
      const double x = fma(d, d, ra2 - rb2) * (0.5 * inv);
      const double h2 = fma(-x, x, ra2);
      const double h2c = fmax(h2, 1e-300);
      const double h = h2 > 0.0 ? h2c * rsqrt_f64(h2c) : 0.0;
      const double xi = x * inv, hb = br * h * inv;
      q[t] = make_double2(fma(-hb, dy, fma(xi, dx, pa.x)), fma(hb, dx, fma(xi, dy, pa.y)));
    }
  }
  return -1;
}

// f64 decision for one (candidate, angle): first locking step or -1
template <bool EXACT>
__device__ __noinline__ int lane_replay(const double* P0, const la_plan* pl, double ct, double st) {
  double2 q[NJ];
  const int n = pl->n, ns = pl->nsteps;
#pragma unroll 1
  for (int j = 0; j < n; ++j) q[j] = ld_pose(P0, j);
  const double r1 = dist64<EXACT>(q[1], q[0]);  // solver.py:180
  q[1] = make_double2(dadd(q[0].x, dmul(r1, ct)), dadd(q[0].y, dmul(r1, st)));
  double margin = INFINITY;
  const int lk = replay_pass<EXACT, true>(P0, pl, ns, q, &margin);
  if (!EXACT || margin > kExactTriage) return lk;
  return replay_pass<true, false>(P0, pl, ns, q, nullptr);
}

struct LaneState {
  long long item = -1;  // work item, -1: free
  long long cand = 0;   // candidate row
  int ns = 0;
  int phase = 0, i = 0, lim = 0;
  int low_t = -1, low_j = -1, first_t = 0, first_j = -1;
  float r1f = 0.f;
  float2 p0f;
  bool blocked = false;
};

template <bool EXACT, bool COUNT>
__global__ void __launch_bounds__(SC_THREADS) screen_kernel(const la_sim_args p, int njmax, int smax,
                                                            int refill_min, int replay_min) {
  extern __shared__ __align__(16) unsigned char sc_smem[];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int T = p.T;
  float2* cs32 = reinterpret_cast<float2*>(sc_smem);
  const size_t cs_bytes = ((size_t)T * sizeof(float2) + 15) & ~(size_t)15;
  for (int t = threadIdx.x; t < T; t += SC_THREADS)
    cs32[t] = make_float2((float)p.crank_cs[2 * t], (float)p.crank_cs[2 * t + 1]);
  __syncthreads();
  const size_t per_warp = (size_t)512 * njmax + (size_t)384 * smax;
  unsigned char* wb = sc_smem + cs_bytes + per_warp * w;
  const uint32_t colb = smem_u32(wb) + lane * 16u;                                 // + j * 512
  const uint32_t geob = smem_u32(wb + 512 * njmax) + lane * 8u;                    // + s * 256
  const uint32_t idxb = smem_u32(wb + 512 * njmax + 256 * smax) + lane * 4u;       // + s * 128
  const uint32_t cs_b = smem_u32(cs32);

  long long nitems = p.cand ? p.n_cand : p.B;
  if (p.cand_count) {
    const long long c = *p.cand_count;
    nitems = c < nitems ? c : nitems;
  }
  const bool coarse = !(p.flags & LA_SIM_NO_COARSE) && (T % 4 == 0) && T >= 8;
  const bool gate_only = (p.flags & LA_SIM_GATE_ONLY) != 0;
  const bool defer = (p.flags & LA_SIM_DEFER) != 0;
  const bool scatter = (p.flags & LA_SIM_SCATTER) != 0;
  const int Tc = T / 4;
  const float tau = p.fixup_tau;
  const long long stride = (long long)gridDim.x * SC_WARPS;
  long long chunk = (long long)blockIdx.x * SC_WARPS + w;
  long long q = chunk * kChunk;
  long long qend = q + kChunk < nitems ? q + kChunk : nitems;
  const unsigned lt_mask = (1u << lane) - 1u;

  LaneState L;
  unsigned long long c_replay = 0, c_iter = 0, c_slots = 0, c_cand = 0, c_events = 0, c_angles = 0, c_dyads = 0;

  auto finish = [&]() {
    const long long o = scatter && p.cand ? p.cand[L.item] : L.item;
    if (p.first_t) p.first_t[o] = L.first_t;
    if (p.first_joint) p.first_joint[o] = L.first_j;
    if (p.low_t) p.low_t[o] = L.low_t;
    if (p.low_joint) p.low_joint[o] = L.low_j;
    L.item = -1;
  };

#pragma unroll 1
  for (;;) {
    // ---- refill free lanes from the warp's chunk queue (batched)
    unsigned freem = __ballot_sync(FULL, L.item < 0);
    if (freem && q < nitems && (__popc(freem) >= refill_min || freem == FULL)) {
      long long mine = -1;
#pragma unroll 1
      while (freem && q < nitems) {
        const int take = min(__popc(freem), (int)(qend - q));
        const int rank = __popc(freem & lt_mask);
        const bool get = ((freem >> lane) & 1u) && rank < take;
        if (get) mine = q + rank;
        freem &= ~__ballot_sync(FULL, get);
        q += take;
        if (q >= qend) {
          chunk += stride;
          q = chunk * kChunk;
          qend = q + kChunk < nitems ? q + kChunk : nitems;
        }
      }
      if (mine >= 0) {
        // ---- prologue: plan, static joints, step geometry (f64 -> fp32)
        L.item = mine;
        L.cand = p.cand ? p.cand[mine] : mine;
        const la_plan* pl = p.plans + (p.topo ? p.topo[L.cand] : 0);
        const int n = pl->n;
        L.ns = pl->nsteps;
        L.low_t = -1;
        L.low_j = -1;
        L.first_t = T;
        L.first_j = -1;
        L.blocked = false;
        if (n > njmax || n < 2 || L.ns > smax || L.ns < 0) {
          L.first_t = -1;  // plan does not fit the launch
          L.first_j = -2;
          finish();
        } else {
          if (COUNT) ++c_cand;
          const double* P0 = p.pos0 + (size_t)L.cand * p.pos_stride * 2;
          const uint32_t fixed = (uint32_t)pl->fixed_mask | 1u;  // joint 0 is static (solver.py:183)
#pragma unroll 1
          for (int j = 0; j < n; ++j) {
            if (j == 1 || !((fixed >> j) & 1u)) continue;
            const double2 v = ld_pose(P0, j);
            sts_f4(colb + 512u * j, make_float4((float)v.x, (float)v.y, kErr0, 0.f));
          }
#pragma unroll 1
          for (int s = 0; s < L.ns; ++s) {
            const int t = (uint8_t)pl->step[s][0], a = (uint8_t)pl->step[s][1], b = (uint8_t)pl->step[s][2];
            double ra, rb, br;
            step_geometry<EXACT>(P0, t, a, b, ra, rb, br);
            sts_f2(geob + 256u * s, make_float2((float)ra, copysignf((float)rb, (float)br)));
            sts_u32(idxb + 128u * s, (uint32_t)a | ((uint32_t)b << 8) | ((uint32_t)t << 16));
          }
          const double2 j0 = ld_pose(P0, 0), j1 = ld_pose(P0, 1);
          L.r1f = (float)dist64<EXACT>(j1, j0);  // solver.py:180
          L.p0f = make_float2((float)j0.x, (float)j0.y);
          sts_f4(colb + 512u, make_float4(0.f, 0.f, kErr0, 0.f));
          if (coarse) {
            L.phase = PH_COARSE;
            L.lim = Tc;
          } else {
            L.phase = PH_NATURAL;
            L.lim = T;
          }
          L.i = 0;
          if (!coarse && defer) {  // nothing to screen: every candidate pending
            L.first_t = LA_PENDING;
            finish();
          }
        }
      }
    }
    if (__ballot_sync(FULL, L.item >= 0) == 0) {
      if (q >= nitems) break;
      continue;
    }

    // ---- one angle per lane
    const int t = L.phase == PH_COARSE ? 4 * L.i : (L.phase == PH_NATURAL ? L.i : fine_angle(L.i));
    const bool run = L.item >= 0 && !L.blocked;
    int lk = -1, ndy = 0;
    bool fix = false;
    if (run) {
      const float2 c = lds_f2(cs_b + 8u * t);
      sts_f2(colb + 512u, make_float2(fmaf(L.r1f, c.x, L.p0f.x), fmaf(L.r1f, c.y, L.p0f.y)));
      int s = 0;
#pragma unroll 1
      for (; s < L.ns; ++s) {
        const uint32_t wd = lds_u32(idxb + 128u * s);
        const float2 g = lds_f2(geob + 256u * s);
        const float4 A = lds_f4(colb + ((wd & 0xffu) << 9));
        const float4 B = lds_f4(colb + (((wd >> 8) & 0xffu) << 9));
        const float dx = B.x - A.x, dy = B.y - A.y;
        const float d2 = fmaf(dy, dy, dx * dx);
        const float inv = rsqrt_approx(d2);
        const float d = d2 * inv;
        const float ra = g.x, rb = fabsf(g.y);
        const float sp = ra + rb, dm = ra - rb;
        const float m = fminf(sp - d, d - fabsf(dm));
        const float ep = fmaxf(A.z, B.z);
        fix |= !(fabsf(m) >= fmaf(kMarginK, ep, tau));  // NaN -> f64 decides
        if (m < 0.0f) {
          lk = s;
          break;
        }
        const float x = fmaf(dm, sp, d2) * (0.5f * inv);
        const float h2 = fmaxf(fmaf(-x, x, ra * ra), 1e-30f);
        const float rh = rsqrt_approx(h2);
        const float h = h2 * rh;
        const float ax = fabsf(x);
        const float kap = ax * fmaf(ax, inv, 1.0f) * rh;  // |x| (1 + |x|/d) / h
        const float e = fmaf(fmaxf(kap, 1.0f), ep, kErrStep);
        const float xi = x * inv;
        const float hb = copysignf(h, g.y) * inv;
        sts_f4(colb + ((wd >> 16) << 9),
               make_float4(fmaf(-hb, dy, fmaf(xi, dx, A.x)), fmaf(hb, dx, fmaf(xi, dy, A.y)), e, 0.f));
      }
      ndy = s < L.ns ? s + 1 : L.ns;
      if (fix) L.blocked = true;
    }
    if (COUNT) {
      ++c_iter;
      c_slots += 32ull * (unsigned)__reduce_max_sync(FULL, (unsigned)ndy);
      if (run) {
        ++c_angles;
        c_dyads += (unsigned)ndy;
      }
    }
    bool decided = run && !fix;
    const unsigned bl = __ballot_sync(FULL, L.blocked);
    if (bl) {
      const unsigned running = __ballot_sync(FULL, L.item >= 0 && !L.blocked);
      if (__popc(bl) >= replay_min || running == 0) {
        if (L.blocked) {
          const la_plan* pl = p.plans + (p.topo ? p.topo[L.cand] : 0);
          const double* P0 = p.pos0 + (size_t)L.cand * p.pos_stride * 2;
          lk = lane_replay<EXACT>(P0, pl, p.crank_cs[2 * t], p.crank_cs[2 * t + 1]);
          L.blocked = false;
          decided = true;
          if (COUNT) ++c_replay;
        }
        if (COUNT && lane == 0) ++c_events;
      }
    }
    if (decided) {
      // ---- advance the lane's angle walk with this angle's outcome
      const int tj = lk >= 0 ? (int)((lds_u32(idxb + 128u * lk) >> 16) & 0xffu) : -1;
      switch (L.phase) {
        case PH_COARSE:
          if (lk >= 0) {
            L.low_t = L.i;
            L.low_j = tj;
            L.first_t = 4 * L.i;
            L.first_j = tj;
            if (gate_only || L.i == 0) {
              finish();
            } else {
              L.phase = PH_BELOW;
              L.lim = 3 * L.i;
              L.i = 0;
            }
          } else if (++L.i == L.lim) {
            if (defer) {
              L.first_t = LA_PENDING;  // coarse survivor: decided by the write pass
              finish();
            } else {
              L.phase = PH_SWEEP;
              L.lim = 3 * Tc;
              L.i = 0;
            }
          }
          break;
        case PH_BELOW:
        case PH_SWEEP:
          if (lk >= 0) {
            L.first_t = fine_angle(L.i);
            L.first_j = tj;
            finish();
          } else if (++L.i == L.lim) {
            if (L.phase == PH_SWEEP) L.first_t = T;
            finish();  // PH_BELOW: first_t stays at the coarse lock
          }
          break;
        default:  // PH_NATURAL
          if (lk >= 0) {
            L.first_t = L.i;
            L.first_j = tj;
            finish();
          } else if (++L.i == L.lim) {
            L.first_t = T;
            finish();
          }
          break;
      }
    }
  }
  if (COUNT && p.counters) {
    unsigned long long f = c_replay, la = c_angles, ld = c_dyads, nc = c_cand;
    for (int o = 16; o > 0; o >>= 1) {
      f += __shfl_xor_sync(FULL, f, o);
      la += __shfl_xor_sync(FULL, la, o);
      ld += __shfl_xor_sync(FULL, ld, o);
      nc += __shfl_xor_sync(FULL, nc, o);
    }
    if (lane == 0) {
      atomicAdd(p.counters + 0, f);
      atomicAdd(p.counters + 1, 32ull * c_iter);
      atomicAdd(p.counters + 2, c_slots);
      atomicAdd(p.counters + 3, nc);
      atomicAdd(p.counters + 4, c_events);
      atomicAdd(p.counters + 5, la);
      atomicAdd(p.counters + 6, ld);
    }
  }
}

}  // namespace

// lane-per-candidate screen launch (la_simulate without LA_SIM_WRITE_TRAJ /
// LA_SIM_FP64); arguments already validated by la_simulate
int launch_screen_lane(const la_sim_args& a, cudaStream_t s) {
  const int njmax = a.pos_stride < NJ ? a.pos_stride : NJ;
  const int smax = njmax - 1 < LA_MAX_STEPS ? njmax - 1 : LA_MAX_STEPS;
  const size_t cs_bytes = ((size_t)a.T * sizeof(float2) + 15) & ~(size_t)15;
  const size_t smem = cs_bytes + ((size_t)512 * njmax + (size_t)384 * smax) * SC_WARPS;
  const bool exact = (a.flags & LA_SIM_EXACT64) != 0;
  using KernT = void (*)(const la_sim_args, int, int, int, int);
  const KernT kern = exact ? (a.counters ? screen_kernel<true, true> : screen_kernel<true, false>)
                           : (a.counters ? screen_kernel<false, true> : screen_kernel<false, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return fail((int)e, "la_simulate(screen): smem attr: %s", cudaGetErrorString(e));
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, SC_THREADS, smem);
  if (e != cudaSuccess) return fail((int)e, "la_simulate(screen): occupancy: %s", cudaGetErrorString(e));
  const int sms = sm_count();
  if (sms <= 0) return fail(LA_EINVAL, "la_simulate: no device");
  const long long items = a.cand ? a.n_cand : a.B;
  const long long chunks = (items + kChunk - 1) / kChunk;
  long long grid = (long long)sms * (occ > 0 ? occ : 1);
  const long long need = (chunks + SC_WARPS - 1) / SC_WARPS;
  if (grid > need) grid = need;
  // refills of >= 8 free lanes share one divergent prologue; parked lanes
  // are replayed in f64 in batches of >= 4
  kern<<<(unsigned)grid, SC_THREADS, smem, s>>>(a, njmax, smax, a.screen_refill > 0 ? a.screen_refill : 8,
                                                a.screen_replay > 0 ? a.screen_replay : 4);
  return cuda_status("la_simulate(screen)");
}

}  // namespace la
