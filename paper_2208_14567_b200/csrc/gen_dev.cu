// Device-side candidate poses for the generation engine: each thread jumps a
// copy of its slot's PCG64 pose stream to its candidate's first draw and
// draws the 2n uniforms of _sample_positions_batch (generator.py:234-238)
// bit for bit (numpy random(): (next64 >> 11) * 2^-53, XSL-RR output).
#include <algorithm>

#include "common.cuh"

namespace la {
namespace {

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 mk(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }

__global__ void __launch_bounds__(256) gen_poses_kernel(const la_gen_batch* __restrict__ batches, int nb,
                                                         int stride, double* __restrict__ pos,
                                                         int32_t* __restrict__ topo) {
  const u128 MULT = mk(0x2360ED051FC65DA4ULL, 0x4385DF649FCCF645ULL);
  for (int bi = blockIdx.x; bi < nb; bi += gridDim.x) {
    const la_gen_batch b = batches[bi];
    const u128 inc = mk(b.inc_hi, b.inc_lo);
    const u128 s0 = mk(b.state_hi, b.state_lo);
    // jump table for this batch: per-thread stride = blockDim.x candidates
    for (int c = threadIdx.x; c < b.k; c += blockDim.x) {
      // advance s0 by c * 2n steps
      u128 delta = (u128)c * (u128)(2 * b.n);
      u128 cm = MULT, cp = inc, am = 1, ap = 0;
      while (delta) {
        if ((uint64_t)delta & 1u) {
          am *= cm;
          ap = ap * cm + cp;
        }
        cp = (cm + 1) * cp;
        cm *= cm;
        delta >>= 1;
      }
      u128 st = am * s0 + ap;
      double* row = pos + (size_t)(b.first + c) * stride * 2;
      for (int j = 0; j < b.n; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          st = st * MULT + inc;
          const uint64_t hi = (uint64_t)(st >> 64), lo = (uint64_t)st;
          const unsigned rot = (unsigned)(hi >> 58);
          const uint64_t x = hi ^ lo;
          const uint64_t r = (x >> rot) | (x << ((64u - rot) & 63u));
          row[2 * j + e] = (double)(r >> 11) * (1.0 / 9007199254740992.0);
        }
      }
      row[0] = 0.5;
      row[1] = 0.5;
      row[2] = 0.55;
      row[3] = 0.5;
      for (int j = b.n; j < stride; ++j) row[2 * j] = row[2 * j + 1] = __longlong_as_double(0x7ff8000000000000LL);
      topo[b.first + c] = b.plan;
    }
  }
}

}  // namespace
}  // namespace la

extern "C" int la_gen_poses(const la_gen_batch* batches, int64_t n_batches, int32_t stride, double* pos,
                            int32_t* topo, void* stream) {
  using namespace la;
  if (n_batches < 0 || stride < 1 || stride > LA_MAX_JOINTS) return fail(LA_EINVAL, "la_gen_poses: bad sizes");
  if (n_batches == 0) return 0;
  if (!batches || !pos || !topo) return fail(LA_EINVAL, "la_gen_poses: null buffer");
  const int grid = (int)(n_batches < 65535 ? n_batches : 65535);
  gen_poses_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(batches, (int)n_batches, stride, pos, topo);
  return cuda_status("gen_poses_kernel");
}

// ---------------------------------------------------------------------------
// Record-keyed curation keep rule (curves.py:104-110): a flagged (arc or
// circle) record survives iff default_rng([seed, mech_id, joint_id]).random()
// < keep_rate.  Thread per record: numpy SeedSequence (entropy words of the
// three ints, pool of 4, hashmix/mix constants of numpy's bit_generator) ->
// 8 state words -> PCG64 seeding -> one 53-bit double.
namespace la {
namespace {

__device__ __forceinline__ int entropy_words(unsigned long long v, uint32_t* w, int n) {
  if (v == 0) {
    w[n++] = 0;
    return n;
  }
  while (v) {
    w[n++] = (uint32_t)(v & 0xffffffffu);
    v >>= 32;
  }
  return n;
}

__device__ double seeded_uniform(const uint32_t* ent, int ne) {
  const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
  const uint32_t ML = 0xca01f9ddu, MR = 0x4973f715u;
  uint32_t hc = INIT_A;
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= MULT_A;
    v *= hc;
    v ^= v >> 16;
    return v;
  };
  auto mix = [](uint32_t x, uint32_t y) {
    uint32_t r = ML * x - MR * y;
    r ^= r >> 16;
    return r;
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < ne ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (int s = 4; s < ne; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s]));
  uint32_t w[8];
  uint32_t hb = INIT_B;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= MULT_B;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  uint64_t v[4];
  for (int i = 0; i < 4; ++i) v[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
  const u128 MULT = mk(0x2360ED051FC65DA4ULL, 0x4385DF649FCCF645ULL);
  const u128 inc = (mk(v[2], v[3]) << 1) | 1u;
  u128 st = 0;
  st = st * MULT + inc;
  st += mk(v[0], v[1]);
  st = st * MULT + inc;
  st = st * MULT + inc;  // next64: step then output
  const uint64_t hi = (uint64_t)(st >> 64), lo = (uint64_t)st;
  const unsigned rot = (unsigned)(hi >> 58);
  const uint64_t x = hi ^ lo;
  const uint64_t r = (x >> rot) | (x << ((64u - rot) & 63u));
  return (double)(r >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void curation_keep_kernel(const int64_t* __restrict__ mech, const int64_t* __restrict__ joint,
                                     const uint8_t* __restrict__ flagged, long long n, long long seed,
                                     double keep_rate, uint8_t* __restrict__ keep) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    if (!flagged[i]) {
      keep[i] = 1;
      continue;
    }
    uint32_t ent[6];
    int ne = entropy_words((unsigned long long)seed, ent, 0);
    ne = entropy_words((unsigned long long)mech[i], ent, ne);
    ne = entropy_words((unsigned long long)joint[i], ent, ne);
    keep[i] = seeded_uniform(ent, ne) < keep_rate;
  }
}

}  // namespace
}  // namespace la

extern "C" int la_curation_keep(const int64_t* mech_ids, const int64_t* joint_ids, const uint8_t* flagged,
                                int64_t n, int64_t seed, double keep_rate, uint8_t* keep, void* stream) {
  using namespace la;
  if (n < 0 || seed < 0) return fail(LA_EINVAL, "la_curation_keep: bad arguments");
  if (n == 0) return 0;
  if (!mech_ids || !joint_ids || !flagged || !keep) return fail(LA_EINVAL, "la_curation_keep: null buffer");
  const long long blocks = std::min<long long>((n + 255) / 256, (long long)sm_count() * 16);
  curation_keep_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(mech_ids, joint_ids, flagged, n, seed,
                                                                           keep_rate, keep);
  return cuda_status("curation_keep_kernel");
}
