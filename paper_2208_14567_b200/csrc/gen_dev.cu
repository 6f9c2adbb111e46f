// Device-side candidate poses for the generation engine: each thread jumps a
// copy of its slot's PCG64 pose stream to its candidate's first draw and
// draws the 2n uniforms of _sample_positions_batch (generator.py:234-238)
// bit for bit (numpy random(): (next64 >> 11) * 2^-53, XSL-RR output).
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
