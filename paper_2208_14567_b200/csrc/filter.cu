// Coarse prefilter of Atlas.coarse_filter (atlas.py:153-177) on the device.
//
//   descriptor (atlas.py:167-172): 16-bin histogram of r = hypot(x-.5, y-.5)
//     over [0, 0.75] (np.histogram semantics: r outside the range dropped,
//     the last bin closed), divided by the point count, then the bbox extent
//     (max - min per axis)                                   -> 18 f64
//   distance (atlas.py:162): L1 to the query descriptor, summed in numpy's
//     pairwise order for 18 contiguous terms (8 accumulators, then the
//     remainder)                                             -> f64, bit-exact
//   keep (atlas.py:163-166): the `budget` smallest by (distance, index)
//     (stable argsort), emitted in scan order (order filtered by the mask)
//
// Selection is a sync-free 8-pass radix select on the distance bit patterns
// (non-negative doubles order like their uint64 bits) with the final tie
// class resolved by index through an ordered ballot compaction, then a
// second ordered compaction over the scan order.
#include <algorithm>

#include "common.cuh"

namespace la {
namespace {

constexpr int DESC = 18;
constexpr int NBINS = 16;
constexpr int FT = 1024;  // tile of the ordered compactions

struct Edges {
  double e[NBINS + 1];
};

// warp per curve
__global__ void __launch_bounds__(256) descriptor_kernel(const double* __restrict__ paths, long long M, int P,
                                                          Edges ed, double* __restrict__ desc) {
  __shared__ int hist[8][NBINS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long m = (long long)blockIdx.x * 8 + w;
  if (m >= M) return;
  if (lane < NBINS) hist[w][lane] = 0;
  __syncwarp();
  const double* p = paths + (size_t)m * P * 2;
  double mnx = INFINITY, mxx = -INFINITY, mny = INFINITY, mxy = -INFINITY;
  for (int i = lane; i < P; i += 32) {
    const double x = p[2 * i], y = p[2 * i + 1];
    mnx = fmin(mnx, x);
    mxx = fmax(mxx, x);
    mny = fmin(mny, y);
    mxy = fmax(mxy, y);
    const double r = np_hypot(__dsub_rn(x, 0.5), __dsub_rn(y, 0.5));
    if (r >= ed.e[0] && r <= ed.e[NBINS]) {
      int b = NBINS - 1;  // last bin closed on the right
      for (int k = 1; k < NBINS; ++k)
        if (r < ed.e[k]) {
          b = k - 1;
          break;
        }
      atomicAdd(&hist[w][b], 1);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    mnx = fmin(mnx, __shfl_xor_sync(FULL, mnx, o));
    mxx = fmax(mxx, __shfl_xor_sync(FULL, mxx, o));
    mny = fmin(mny, __shfl_xor_sync(FULL, mny, o));
    mxy = fmax(mxy, __shfl_xor_sync(FULL, mxy, o));
  }
  __syncwarp();
  double* d = desc + (size_t)m * DESC;
  const double denom = (double)(P > 1 ? P : 1);
  if (lane < NBINS) d[lane] = __ddiv_rn((double)hist[w][lane], denom);
  if (lane == NBINS) d[NBINS] = __dsub_rn(mxx, mnx);
  if (lane == NBINS + 1) d[NBINS + 1] = __dsub_rn(mxy, mny);
}

struct SelState {
  unsigned long long prefix, mask;
  long long k;  // how many still to take from the prefix class
  long long pad;
};

// L1 distance in numpy's pairwise order; key = distance bits
__global__ void dist_kernel(const double* __restrict__ desc, long long M, const double* __restrict__ q,
                            unsigned long long* __restrict__ key, double* __restrict__ dist_out) {
  __shared__ double qs[DESC];
  if (threadIdx.x < DESC) qs[threadIdx.x] = q[threadIdx.x];
  __syncthreads();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (long long)gridDim.x * blockDim.x) {
    const double* a = desc + (size_t)i * DESC;
    double t[DESC];
#pragma unroll
    for (int j = 0; j < DESC; ++j) t[j] = fabs(__dsub_rn(a[j], qs[j]));
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(t[j], t[8 + j]);
    double s = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    s = __dadd_rn(s, t[16]);
    s = __dadd_rn(s, t[17]);
    key[i] = (unsigned long long)__double_as_longlong(s);
    if (dist_out) dist_out[i] = s;
  }
}

__global__ void radix_hist(const unsigned long long* __restrict__ key, long long M, const SelState* st, int shift,
                           unsigned int* __restrict__ ghist) {
  __shared__ unsigned int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const unsigned long long pre = st->prefix, msk = st->mask;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long k = key[i];
    if ((k & msk) == pre) atomicAdd(&h[(k >> shift) & 255u], 1u);
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&ghist[threadIdx.x], h[threadIdx.x]);
}

// one block of 256: choose the digit holding the k-th smallest, clear hist
__global__ void radix_choose(unsigned int* ghist, SelState* st, int shift) {
  __shared__ unsigned long long cum[256];
  const int t = threadIdx.x;
  cum[t] = ghist[t];
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {
    const unsigned long long v = t >= o ? cum[t - o] : 0;
    __syncthreads();
    cum[t] += v;
    __syncthreads();
  }
  const long long k = st->k;
  const unsigned long long incl = cum[t], excl = t ? cum[t - 1] : 0;
  __syncthreads();
  if ((long long)excl < k && k <= (long long)incl) {
    st->prefix |= (unsigned long long)t << shift;
    st->mask |= 255ull << shift;
    st->k = k - (long long)excl;
  }
  ghist[t] = 0;
}

// ---- ordered compactions (tile = FT items, ballot + warp scan) ----------
template <class Pred>
__device__ __forceinline__ void tile_rank(bool v, int* wsum, unsigned& bal, int& before) {
  bal = __ballot_sync(FULL, v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) wsum[w] = __popc(bal);
  __syncthreads();
  if (threadIdx.x < 32) {
    const int s = wsum[lane];
    int x = s;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    wsum[32 + lane] = x - s;  // exclusive warp offsets
    if (lane == 31) wsum[64] = x;
  }
  __syncthreads();
  before = wsum[32 + w] + __popc(bal & ((1u << lane) - 1u));
}

struct TiePred {
  const unsigned long long* key;
  const SelState* st;
  __device__ bool operator()(long long i) const { return key[i] == st->prefix; }
};

struct ScanPred {
  const unsigned char* keep;
  const int64_t* order;
  __device__ bool operator()(long long p) const { return keep[order ? order[p] : p] != 0; }
};

template <class Pred>
__global__ void tile_count(Pred pred, long long n, long long* cnt) {
  __shared__ int wsum[65];
  const long long i = (long long)blockIdx.x * FT + threadIdx.x;
  const bool v = i < n && pred(i);
  unsigned bal;
  int before;
  tile_rank<Pred>(v, wsum, bal, before);
  if (threadIdx.x == 0) cnt[blockIdx.x] = wsum[64];
}

// single block exclusive scan of tile counts (in place)
__global__ void tile_scan(long long* cnt, long long ntiles) {
  __shared__ long long carry;
  __shared__ long long ws[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (long long base = 0; base < ntiles; base += 1024) {
    const long long i = base + threadIdx.x;
    const long long v = i < ntiles ? cnt[i] : 0;
    long long x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(FULL, x, o);
      if ((threadIdx.x & 31) >= o) x += y;
    }
    if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      long long s = ws[threadIdx.x];
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(FULL, s, o);
        if (threadIdx.x >= o) s += y;
      }
      ws[threadIdx.x] = s;
    }
    __syncthreads();
    const long long wb = threadIdx.x >= 32 ? ws[(threadIdx.x >> 5) - 1] : 0;
    const long long excl = carry + wb + x - v;
    __syncthreads();
    if (i < ntiles) cnt[i] = excl;
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
}

// keep[i] = key < K  or  (key == K and rank among ties < k)
__global__ void keep_kernel(const unsigned long long* __restrict__ key, long long n, const SelState* st,
                            const long long* __restrict__ off, unsigned char* __restrict__ keep) {
  __shared__ int wsum[65];
  const long long i = (long long)blockIdx.x * FT + threadIdx.x;
  const unsigned long long K = st->prefix;
  const unsigned long long ki = i < n ? key[i] : ~0ull;
  const bool tie = i < n && ki == K;
  unsigned bal;
  int before;
  tile_rank<TiePred>(tie, wsum, bal, before);
  if (i < n) keep[i] = (ki < K) || (tie && off[blockIdx.x] + before < st->k);
}

__global__ void emit_kernel(ScanPred pred, long long n, const long long* __restrict__ off, int64_t* __restrict__ out) {
  __shared__ int wsum[65];
  const long long p = (long long)blockIdx.x * FT + threadIdx.x;
  const bool v = p < n && pred(p);
  unsigned bal;
  int before;
  tile_rank<ScanPred>(v, wsum, bal, before);
  if (v) out[off[blockIdx.x] + before] = pred.order ? pred.order[p] : p;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace
}  // namespace la

extern "C" int la_coarse_descriptors(const double* paths, int64_t M, int32_t P, const double* edges, double* desc,
                                     void* stream) {
  using namespace la;
  if (M < 0 || P < 1) return fail(LA_EINVAL, "la_coarse_descriptors: bad sizes");
  if (M == 0) return 0;
  if (!paths || !edges || !desc) return fail(LA_EINVAL, "la_coarse_descriptors: null buffer");
  Edges ed;
  for (int k = 0; k <= NBINS; ++k) ed.e[k] = edges[k];
  const long long blocks = (M + 7) / 8;
  descriptor_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(paths, M, P, ed, desc);
  return cuda_status("descriptor_kernel");
}

extern "C" size_t la_coarse_workspace(int64_t M) {
  using namespace la;
  const long long tiles = (M + FT - 1) / FT;
  return align256(sizeof(SelState)) + align256(256 * sizeof(unsigned int)) + align256((size_t)M * 8) +
         align256((size_t)M) + align256((size_t)(tiles + 1) * 8);
}

extern "C" int la_coarse_select(const double* desc, int64_t M, const double* qdesc, int64_t budget,
                                const int64_t* order, int64_t* out, double* dist_out, void* ws, size_t ws_bytes,
                                void* stream) {
  using namespace la;
  if (M < 0 || budget < 0) return fail(LA_EINVAL, "la_coarse_select: bad sizes");
  if (M == 0 || budget == 0) return 0;
  if (!desc || !qdesc || !out || !ws) return fail(LA_EINVAL, "la_coarse_select: null buffer");
  if (ws_bytes < la_coarse_workspace(M)) return fail(LA_EWS, "la_coarse_select: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  char* w = (char*)ws;
  SelState* st = (SelState*)w;
  w += align256(sizeof(SelState));
  unsigned int* hist = (unsigned int*)w;
  w += align256(256 * sizeof(unsigned int));
  unsigned long long* key = (unsigned long long*)w;
  w += align256((size_t)M * 8);
  unsigned char* keep = (unsigned char*)w;
  w += align256((size_t)M);
  long long* off = (long long*)w;
  const long long tiles = (M + FT - 1) / FT;
  const long long k = budget < M ? budget : M;
  SelState init = {0ull, 0ull, k, 0};
  cudaMemcpyAsync(st, &init, sizeof(init), cudaMemcpyHostToDevice, s);
  cudaMemsetAsync(hist, 0, 256 * sizeof(unsigned int), s);
  const int sms = sm_count();
  const long long gblocks = std::min<long long>((M + 255) / 256, (long long)sms * 8);
  dist_kernel<<<(unsigned)gblocks, 256, 0, s>>>(desc, M, qdesc, key, dist_out);
  for (int shift = 56; shift >= 0; shift -= 8) {
    radix_hist<<<(unsigned)gblocks, 256, 0, s>>>(key, M, st, shift, hist);
    radix_choose<<<1, 256, 0, s>>>(hist, st, shift);
  }
  tile_count<TiePred><<<(unsigned)tiles, FT, 0, s>>>(TiePred{key, st}, M, off);
  tile_scan<<<1, 1024, 0, s>>>(off, tiles);
  keep_kernel<<<(unsigned)tiles, FT, 0, s>>>(key, M, st, off, keep);
  ScanPred sp{keep, order};
  tile_count<ScanPred><<<(unsigned)tiles, FT, 0, s>>>(sp, M, off);
  tile_scan<<<1, 1024, 0, s>>>(off, tiles);
  emit_kernel<<<(unsigned)tiles, FT, 0, s>>>(sp, M, off, out);
  return cuda_status("la_coarse_select");
}
