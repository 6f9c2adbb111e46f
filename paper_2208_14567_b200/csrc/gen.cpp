// Native (host, multi-threaded) candidate generator: the reference's random
// topology operator and pose sampling, reproducing numpy's PCG64 streams.
//
// Reference: linkatlas generator.py
//   _grow_topology          generator.py:156-197
//   sample_topology         generator.py:200-222 (compile_plan solver.py:71-102,
//                           plan_ancestry curves.py:132-150)
//   _sample_positions_batch generator.py:234-238
//   _generate_slot streams  generator.py:290-292: default_rng([seed, slot, k])
// numpy pieces restated (numpy 2.x, verified bit-for-bit by
// tests/test_native_gen.py): SeedSequence entropy mixing and generate_state,
// PCG64 (128-bit LCG, XSL-RR output) seeding, Generator.random() /
// uniform() (53-bit doubles), Generator.integers() (Lemire bounded draw on
// the buffered 32-bit stream).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "links_b200.h"

namespace la {
void set_error(const char* fmt, ...);
}

namespace {

typedef unsigned __int128 u128;

// ---------------------------------------------------------------- SeedSequence
constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u;
constexpr uint32_t INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
constexpr uint32_t MIX_MULT_L = 0xca01f9ddu, MIX_MULT_R = 0x4973f715u;
constexpr int XSHIFT = 16;
constexpr int POOL = 4;

void int_words(uint64_t v, std::vector<uint32_t>& out) {
  if (v == 0) {
    out.push_back(0);
    return;
  }
  while (v > 0) {
    out.push_back((uint32_t)(v & 0xffffffffu));
    v >>= 32;
  }
}

struct SeedSeq {
  uint32_t pool[POOL];
  explicit SeedSeq(const std::vector<uint32_t>& ent) {
    uint32_t hc = INIT_A;
    auto hashmix = [&](uint32_t v) {
      v ^= hc;
      hc *= MULT_A;
      v *= hc;
      v ^= v >> XSHIFT;
      return v;
    };
    auto mix = [](uint32_t x, uint32_t y) {
      uint32_t r = MIX_MULT_L * x - MIX_MULT_R * y;
      r ^= r >> XSHIFT;
      return r;
    };
    for (int i = 0; i < POOL; ++i) pool[i] = hashmix(i < (int)ent.size() ? ent[i] : 0u);
    for (int s = 0; s < POOL; ++s)
      for (int d = 0; d < POOL; ++d)
        if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
    for (size_t s = POOL; s < ent.size(); ++s)
      for (int d = 0; d < POOL; ++d) pool[d] = mix(pool[d], hashmix(ent[s]));
  }
  void generate(uint32_t* out, int n) const {
    uint32_t hc = INIT_B;
    for (int i = 0; i < n; ++i) {
      uint32_t v = pool[i % POOL];
      v ^= hc;
      hc *= MULT_B;
      v *= hc;
      v ^= v >> XSHIFT;
      out[i] = v;
    }
  }
};

// ---------------------------------------------------------------- PCG64
const u128 PCG_MULT = ((u128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;

struct Pcg64 {
  u128 state, inc;
  int has32 = 0;
  uint32_t u32 = 0;
  explicit Pcg64(const std::vector<uint32_t>& entropy) {
    SeedSeq sq(entropy);
    uint32_t w[8];
    sq.generate(w, 8);
    uint64_t v[4];
    for (int i = 0; i < 4; ++i) v[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
    const u128 s = ((u128)v[0] << 64) | v[1];
    const u128 q = ((u128)v[2] << 64) | v[3];
    state = 0;
    inc = (q << 1) | 1u;
    step();
    state += s;
    step();
  }
  void step() { state = state * PCG_MULT + inc; }
  uint64_t next64() {
    step();
    const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    const unsigned rot = (unsigned)(state >> 122);
    const uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  uint32_t next32() {
    if (has32) {
      has32 = 0;
      return u32;
    }
    const uint64_t n = next64();
    has32 = 1;
    u32 = (uint32_t)(n >> 32);
    return (uint32_t)(n & 0xffffffffu);
  }
  double random() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
  // Generator.integers(low, high) for a 32-bit range (Lemire, numpy's
  // buffered_bounded_lemire_uint32 on the 32-bit stream)
  int64_t integers(int64_t low, int64_t high) {
    const uint64_t rng = (uint64_t)(high - low - 1);
    if (rng == 0) return low;
    const uint32_t rexcl = (uint32_t)rng + 1u;
    uint64_t m = (uint64_t)next32() * rexcl;
    uint32_t left = (uint32_t)m;
    if (left < rexcl) {
      const uint32_t thr = (uint32_t)(-rexcl) % rexcl;
      while (left < thr) {
        m = (uint64_t)next32() * rexcl;
        left = (uint32_t)m;
      }
    }
    return low + (int64_t)(m >> 32);
  }
};

Pcg64 stream(int64_t seed, int64_t slot, int64_t k) {
  std::vector<uint32_t> e;
  int_words((uint64_t)seed, e);
  int_words((uint64_t)slot, e);
  int_words((uint64_t)k, e);
  return Pcg64(e);
}

// ---------------------------------------------------------------- topology
constexpr int MAXJ = LA_MAX_JOINTS;
enum { FIXED = 0, SIMPLE = 1, ACTUATED = 2 };

struct Mech {
  int n = 0;
  uint32_t adj[MAXJ];  // neighbour bitmask
  int8_t type[MAXJ];
};

Mech initial() {
  Mech m;
  m.n = 3;
  std::memset(m.adj, 0, sizeof(m.adj));
  m.adj[0] = 1u << 1;
  m.adj[1] = 1u << 0;
  m.type[0] = FIXED;
  m.type[1] = ACTUATED;
  m.type[2] = FIXED;
  return m;
}

// _grow_topology (generator.py:156-197); false on a dead end
bool grow(Pcg64& rng, int n, double ngp, Mech& m) {
  m = initial();
  uint32_t term = (1u << 1) | (1u << 2);
  std::vector<std::pair<int, int>> pairs;
  while (m.n < n) {
    const int left = n - m.n;
    const int slack = left - __builtin_popcount(term) + 1;
    if (slack < 0) return false;
    if (slack >= 2 && rng.random() < ngp) {
      m.adj[m.n] = 0;
      m.type[m.n] = FIXED;
      term |= 1u << m.n;
      ++m.n;
      continue;
    }
    const int tmin = slack >= 2 ? 0 : 2 - slack;
    const bool last = left == 1;
    pairs.clear();
    for (int i = 0; i < m.n; ++i)
      for (int j = i + 1; j < m.n; ++j) {
        const bool fi = m.type[i] == FIXED, fj = m.type[j] == FIXED;
        if (fi && fj) continue;
        if (last && (fi || fj)) continue;
        const int t = ((term >> i) & 1) + ((term >> j) & 1);
        if (t < tmin) continue;
        pairs.emplace_back(i, j);
      }
    if (pairs.empty()) return false;
    const auto pr = pairs[(size_t)rng.integers(0, (int64_t)pairs.size())];
    const int k = m.n;
    m.adj[k] = (1u << pr.first) | (1u << pr.second);
    m.adj[pr.first] |= 1u << k;
    m.adj[pr.second] |= 1u << k;
    m.type[k] = SIMPLE;
    term &= ~((1u << pr.first) | (1u << pr.second));
    term |= 1u << k;
    ++m.n;
  }
  return true;
}

struct Plan {
  int ns = 0;
  int8_t st[LA_MAX_STEPS][3];
};

// compile_plan walk (solver.py:71-94): false if not solvable / too long
bool compile(const Mech& m, Plan& p) {
  uint32_t known = 1u << 1;
  for (int k = 0; k < m.n; ++k)
    if (m.type[k] == FIXED) known |= 1u << k;
  std::vector<int> pending;
  for (int k = 0; k < m.n; ++k)
    if (!((known >> k) & 1)) pending.push_back(k);
  p.ns = 0;
  while (!pending.empty()) {
    bool moved = false;
    std::vector<int> rest;
    for (int k : pending) {
      const uint32_t kn = m.adj[k] & known;
      if (__builtin_popcount(kn) >= 2) {
        if (p.ns >= LA_MAX_STEPS) return false;
        const int a = __builtin_ctz(kn);
        const int b = __builtin_ctz(kn & (kn - 1));
        p.st[p.ns][0] = (int8_t)k;
        p.st[p.ns][1] = (int8_t)a;
        p.st[p.ns][2] = (int8_t)b;
        ++p.ns;
        known |= 1u << k;
        moved = true;
      } else {
        rest.push_back(k);
      }
    }
    if (!moved) return false;
    pending.swap(rest);
  }
  return true;
}

// |plan_ancestry(plan, joint)| (curves.py:132-150)
int ancestry_size(const Plan& p, int joint) {
  int pa[MAXJ], pb[MAXJ];
  for (int i = 0; i < MAXJ; ++i) pa[i] = pb[i] = -1;
  for (int s = 0; s < p.ns; ++s) {
    pa[p.st[s][0]] = p.st[s][1];
    pb[p.st[s][0]] = p.st[s][2];
  }
  uint32_t seen = 0;
  int stack[4 * MAXJ], sp = 0;
  stack[sp++] = joint;
  while (sp) {
    const int k = stack[--sp];
    if ((seen >> k) & 1) continue;
    seen |= 1u << k;
    if (pa[k] >= 0) {
      stack[sp++] = pa[k];
      stack[sp++] = pb[k];
    } else if (k == 1) {
      stack[sp++] = 0;
    }
  }
  seen |= 3u;
  return __builtin_popcount(seen);
}

// sample_topology (generator.py:200-222)
bool sample_topology(Pcg64& rng, int n, double ngp, int retries, Mech& m, Plan& p) {
  for (int r = 0; r < retries; ++r) {
    if (!grow(rng, n, ngp, m)) continue;
    if (!compile(m, p)) continue;
    if (p.ns == 0) continue;
    const int last = p.st[p.ns - 1][0];
    bool fixed_nb = false;
    for (int v = 0; v < m.n; ++v)
      if (((m.adj[last] >> v) & 1) && m.type[v] == FIXED) fixed_nb = true;
    if (fixed_nb) continue;
    if (ancestry_size(p, last) != n) continue;
    return true;
  }
  return false;
}

template <typename F>
void parallel_for(int64_t G, int threads, F f) {
  if (threads <= 1 || G < 2) {
    for (int64_t g = 0; g < G; ++g) f(g);
    return;
  }
  std::vector<std::thread> ts;
  const int T = (int)std::min<int64_t>(threads, G);
  for (int t = 0; t < T; ++t)
    ts.emplace_back([&, t] {
      for (int64_t g = t; g < G; g += T) f(g);
    });
  for (auto& th : ts) th.join();
}

}  // namespace

extern "C" {

int la_sample_topologies(int64_t seed, int64_t g0, int64_t G, int32_t n_lo, int32_t n_hi, double ng_prob,
                         int32_t retries, int32_t threads, la_plan* plans, int8_t* types, uint8_t* adj,
                         int32_t* n_out) {
  if (G < 0 || n_lo < 4 || n_hi < n_lo || n_hi > LA_MAX_JOINTS || !plans || !n_out || retries < 1 || seed < 0 ||
      g0 < 0) {
    la::set_error("la_sample_topologies: bad arguments");
    return LA_EINVAL;
  }
  std::vector<int> bad(G > 0 ? G : 1, 0);
  parallel_for(G, threads, [&](int64_t g) {
    Pcg64 rng = stream(seed, g0 + g, 0);
    const int n = (int)rng.integers(n_lo, (int64_t)n_hi + 1);
    Mech m;
    Plan p;
    if (!sample_topology(rng, n, ng_prob, retries, m, p)) {
      bad[g] = 1;
      return;
    }
    la_plan rec;
    std::memset(&rec, 0, sizeof(rec));
    rec.n = (int16_t)m.n;
    rec.nsteps = (int16_t)p.ns;
    uint32_t fm = 0;
    for (int k = 0; k < m.n; ++k)
      if (m.type[k] == FIXED) fm |= 1u << k;
    rec.fixed_mask = fm;
    for (int s = 0; s < p.ns; ++s)
      for (int c = 0; c < 3; ++c) rec.step[s][c] = p.st[s][c];
    plans[g] = rec;
    n_out[g] = m.n;
    if (types)
      for (int k = 0; k < LA_MAX_JOINTS; ++k) types[g * LA_MAX_JOINTS + k] = k < m.n ? m.type[k] : (int8_t)-1;
    if (adj)
      for (int i = 0; i < LA_MAX_JOINTS; ++i)
        for (int j = 0; j < LA_MAX_JOINTS; ++j)
          adj[(g * LA_MAX_JOINTS + i) * LA_MAX_JOINTS + j] =
              (i < m.n && j < m.n) ? (uint8_t)((m.adj[i] >> j) & 1u) : 0;
  });
  for (int64_t g = 0; g < G; ++g)
    if (bad[g]) {
      la::set_error("la_sample_topologies: no valid topology for group %lld", (long long)(g0 + g));
      return LA_ERANGE;
    }
  return 0;
}

int la_sample_poses(int64_t seed, int64_t g0, int64_t G, int32_t per_group, const int32_t* n_of_group,
                    int32_t stride, int32_t threads, double* pos) {
  if (G < 0 || per_group < 0 || !n_of_group || !pos || stride < 2 || seed < 0 || g0 < 0) {
    la::set_error("la_sample_poses: bad arguments");
    return LA_EINVAL;
  }
  for (int64_t g = 0; g < G; ++g)
    if (n_of_group[g] < 2 || n_of_group[g] > stride) {
      la::set_error("la_sample_poses: n=%d does not fit stride %d", n_of_group[g], stride);
      return LA_EINVAL;
    }
  parallel_for(G, threads, [&](int64_t g) {
    Pcg64 rng = stream(seed, g0 + g, 1);
    const int n = n_of_group[g];
    double* base = pos + (size_t)g * per_group * stride * 2;
    for (int c = 0; c < per_group; ++c) {
      double* row = base + (size_t)c * stride * 2;
      for (int j = 0; j < n; ++j) {
        row[2 * j] = rng.random();
        row[2 * j + 1] = rng.random();
      }
      row[0] = 0.5;  // ARM_PIVOT (generator.py:236-237)
      row[1] = 0.5;
      row[2] = 0.55;  // ARM_TIP
      row[3] = 0.5;
      for (int j = n; j < stride; ++j) row[2 * j] = row[2 * j + 1] = NAN;
    }
  });
  return 0;
}

// raw stream access for the parity tests: n doubles / ints of
// default_rng(entropy) where entropy = [e0, e1, e2][:n_ent]
int la_rng_draw(const int64_t* entropy, int32_t n_ent, int32_t kind, int64_t bound, int64_t count,
                double* out_d, int64_t* out_i) {
  std::vector<uint32_t> e;
  for (int i = 0; i < n_ent; ++i) int_words((uint64_t)entropy[i], e);
  Pcg64 r(e);
  for (int64_t i = 0; i < count; ++i) {
    if (kind == 0) out_d[i] = r.random();
    else out_i[i] = r.integers(0, bound);
  }
  return 0;
}

}  // extern "C"
