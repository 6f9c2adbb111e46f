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
#include <mutex>
#include <exception>
#include <cmath>
#include <cstdint>
#include <cstdio>
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
  Pcg64() : state(0), inc(1) {}
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
  // jump the LCG ahead by `delta` steps (square-and-multiply on the affine map)
  void advance(u128 delta) {
    u128 cm = PCG_MULT, cp = inc, am = 1, ap = 0;
    while (delta) {
      if (delta & 1u) {
        am *= cm;
        ap = ap * cm + cp;
      }
      cp = (cm + 1) * cp;
      cm *= cm;
      delta >>= 1;
    }
    state = am * state + ap;
  }
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
  // exception-safe: a worker's exception is rethrown on the calling thread
  // (then turned into LA_EHOST at the C ABI), a failed thread creation
  // joins the workers already started
  std::vector<std::thread> ts;
  const int T = (int)std::min<int64_t>(threads, G);
  std::exception_ptr err;
  std::mutex mu;
  auto work = [&](int t) {
    try {
      for (int64_t g = t; g < G; g += T) f(g);
    } catch (...) {
      std::lock_guard<std::mutex> lock(mu);
      if (!err) err = std::current_exception();
    }
  };
  try {
    for (int t = 0; t < T; ++t) ts.emplace_back(work, t);
  } catch (...) {
    for (auto& th : ts) th.join();
    throw;
  }
  for (auto& th : ts) th.join();
  if (err) std::rethrow_exception(err);
}

}  // namespace

// C-ABI guard: no C++ exception (allocation, thread creation) may cross
// into the caller; it becomes LA_EHOST (or a null engine) + la_last_error
#define LA_HOST_TRY try {
#define LA_HOST_CATCH(err)                                         \
  }                                                                \
  catch (const std::exception& e) {                                \
    la::set_error("%s: %s", __func__, e.what());                   \
    return err;                                                    \
  }                                                                \
  catch (...) {                                                    \
    la::set_error("%s: unknown host exception", __func__);         \
    return err;                                                    \
  }

extern "C" {

int la_sample_topologies(int64_t seed, int64_t g0, int64_t G, int32_t n_lo, int32_t n_hi, double ng_prob,
                         int32_t retries, int32_t threads, la_plan* plans, int8_t* types, uint8_t* adj,
                         int32_t* n_out) {
  LA_HOST_TRY
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
  LA_HOST_CATCH(LA_EHOST)
}

int la_sample_poses(int64_t seed, int64_t g0, int64_t G, int32_t per_group, const int32_t* n_of_group,
                    int32_t stride, int32_t threads, double* pos) {
  LA_HOST_TRY
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
  LA_HOST_CATCH(LA_EHOST)
}

// raw stream access for the parity tests: n doubles / ints of
// default_rng(entropy) where entropy = [e0, e1, e2][:n_ent]
int la_rng_draw(const int64_t* entropy, int32_t n_ent, int32_t kind, int64_t bound, int64_t count,
                double* out_d, int64_t* out_i) {
  LA_HOST_TRY
  std::vector<uint32_t> e;
  for (int i = 0; i < n_ent; ++i) int_words((uint64_t)entropy[i], e);
  Pcg64 r(e);
  for (int64_t i = 0; i < count; ++i) {
    if (kind == 0) out_d[i] = r.random();
    else out_i[i] = r.integers(0, bound);
  }
  return 0;
  LA_HOST_CATCH(LA_EHOST)
}

}  // extern "C"

// ===========================================================================
// Dataset-generation engine: GenerationRun / _generate_slot /
// find_valid_variant (generator.py:241-375) with the two-fidelity gate
// evaluated on the GPU.  The host engine owns every slot's three PCG64
// streams (topology, poses, negatives) and replays the reference control
// flow exactly; the device only answers "T_low lock step / valid at T_high"
// for look-ahead windows of candidate batches drawn from a COPY of each
// slot's pose stream (the real stream advances only by what the reference
// consumes).
// ===========================================================================
namespace {

struct Accepted {
  double pos[LA_MAX_JOINTS][2];
  int64_t attempts;
};

struct Batch {
  int64_t first = 0;  // index of its first candidate in the window
  int k = 0;          // candidates
  Pcg64 start;        // pose stream state before drawing it
  Pcg64 after;        // pose stream state after drawing it
  explicit Batch(const Pcg64& r) : start(r), after(r) {}
};

struct Slot {
  int64_t id;
  Pcg64 topo, pos, neg;
  int n = 0;
  Mech mech;
  Plan plan;
  int state = 0;           // 0 need topology, 1 searching, 2 done, 3 failed
  int tries = 0;           // topologies sampled
  int64_t consumed = 0;    // candidates consumed by the current variant
  std::vector<Accepted> acc;
  std::vector<Batch> win;  // current look-ahead window
  int64_t plan_slot = -1;  // plan index of this slot in the last window
  int64_t sim = 0, nacc = 0, disc = 0;  // GenerationStats tallies of this slot (joint count n)
  Slot(int64_t s, int64_t seed) : id(s), topo(stream(seed, s, 0)), pos(stream(seed, s, 1)), neg(stream(seed, s, 2)) {}
};

struct Record {
  int64_t slot, variant, attempts;
  Mech mech;
  Plan plan;
  double pos[LA_MAX_JOINTS][2];
};

struct Negative {
  int64_t slot, step;
  Mech mech;
  double pos[LA_MAX_JOINTS][2];
};

struct Engine {
  la_gen_cfg cfg;
  std::vector<Slot> slots;
  std::vector<std::vector<Record>> slot_records;
  std::vector<std::vector<Negative>> slot_negs;
  int error = 0;
  char err[200] = "";
};

void draw_pose(Pcg64& r, int n, double* row /* [20][2] */) {
  for (int j = 0; j < n; ++j) {
    row[2 * j] = r.random();
    row[2 * j + 1] = r.random();
  }
  row[0] = 0.5;
  row[1] = 0.5;
  row[2] = 0.55;
  row[3] = 0.5;
  for (int j = n; j < LA_MAX_JOINTS; ++j) row[2 * j] = row[2 * j + 1] = NAN;
}

la_plan to_rec(const Mech& m, const Plan& p) {
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
  return rec;
}

// next topology of a slot (sample_topology on the slot's topology stream)
bool next_topology(Engine& E, Slot& S) {
  if (S.tries >= E.cfg.retries) return false;
  ++S.tries;
  if (!sample_topology(S.topo, S.n, E.cfg.ng_prob, E.cfg.retries, S.mech, S.plan)) return false;
  S.acc.clear();
  S.consumed = 0;
  S.win.clear();
  S.state = 1;
  return true;
}

int batch_size(const Engine& E, int64_t consumed) {
  const int64_t left = E.cfg.max_attempts - consumed;
  return (int)(left < E.cfg.batch ? left : E.cfg.batch);
}

// Lay out the next look-ahead window: for every searching slot, up to
// `lookahead` consecutive batches of its current variant schedule (batch
// states chained from the slot's real pose stream).  Slots that would
// overflow `cap` wait for the next window.  Returns the candidate count, 0
// when every slot is done, <0 on error.
int64_t layout(Engine& E, int32_t lookahead, int64_t cap, la_plan* plans, int32_t* n_plans,
               std::vector<Slot*>& act) {
  if (E.error) {
    la::set_error("%s", E.err);
    return E.error;
  }
  if (lookahead < 1) lookahead = 1;
  int64_t total = 0;
  int np = 0;
  for (auto& S : E.slots) {
    S.win.clear();
    if (S.state != 1) continue;
    int64_t consumed = S.consumed, need = 0;
    std::vector<Batch> w;
    Pcg64 r = S.pos;
    for (int i = 0; i < lookahead; ++i) {
      const int k = batch_size(E, consumed);
      if (k <= 0) break;
      Batch b(r);
      b.first = total + need;
      b.k = k;
      r.advance((u128)k * (u128)(2 * S.n));
      w.push_back(b);
      need += k;
      consumed += k;
    }
    if (total + need > cap) {
      if (total > 0) break;
      la::set_error("la_gen_window: one window (%lld) exceeds cap %lld", (long long)need, (long long)cap);
      return LA_EWS;
    }
    if (!plans) {
      la::set_error("la_gen_window: null plan table");
      return LA_EINVAL;
    }
    S.plan_slot = np;
    plans[np++] = to_rec(S.mech, S.plan);
    S.win.swap(w);
    act.push_back(&S);
    total += need;
  }
  *n_plans = np;
  return total;
}

}  // namespace

extern "C" {

void* la_gen_create(const la_gen_cfg* cfg, int64_t slot0, int64_t n_slots) {
  LA_HOST_TRY
  if (!cfg || n_slots < 0 || cfg->n_min < 4 || cfg->n_max < cfg->n_min || cfg->n_max > LA_MAX_JOINTS ||
      cfg->variants < 1 || cfg->batch < 1 || cfg->max_attempts < 1 || cfg->retries < 1 || cfg->seed < 0) {
    la::set_error("la_gen_create: bad configuration");
    return nullptr;
  }
  Engine* E = new Engine();
  E->cfg = *cfg;
  E->slots.reserve((size_t)n_slots);
  for (int64_t s = 0; s < n_slots; ++s) E->slots.emplace_back(slot0 + s, cfg->seed);
  // first topology of every slot (independent streams: host threads)
  parallel_for(n_slots, cfg->threads, [&](int64_t s) {
    Slot& S = E->slots[(size_t)s];
    S.n = (int)S.topo.integers(cfg->n_min, (int64_t)cfg->n_max + 1);
    if (!next_topology(*E, S)) S.state = 3;
  });
  E->slot_records.resize((size_t)n_slots);
  E->slot_negs.resize((size_t)n_slots);
  for (auto& S : E->slots)
    if (S.state == 3) {
      E->error = LA_ERANGE;
      snprintf(E->err, sizeof(E->err), "slot %lld: no valid topology with n=%d", (long long)S.id, S.n);
    }
  return E;
  LA_HOST_CATCH(nullptr)
}

void la_gen_destroy(void* h) { delete static_cast<Engine*>(h); }

// Draw the next look-ahead window: for every searching slot, up to
// `lookahead` consecutive batches of its current variant schedule, drawn from
// a copy of its pose stream.  Writes poses [cand][20][2], the plan index of
// each candidate and the plan table (one record per slot in the window).
// Slots that would overflow `cap` wait for the next window.  Returns the
// candidate count, 0 when every slot is done, <0 on error.
int64_t la_gen_window(void* h, int32_t lookahead, int64_t cap, int32_t threads, double* pos, int32_t* cand_plan,
                      la_plan* plans, int32_t* n_plans) {
  LA_HOST_TRY
  if (!h || !n_plans) {
    la::set_error("la_gen_window: null argument");
    return LA_EINVAL;
  }
  Engine& E = *static_cast<Engine*>(h);
  std::vector<Slot*> act;
  const int64_t total = layout(E, lookahead, cap, plans, n_plans, act);
  if (total <= 0) return total;
  if (!pos || !cand_plan) {
    la::set_error("la_gen_window: null pose buffer");
    return LA_EINVAL;
  }
  parallel_for((int64_t)act.size(), threads, [&](int64_t a) {
    Slot& S = *act[a];
    Pcg64 r = S.pos;
    for (auto& b : S.win) {
      for (int c = 0; c < b.k; ++c) {
        const int64_t off = b.first + c;
        draw_pose(r, S.n, pos + (size_t)off * LA_MAX_JOINTS * 2);
        cand_plan[off] = (int32_t)S.plan_slot;
      }
      b.after = r;
    }
  });
  return total;
  LA_HOST_CATCH(LA_EHOST)
}

// Same window, drawn on the device: one descriptor per batch (its pose
// stream state, first candidate, size, joint count, plan index) for
// la_gen_poses.  Candidate c of a batch uses stream draws [2nc, 2n(c+1)).
int64_t la_gen_window_dev(void* h, int32_t lookahead, int64_t cap, la_gen_batch* batches, int64_t max_batches,
                          int64_t* n_batches, la_plan* plans, int32_t* n_plans) {
  LA_HOST_TRY
  if (!h || !n_batches || !n_plans) {
    la::set_error("la_gen_window_dev: null argument");
    return LA_EINVAL;
  }
  Engine& E = *static_cast<Engine*>(h);
  std::vector<Slot*> act;
  const int64_t total = layout(E, lookahead, cap, plans, n_plans, act);
  if (total <= 0) return total;
  if (!batches) {
    la::set_error("la_gen_window_dev: null descriptor buffer");
    return LA_EINVAL;
  }
  int64_t nb = 0;
  for (Slot* S : act)
    for (auto& b : S->win) {
      if (nb >= max_batches) {
        la::set_error("la_gen_window_dev: more than %lld batches", (long long)max_batches);
        return LA_EWS;
      }
      la_gen_batch& d = batches[nb++];
      d.state_hi = (uint64_t)(b.start.state >> 64);
      d.state_lo = (uint64_t)b.start.state;
      d.inc_hi = (uint64_t)(b.start.inc >> 64);
      d.inc_lo = (uint64_t)b.start.inc;
      d.first = b.first;
      d.k = b.k;
      d.n = S->n;
      d.plan = (int32_t)S->plan_slot;
      d._pad = 0;
      b.after = b.start;
      b.after.advance((u128)b.k * (u128)(2 * S->n));
    }
  *n_batches = nb;
  return total;
  LA_HOST_CATCH(LA_EHOST)
}

// Walk the device flags of the last window in each slot's stream order:
// first_t[c] == T_high -> valid; low_t[c] >= 0 -> locked at T_low (step).
int la_gen_consume(void* h, const double* pos, const int32_t* first_t, const int32_t* low_t) {
  LA_HOST_TRY
  if (!h || !first_t || !low_t) {
    la::set_error("la_gen_consume: null argument");
    return LA_EINVAL;
  }
  Engine& E = *static_cast<Engine*>(h);
  const la_gen_cfg& cfg = E.cfg;
  // pose of candidate c of batch b: from the window buffer, or redrawn from
  // the batch's stream state (device-drawn windows)
  auto pose = [&](const Slot& S, const Batch& b, int c, double* row) {
    if (pos) {
      std::memcpy(row, pos + (size_t)(b.first + c) * LA_MAX_JOINTS * 2, sizeof(double) * LA_MAX_JOINTS * 2);
      return;
    }
    Pcg64 r = b.start;
    r.advance((u128)c * (u128)(2 * S.n));
    draw_pose(r, S.n, row);
  };
  // slots are independent: walk them in parallel, each in its own stream order
  parallel_for((int64_t)E.slots.size(), cfg.threads, [&](int64_t si) {
    Slot& S = E.slots[(size_t)si];
    if (S.state != 1 || S.win.empty()) return;
    size_t used = 0;  // batches fully consumed
    bool restart_window = false;
    for (size_t bi = 0; bi < S.win.size() && S.state == 1 && !restart_window; ++bi) {
      const Batch& b = S.win[bi];
      if (b.k != batch_size(E, S.consumed)) {  // schedule changed (new variant near the cap)
        restart_window = true;
        break;
      }
      int hit = -1;
      for (int c = 0; c < b.k; ++c) {
        const int64_t g = b.first + c;
        if (low_t[g] >= 0) {  // T_low lock: negative sample draw (generator.py:267-272)
          if (cfg.negative_rate > 0.0 && S.neg.random() < cfg.negative_rate) {
            Negative ng;
            ng.slot = S.id;
            ng.step = low_t[g];
            ng.mech = S.mech;
            pose(S, b, c, &ng.pos[0][0]);
            E.slot_negs[(size_t)si].push_back(ng);
          }
          continue;
        }
        if (first_t[g] != cfg.T_high) continue;
        hit = c;
        break;
      }
      S.pos = b.after;  // the reference draws whole batches
      ++used;
      if (hit >= 0) {
        Accepted a;
        pose(S, b, hit, &a.pos[0][0]);
        a.attempts = S.consumed + hit + 1;
        S.acc.push_back(a);
        S.consumed = 0;
        if ((int)S.acc.size() == cfg.variants) {
          for (size_t v = 0; v < S.acc.size(); ++v) {
            Record r;
            r.slot = S.id;
            r.variant = (int64_t)v;
            r.attempts = S.acc[v].attempts;
            r.mech = S.mech;
            r.plan = S.plan;
            std::memcpy(r.pos, S.acc[v].pos, sizeof(r.pos));
            E.slot_records[(size_t)si].push_back(r);
            S.sim += r.attempts;
            S.nacc += 1;
          }
          S.state = 2;
        }
        continue;  // next variant continues on the next batch of the window
      }
      S.consumed += b.k;
      if (S.consumed >= cfg.max_attempts) {  // variant failed: discard topology (generator.py:318-320)
        int64_t wasted = cfg.max_attempts;
        for (auto& a : S.acc) wasted += a.attempts;
        S.sim += wasted;
        S.disc += 1;
        if (!next_topology(E, S)) S.state = 3;
        restart_window = true;  // next_topology cleared the window
      }
    }
    (void)used;
    S.win.clear();  // unconsumed look-ahead is dropped; the real stream sits after the last consumed batch
  });
  for (auto& S : E.slots)
    if (S.state == 3 && !E.error) {
      E.error = LA_ERANGE;
      snprintf(E.err, sizeof(E.err), "slot %lld: no topology with feasible variants (n=%d)", (long long)S.id, S.n);
    }
  if (E.error) {
    la::set_error("%s", E.err);
    return E.error;
  }
  return 0;
  LA_HOST_CATCH(LA_EHOST)
}

int64_t la_gen_count(void* h, int32_t what) {
  LA_HOST_TRY
  if (!h) {
    la::set_error("la_gen_count: null engine");
    return LA_EINVAL;
  }
  Engine& E = *static_cast<Engine*>(h);
  int64_t n = 0;
  if (what == 0)
    for (auto& v : E.slot_records) n += (int64_t)v.size();
  else
    for (auto& v : E.slot_negs) n += (int64_t)v.size();
  return n;
  LA_HOST_CATCH(LA_EHOST)
}

// records in slot order: meta [R][4] (slot, variant, attempts, n), poses
// [R][20][2], plans [R], adjacency [R][20][20], types [R][20]
int la_gen_records(void* h, int64_t* meta, double* pos, la_plan* plans, uint8_t* adj, int8_t* types) {
  LA_HOST_TRY
  if (!h || !meta || !pos || !plans || !adj || !types) {
    la::set_error("la_gen_records: null argument");
    return LA_EINVAL;
  }
  Engine& E = *static_cast<Engine*>(h);
  int64_t r = 0;
  for (auto& v : E.slot_records)
    for (auto& rec : v) {
      meta[4 * r] = rec.slot;
      meta[4 * r + 1] = rec.variant;
      meta[4 * r + 2] = rec.attempts;
      meta[4 * r + 3] = rec.mech.n;
      std::memcpy(pos + (size_t)r * LA_MAX_JOINTS * 2, rec.pos, sizeof(rec.pos));
      plans[r] = to_rec(rec.mech, rec.plan);
      for (int i = 0; i < LA_MAX_JOINTS; ++i) {
        types[r * LA_MAX_JOINTS + i] = i < rec.mech.n ? rec.mech.type[i] : (int8_t)-1;
        for (int j = 0; j < LA_MAX_JOINTS; ++j)
          adj[(r * LA_MAX_JOINTS + i) * LA_MAX_JOINTS + j] =
              (i < rec.mech.n && j < rec.mech.n) ? (uint8_t)((rec.mech.adj[i] >> j) & 1u) : 0;
      }
      ++r;
    }
  return 0;
  LA_HOST_CATCH(LA_EHOST)
}

// negatives in slot order: meta [R][3] (slot, locking step, n), poses [R][20][2]
int la_gen_negatives(void* h, int64_t* meta, double* pos, uint8_t* adj, int8_t* types) {
  LA_HOST_TRY
  if (!h || !meta || !pos || !adj || !types) {
    la::set_error("la_gen_negatives: null argument");
    return LA_EINVAL;
  }
  Engine& E = *static_cast<Engine*>(h);
  int64_t r = 0;
  for (auto& v : E.slot_negs)
    for (auto& ng : v) {
      meta[3 * r] = ng.slot;
      meta[3 * r + 1] = ng.step;
      meta[3 * r + 2] = ng.mech.n;
      std::memcpy(pos + (size_t)r * LA_MAX_JOINTS * 2, ng.pos, sizeof(ng.pos));
      for (int i = 0; i < LA_MAX_JOINTS; ++i) {
        types[r * LA_MAX_JOINTS + i] = i < ng.mech.n ? ng.mech.type[i] : (int8_t)-1;
        for (int j = 0; j < LA_MAX_JOINTS; ++j)
          adj[(r * LA_MAX_JOINTS + i) * LA_MAX_JOINTS + j] =
              (i < ng.mech.n && j < ng.mech.n) ? (uint8_t)((ng.mech.adj[i] >> j) & 1u) : 0;
      }
      ++r;
    }
  return 0;
  LA_HOST_CATCH(LA_EHOST)
}

// stats: out [21][2] simulated / accepted by joint count; *discarded
int la_gen_stats(void* h, int64_t* out, int64_t* discarded) {
  LA_HOST_TRY
  if (!h || !out || !discarded) {
    la::set_error("la_gen_stats: null argument");
    return LA_EINVAL;
  }
  Engine& E = *static_cast<Engine*>(h);
  for (int n = 0; n <= LA_MAX_JOINTS; ++n) out[2 * n] = out[2 * n + 1] = 0;
  int64_t disc = 0;
  for (auto& S : E.slots) {
    out[2 * S.n] += S.sim;
    out[2 * S.n + 1] += S.nacc;
    disc += S.disc;
  }
  *discarded = disc;
  return 0;
  LA_HOST_CATCH(LA_EHOST)
}

}  // extern "C"

// Moving-joint curve enumeration of a generated block (cli.normalize order,
// cli.py:124-136): records in order, non-Fixed joints ascending; row into
// the packed trajectory block, mech id slot * variants + variant, is_arc =
// any Fixed neighbour (curves.py:87-92).  Returns the curve count; outputs
// may be NULL to count only.
extern "C" int64_t la_moving_joints(const int64_t* meta /* [R][4] */, const int8_t* types /* [R][20] */,
                                    const uint8_t* adj /* [R][20][20] */, const int64_t* row0, int64_t R,
                                    int32_t variants, int64_t* rows, int64_t* mech_ids, int64_t* joint_ids,
                                    uint8_t* is_arc) {
  int64_t c = 0;
  for (int64_t r = 0; r < R; ++r) {
    const int n = (int)meta[4 * r + 3];
    const int8_t* ty = types + r * LA_MAX_JOINTS;
    uint8_t fixed[LA_MAX_JOINTS];  // 1 for Fixed joints < n (fixed-length: the arc test vectorises)
    for (int k = 0; k < LA_MAX_JOINTS; ++k) fixed[k] = (k < n && ty[k] == 0) ? 1 : 0;
    const int64_t base = row0[r], mid = meta[4 * r] * variants + meta[4 * r + 1];
    for (int j = 0; j < n; ++j) {
      if (ty[j] == 0) continue;
      if (rows) {
        const uint8_t* a = adj + (r * LA_MAX_JOINTS + j) * LA_MAX_JOINTS;
        uint8_t acc = 0;
        for (int k = 0; k < LA_MAX_JOINTS; ++k) acc |= (uint8_t)(a[k] & fixed[k]);
        rows[c] = base + j;
        mech_ids[c] = mid;
        joint_ids[c] = j;
        is_arc[c] = acc ? 1 : 0;
      }
      ++c;
    }
  }
  return c;
}

// One sample_topology(rng, n, ng_probability, retries) draw
// (generator.py:200-222) on a caller's numpy PCG64 bit generator: st =
// {state hi, state lo, inc hi, inc lo} (64-bit words), buf = {has_uint32,
// uinteger}, both advanced in place exactly as the reference's draws advance
// the Generator.  Writes the topology (n, types [20], adj [20][20]) and its
// compiled plan record.  LA_ERANGE when every retry fails (GenerationError).
extern "C" int la_sample_topology_rng(uint64_t* st, uint32_t* buf, int32_t n, double ng_prob, int32_t retries,
                                      la_plan* plan, int8_t* types, uint8_t* adj) {
  LA_HOST_TRY
  if (!st || !buf || !plan || !types || !adj || n < 4 || n > LA_MAX_JOINTS || retries < 1) {
    la::set_error("la_sample_topology_rng: bad arguments");
    return LA_EINVAL;
  }
  Pcg64 rng;
  rng.state = ((u128)st[0] << 64) | st[1];
  rng.inc = ((u128)st[2] << 64) | st[3];
  rng.has32 = (int)buf[0];
  rng.u32 = buf[1];
  Mech m;
  Plan pl;
  const bool ok = sample_topology(rng, n, ng_prob, retries, m, pl);
  st[0] = (uint64_t)(rng.state >> 64);
  st[1] = (uint64_t)rng.state;
  buf[0] = (uint32_t)rng.has32;
  buf[1] = rng.u32;
  if (!ok) {
    la::set_error("no valid topology with n=%d after %d tries", n, retries);
    return LA_ERANGE;
  }
  *plan = to_rec(m, pl);
  for (int k = 0; k < LA_MAX_JOINTS; ++k) types[k] = k < m.n ? m.type[k] : (int8_t)-1;
  for (int i = 0; i < LA_MAX_JOINTS; ++i)
    for (int j = 0; j < LA_MAX_JOINTS; ++j)
      adj[i * LA_MAX_JOINTS + j] = (i < m.n && j < m.n) ? (uint8_t)((m.adj[i] >> j) & 1u) : 0;
  return 0;
  LA_HOST_CATCH(LA_EHOST)
}
