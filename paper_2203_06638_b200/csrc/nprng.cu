// nprng.cu — the reference's host sampling stream in native code.
//
// The reference draws every updater's minibatches (and, in record modes
// other than "full", 16 sampled tag indices first) from
// numpy.random.default_rng(SeedSequence([seed, q, rank])) (engine.py:293,
// 343-351; objectives.py:70-104).  To run those configurations in the
// native updater loop with the SAME batches, this file restates the pieces
// of numpy (2.x) that stream goes through, bit for bit:
//   SeedSequence(entropy).generate_state(4, uint64)   (hashmix pool, 4 words)
//   PCG64 seeding and next64 / next32 (XSL-RR 128/64, 32-bit halves cached)
//   Generator.integers(0, n, B)          (Lemire bounded ints, 32/64 bit)
//   Generator.choice(d, k, replace=False) (tail shuffle or Floyd + shuffle,
//                                          Lemire-bounded swaps)
//   Generator.permutation(m)              (Fisher-Yates, random_interval swaps)
// tests/test_native_cpu.py checks every entry point against numpy itself.
// Host code only (no kernels): the C ABI exposes it for the tests and the
// updater loop uses it directly.

#include "common.cuh"

#include <cstdint>
#include <cstring>
#include <vector>

namespace nprng {

typedef unsigned __int128 u128;

// ---- SeedSequence (numpy/random/bit_generator.pyx) ------------------------
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
constexpr int kXShift = 16, kPool = 4;

static inline uint32_t hashmix(uint32_t v, uint32_t* hc) {
  v ^= *hc;
  *hc *= kMultA;
  v *= *hc;
  v ^= v >> kXShift;
  return v;
}
static inline uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  r ^= r >> kXShift;
  return r;
}

// entropy: Python ints -> little-endian 32-bit words each (0 -> one word)
static void entropy_words(const uint64_t* ints, int n, std::vector<uint32_t>* out) {
  for (int i = 0; i < n; ++i) {
    uint64_t v = ints[i];
    if (v == 0) {
      out->push_back(0);
      continue;
    }
    while (v) {
      out->push_back((uint32_t)(v & 0xffffffffu));
      v >>= 32;
    }
  }
}

static void seedseq_state(const std::vector<uint32_t>& ent, uint32_t* words, int nwords) {
  uint32_t pool[kPool];
  uint32_t hc = kInitA;
  for (int i = 0; i < kPool; ++i) pool[i] = hashmix(i < (int)ent.size() ? ent[i] : 0u, &hc);
  for (int s = 0; s < kPool; ++s)
    for (int d = 0; d < kPool; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], &hc));
  for (int s = kPool; s < (int)ent.size(); ++s)
    for (int d = 0; d < kPool; ++d) pool[d] = mix(pool[d], hashmix(ent[s], &hc));
  uint32_t hb = kInitB;
  for (int i = 0; i < nwords; ++i) {
    uint32_t v = pool[i % kPool];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> kXShift;
    words[i] = v;
  }
}

// ---- PCG64 ------------------------------------------------------------------
static const u128 kMult = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;

struct Pcg64 {
  u128 state = 0, inc = 0;
  bool has32 = false;
  uint32_t u32 = 0;

  inline void step() { state = state * kMult + inc; }
  uint64_t next64() {
    step();
    uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    unsigned rot = (unsigned)(state >> 122);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  uint32_t next32() {
    if (has32) {
      has32 = false;
      return u32;
    }
    uint64_t v = next64();
    has32 = true;
    u32 = (uint32_t)(v >> 32);
    return (uint32_t)(v & 0xffffffffu);
  }
};

static void pcg64_seed(Pcg64* g, const uint64_t* ints, int n) {
  std::vector<uint32_t> ent;
  entropy_words(ints, n, &ent);
  uint32_t w[8];
  seedseq_state(ent, w, 8);
  uint64_t v[4];
  for (int i = 0; i < 4; ++i) v[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
  u128 initstate = ((u128)v[0] << 64) | v[1];
  u128 initseq = ((u128)v[2] << 64) | v[3];
  g->state = 0;
  g->inc = (initseq << 1) | 1;
  g->step();
  g->state += initstate;
  g->step();
  g->has32 = false;
  g->u32 = 0;
}

// ---- bounded integers (numpy/random/src/distributions) ----------------------
static uint32_t lemire32(Pcg64* g, uint32_t rng) {
  const uint32_t excl = rng + 1;
  uint64_t m = (uint64_t)g->next32() * excl;
  uint32_t left = (uint32_t)m;
  if (left < excl) {
    const uint32_t thr = (uint32_t)(0xFFFFFFFFu - rng) % excl;
    while (left < thr) {
      m = (uint64_t)g->next32() * excl;
      left = (uint32_t)m;
    }
  }
  return (uint32_t)(m >> 32);
}
static uint64_t lemire64(Pcg64* g, uint64_t rng) {
  const uint64_t excl = rng + 1;
  u128 m = (u128)g->next64() * excl;
  uint64_t left = (uint64_t)m;
  if (left < excl) {
    const uint64_t thr = (0xFFFFFFFFFFFFFFFFull - rng) % excl;
    while (left < thr) {
      m = (u128)g->next64() * excl;
      left = (uint64_t)m;
    }
  }
  return (uint64_t)(m >> 64);
}
static uint64_t bounded(Pcg64* g, uint64_t rng) {  // uniform in [0, rng]
  if (rng == 0) return 0;
  if (rng <= 0xFFFFFFFFull) {
    if (rng == 0xFFFFFFFFull) return g->next32();
    return lemire32(g, (uint32_t)rng);
  }
  if (rng == 0xFFFFFFFFFFFFFFFFull) return g->next64();
  return lemire64(g, rng);
}
static uint64_t interval(Pcg64* g, uint64_t max) {  // random_interval
  if (max == 0) return 0;
  uint64_t mask = max;
  mask |= mask >> 1;
  mask |= mask >> 2;
  mask |= mask >> 4;
  mask |= mask >> 8;
  mask |= mask >> 16;
  mask |= mask >> 32;
  uint64_t v;
  if (max <= 0xffffffffull) {
    while ((v = (g->next32() & mask)) > max) {
    }
  } else {
    while ((v = (g->next64() & mask)) > max) {
    }
  }
  return v;
}
// Fisher-Yates from the top: Generator.shuffle / permutation draw j with
// random_interval (masked rejection), choice's _shuffle_int with the Lemire
// bounded draw — two different streams, both restated
static void shuffle_int(Pcg64* g, int64_t n, int64_t first, int64_t* data, bool lemire) {
  for (int64_t i = n - 1; i >= first; --i) {
    int64_t j = (int64_t)(lemire ? bounded(g, (uint64_t)i) : interval(g, (uint64_t)i));
    int64_t t = data[j];
    data[j] = data[i];
    data[i] = t;
  }
}

}  // namespace nprng

using nprng::Pcg64;

// integers(0, n, B)
void lpp_nprng_integers_impl(Pcg64* g, int64_t n, int32_t b, int64_t* out) {
  for (int i = 0; i < b; ++i) out[i] = (int64_t)nprng::bounded(g, (uint64_t)(n - 1));
}

// choice(pop, k, replace=False) (shuffle=True)
void lpp_nprng_choice_impl(Pcg64* g, int64_t pop, int32_t k, int64_t* out) {
  const int64_t cutoff = 50;
  // numpy 2.x: a tail shuffle of arange(pop) only for large populations
  // with a large sample; Floyd's algorithm otherwise (determined against
  // numpy itself, tests/test_native_cpu.py)
  if (pop > 10000 && k > pop / cutoff) {
    std::vector<int64_t> idx(pop);
    for (int64_t i = 0; i < pop; ++i) idx[i] = i;
    int64_t first = pop - k > 1 ? pop - k : 1;
    nprng::shuffle_int(g, pop, first, idx.data(), true);
    std::memcpy(out, idx.data() + (pop - k), sizeof(int64_t) * (size_t)k);
    return;
  }
  // Floyd's algorithm over a linear-probing hash set
  uint64_t set_size = (uint64_t)(1.2 * (double)k);
  uint64_t mask = set_size;
  mask |= mask >> 1;
  mask |= mask >> 2;
  mask |= mask >> 4;
  mask |= mask >> 8;
  mask |= mask >> 16;
  mask |= mask >> 32;
  std::vector<uint64_t> hs(mask + 1, ~0ull);
  for (int64_t j = pop - k; j < pop; ++j) {
    uint64_t val = nprng::bounded(g, (uint64_t)j);
    uint64_t loc = val & mask;
    while (hs[loc] != ~0ull && hs[loc] != val) loc = (loc + 1) & mask;
    if (hs[loc] == ~0ull) {
      hs[loc] = val;
      out[j - pop + k] = (int64_t)val;
    } else {
      loc = (uint64_t)j & mask;
      while (hs[loc] != ~0ull) loc = (loc + 1) & mask;
      hs[loc] = (uint64_t)j;
      out[j - pop + k] = j;
    }
  }
  nprng::shuffle_int(g, k, 1, out, true);
}

// permutation(m)
void lpp_nprng_permutation_impl(Pcg64* g, int64_t m, int64_t* out) {
  for (int64_t i = 0; i < m; ++i) out[i] = i;
  nprng::shuffle_int(g, m, 1, out, false);
}

void lpp_nprng_free_impl(Pcg64* g) { delete g; }

Pcg64* lpp_nprng_new_impl(const uint64_t* ints, int n) {
  Pcg64* g = new Pcg64();
  nprng::pcg64_seed(g, ints, n);
  return g;
}

extern "C" int lpp_nprng_create(const uint64_t* entropy, int n, void** out) {
  if (!entropy || n <= 0 || !out) return set_err(LPP_E_VALUE, "nprng_create: empty entropy");
  *out = lpp_nprng_new_impl(entropy, n);
  return LPP_OK;
}
extern "C" int lpp_nprng_destroy(void* h) {
  delete static_cast<Pcg64*>(h);
  return LPP_OK;
}
extern "C" int lpp_nprng_integers(void* h, int64_t n, int32_t b, int64_t* out) {
  if (!h || !out || n <= 0 || b < 0) return set_err(LPP_E_VALUE, "nprng_integers: bad arguments");
  lpp_nprng_integers_impl(static_cast<Pcg64*>(h), n, b, out);
  return LPP_OK;
}
extern "C" int lpp_nprng_choice(void* h, int64_t pop, int32_t k, int64_t* out) {
  if (!h || !out || pop <= 0 || k < 0 || k > pop)
    return set_err(LPP_E_VALUE, "nprng_choice: bad arguments");
  lpp_nprng_choice_impl(static_cast<Pcg64*>(h), pop, k, out);
  return LPP_OK;
}
extern "C" int lpp_nprng_permutation(void* h, int64_t m, int64_t* out) {
  if (!h || !out || m <= 0) return set_err(LPP_E_VALUE, "nprng_permutation: bad arguments");
  lpp_nprng_permutation_impl(static_cast<Pcg64*>(h), m, out);
  return LPP_OK;
}
