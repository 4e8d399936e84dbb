// The reference's prediction model in C++ (prefetch.py:54-101): noisy ground
// truth drawn from numpy's default_rng([seed, pass, layer, 0x5EED]) stream.
// numpy 2.x algorithms restated: SeedSequence entropy mixing (hashmix/mix over
// a 4-word pool), PCG64 (XSL-RR 128/64, seeded via generate_state(4, uint64)),
// Generator.random() = (next64 >> 11) * 2^-53, Generator.integers(n) = Lemire's
// bounded draw on next_uint32 (PCG64 buffers the high half of a 64-bit draw).
// tests/test_predict_native.py checks it draw-for-draw against numpy.
#include <algorithm>
#include <cstring>
#include <utility>
#include <vector>

#include "common.hpp"

namespace hm {
namespace {

using u32 = uint32_t;
using u64 = uint64_t;
using u128 = unsigned __int128;

constexpr u32 kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u, kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr u32 kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
constexpr int kXShift = 16;

struct SeedSeq {
  u32 pool[4];
  explicit SeedSeq(const std::vector<u32> &entropy) {
    u32 hc = kInitA;
    auto hashmix = [&hc](u32 v) {
      v ^= hc;
      hc *= kMultA;
      v *= hc;
      v ^= v >> kXShift;
      return v;
    };
    auto mix = [](u32 x, u32 y) {
      u32 r = kMixL * x - kMixR * y;
      r ^= r >> kXShift;
      return r;
    };
    for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < static_cast<int>(entropy.size()) ? entropy[i] : 0u);
    for (int s = 0; s < 4; ++s)
      for (int d = 0; d < 4; ++d)
        if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
    for (size_t s = 4; s < entropy.size(); ++s)
      for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(entropy[s]));
  }
  void generate_u64(u64 *out, int n) const {
    u32 hc = kInitB;
    std::vector<u32> w(static_cast<size_t>(2 * n));
    for (int i = 0; i < 2 * n; ++i) {
      u32 v = pool[i % 4];
      v ^= hc;
      hc *= kMultB;
      v *= hc;
      v ^= v >> kXShift;
      w[i] = v;
    }
    for (int i = 0; i < n; ++i) out[i] = static_cast<u64>(w[2 * i]) | (static_cast<u64>(w[2 * i + 1]) << 32);
  }
};

struct Pcg64 {
  u128 state = 0, inc = 0;
  bool has32 = false;
  u32 buf32 = 0;
  static constexpr u128 kMult = (static_cast<u128>(0x2360ED051FC65DA4ULL) << 64) | 0x4385DF649FCCF645ULL;
  void step() { state = state * kMult + inc; }
  Pcg64(u64 s_hi, u64 s_lo, u64 i_hi, u64 i_lo) {
    const u128 s = (static_cast<u128>(s_hi) << 64) | s_lo, q = (static_cast<u128>(i_hi) << 64) | i_lo;
    state = 0;
    inc = (q << 1) | 1u;
    step();
    state += s;
    step();
  }
  u64 next64() {
    step();
    const u64 hi = static_cast<u64>(state >> 64), lo = static_cast<u64>(state);
    const unsigned rot = static_cast<unsigned>(state >> 122);
    const u64 x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  u32 next32() {
    if (has32) {
      has32 = false;
      return buf32;
    }
    const u64 v = next64();
    has32 = true;
    buf32 = static_cast<u32>(v >> 32);
    return static_cast<u32>(v);
  }
  double random() { return static_cast<double>(next64() >> 11) * (1.0 / 9007199254740992.0); }
  int64_t integers(int64_t n) {  // [0, n)
    const u64 rng = static_cast<u64>(n - 1);
    if (rng == 0) return 0;
    // n is always < 2^32 here (an expert index range)
    const u32 excl = static_cast<u32>(rng) + 1u;
    u64 m = static_cast<u64>(next32()) * excl;
    u32 left = static_cast<u32>(m);
    if (left < excl) {
      const u32 thr = static_cast<u32>((0xFFFFFFFFu - static_cast<u32>(rng)) % excl);
      while (left < thr) {
        m = static_cast<u64>(next32()) * excl;
        left = static_cast<u32>(m);
      }
    }
    return static_cast<int64_t>(m >> 32);
  }
};

std::vector<u32> entropy_words(const int64_t *vals, int n) {  // _coerce_to_uint32_array on non-negative ints
  std::vector<u32> out;
  for (int i = 0; i < n; ++i) {
    u64 v = static_cast<u64>(vals[i]);
    HM_REQUIRE(vals[i] >= 0, HM_EVALUE, "seed words must be non-negative");
    if (v == 0) out.push_back(0);
    while (v) {
      out.push_back(static_cast<u32>(v));
      v >>= 32;
    }
  }
  return out;
}

}  // namespace
}  // namespace hm

extern "C" {

// Future LayerRequests of one pass as the prediction model sees them
// (prefetch.py:54-101).  pass_loads [L*N] are the pass's true loads; the
// predicted loads of layers layer+1 .. min(layer+horizon, L-1) are written to
// out_loads [horizon*N], their layer ids to out_layers; *n_out = count.
int hm_predict_layers(const int64_t *pass_loads, int L, int N, int64_t pass_index, int layer, int64_t seed,
                      int horizon, double accuracy, int32_t *out_layers, int64_t *out_loads, int *n_out) {
  HM_API_BEGIN
  HM_REQUIRE(layer >= 0 && layer < L, HM_EVALUE, "layer out of range");
  HM_REQUIRE(horizon >= 1, HM_EVALUE, "horizon must be >= 1");
  const int last = std::min(layer + horizon, L - 1);
  const int64_t ent[4] = {seed, pass_index, layer, 0x5EED};
  hm::SeedSeq ss(hm::entropy_words(ent, 4));
  uint64_t st[4];
  ss.generate_u64(st, 4);
  hm::Pcg64 rng(st[0], st[1], st[2], st[3]);
  const double miss = 1.0 - accuracy;
  int k = 0;
  std::vector<uint8_t> active(static_cast<size_t>(N));
  std::vector<int> pool;
  for (int fl = layer + 1; fl <= last; ++fl, ++k) {
    int64_t *loads = out_loads + static_cast<size_t>(k) * N;
    std::memcpy(loads, pass_loads + static_cast<size_t>(fl) * N, sizeof(int64_t) * N);
    out_layers[k] = fl;
    if (accuracy >= 1.0) continue;
    std::vector<int> orig;
    for (int i = 0; i < N; ++i) {
      active[i] = loads[i] > 0;
      if (active[i]) orig.push_back(i);
    }
    for (int i : orig) {  // sorted(req.activated)
      if (rng.random() < miss) {
        pool.clear();
        for (int j = 0; j < N; ++j)
          if (!active[j]) pool.push_back(j);
        if (pool.empty()) continue;
        const int j = pool[static_cast<size_t>(rng.integers(static_cast<int64_t>(pool.size())))];
        std::swap(loads[i], loads[j]);
        active[i] = 0;
        active[j] = 1;
      }
    }
  }
  *n_out = k;
  HM_API_END
}

}  // extern "C"
