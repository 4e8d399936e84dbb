// Host worker: executes the experts the schedule assigns to the CPU
// (the CPU timeline of scheduling.py:257-268).  bf16 expert
// images are read straight from the pinned host master store in the slot
// layout (include/hybrimoe.h, hm_group); arithmetic is AVX-512 BF16
// (vdpbf16ps: bf16 pairs, fp32 accumulate), the intermediate h is rounded to
// bf16 exactly like the GPU path, outputs are fp32 rows in permuted order.
// Decode (1 token) is a DRAM-bandwidth-bound GEMV split over all threads;
// prefill blocks 16 weight rows x 4 tokens so weights are reused from L2.
#include <immintrin.h>
#include <pthread.h>
#include <sched.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "host_worker.hpp"

namespace hm {

// ------------------------------------------------------------ thread pool
// Waits spin for a few microseconds and then yield the CPU: on an
// oversubscribed VM a pure spin starves the thread being waited for.
static inline void spin_relax() { asm volatile("" ::: "memory"); }
template <class Pred>
static inline void wait_until(Pred done) {
  for (int i = 0; i < 4096; ++i) {
    if (done()) return;
    spin_relax();
  }
  while (!done()) std::this_thread::yield();
}

// HM_PIN_THREADS=1: worker t runs on the t-th CPU of the process's affinity
// mask (the caller, thread 0, is left where it is) -- A/B knob for the
// in-step straggler variance.
static void pin_to_nth_cpu(int t) {
  static const bool on = [] {
    const char *e = std::getenv("HM_PIN_THREADS");
    return e && std::atoi(e) != 0;
  }();
  if (!on) return;
  cpu_set_t mask;
  if (sched_getaffinity(0, sizeof(mask), &mask) != 0) return;
  int seen = 0;
  for (int c = 0; c < CPU_SETSIZE; ++c) {
    if (!CPU_ISSET(c, &mask)) continue;
    if (seen++ == t) {
      cpu_set_t one;
      CPU_ZERO(&one);
      CPU_SET(c, &one);
      pthread_setaffinity_np(pthread_self(), sizeof(one), &one);
      return;
    }
  }
}

ThreadPool::ThreadPool(int n, int spin_us)
    : n_(std::max(1, n)), spin_us_(spin_us), ranges_(new Range[static_cast<size_t>(2) * std::max(1, n)]) {
  for (int t = 1; t < n_; ++t)
    threads_.emplace_back([this, t] {
      pin_to_nth_cpu(t);
      loop(t);
    });
}

ThreadPool::~ThreadPool() {
  {
    std::lock_guard<std::mutex> g(mu_);
    stop_.store(true);
    gen_.fetch_add(1, std::memory_order_release);
  }
  cv_.notify_all();
  for (auto &th : threads_) th.join();
}

void ThreadPool::loop(int tid) {
  uint64_t seen = 0;
  for (;;) {
    // spin briefly (decode issues experts back to back), then sleep
    const auto t0 = std::chrono::steady_clock::now();
    int iter = 0;
    while (gen_.load(std::memory_order_acquire) == seen) {
      if (++iter > 4096) std::this_thread::yield();
      if ((iter & 255) == 0 &&
          std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(spin_us_)) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
        break;
      }
    }
    seen = gen_.load(std::memory_order_acquire);
    if (stop_.load()) return;
    (*job_)(tid, n_);
    pending_.fetch_sub(1, std::memory_order_acq_rel);
  }
}

void ThreadPool::run(const std::function<void(int, int)> &fn, const std::function<void()> *before_self) {
  if (n_ == 1) {
    if (before_self) (*before_self)();
    fn(0, 1);
    return;
  }
  job_ = &fn;
  pending_.store(n_ - 1, std::memory_order_release);
  {
    std::lock_guard<std::mutex> g(mu_);
    gen_.fetch_add(1, std::memory_order_release);
  }
  cv_.notify_all();
  // tid 0 must still take part (the job's barriers count it) even if the
  // caller's own work throws: rethrow only after the job completed
  std::exception_ptr err;
  if (before_self) {
    try {
      (*before_self)();
    } catch (...) {
      err = std::current_exception();
    }
  }
  fn(0, n_);
  wait_until([&] { return pending_.load(std::memory_order_acquire) == 0; });
  if (err) std::rethrow_exception(err);
}

void ThreadPool::barrier() { wait(arrive()); }

uint32_t ThreadPool::arrive() {
  const uint32_t sense = bar_sense_.load(std::memory_order_acquire);
  if (bar_count_.fetch_add(1, std::memory_order_acq_rel) == n_ - 1) {
    bar_count_.store(0, std::memory_order_relaxed);
    bar_sense_.store(sense + 1, std::memory_order_release);
  }
  return sense;
}

bool ThreadPool::passed(uint32_t token) const { return bar_sense_.load(std::memory_order_acquire) != token; }

void ThreadPool::wait(uint32_t token) {
  wait_until([&] { return passed(token); });
}

// Run this thread's [front, back) of `rs` in chunks from the front, then
// steal chunks from the back of the other threads' ranges until all are
// empty.  process(a, b) handles indices [a, b).  The owner keeps one
// sequential stream (hardware prefetch); stealing only trims the tails, so a
// thread slowed by the OS or a busier memory channel no longer holds the
// phase barrier (measured: the slowest of 16 threads ran phase 1 of a
// Mixtral expert 1.5x longer than the median one).
bool &decode_steal() {  // HM_DECODE_STEAL=0 / hm_cpu_set_decode_steal(0): static ranges only (A/B)
  static bool on = [] {
    const char *s = std::getenv("HM_DECODE_STEAL");
    return !s || std::atoi(s) != 0;
  }();
  return on;
}

// chunk: the owner's take from its front; steal_chunk (0 = chunk): what a
// thief takes from another range's back -- small steals trim the tails finely
// while the owner keeps long sequential runs.
template <class F>
void run_ranges(ThreadPool::Range *rs, int tid, int nt, uint32_t chunk, F &&process, uint32_t steal_chunk = 0) {
  if (steal_chunk == 0) steal_chunk = chunk;
  auto take = [&](ThreadPool::Range &r, bool front, uint32_t &a, uint32_t &b) {
    uint64_t v = r.fb.load(std::memory_order_relaxed);
    for (;;) {
      const uint32_t f = static_cast<uint32_t>(v >> 32), k = static_cast<uint32_t>(v);
      if (f >= k) return false;
      if (!front && k - f < 2 * steal_chunk) return false;  // leave the owner a last piece
      uint32_t nf = f, nk = k;
      if (front) {
        nf = std::min(k, f + chunk);
        a = f;
        b = nf;
      } else {
        nk = k - steal_chunk;
        a = nk;
        b = k;
      }
      if (r.fb.compare_exchange_weak(v, (static_cast<uint64_t>(nf) << 32) | nk, std::memory_order_acq_rel))
        return true;
    }
  };
  uint32_t a = 0, b = 0;
  while (take(rs[tid], true, a, b)) process(a, b);
  if (!decode_steal()) return;
  for (int k = 1; k < nt; ++k) {
    ThreadPool::Range &r = rs[(tid + k) % nt];
    while (take(r, false, a, b)) process(a, b);
  }
}

// ------------------------------------------------------------ kernels
namespace {

constexpr int kIlv = 128;

inline float bf2f(uint16_t v) {
  uint32_t u = static_cast<uint32_t>(v) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
inline uint16_t f2bf(float f) {  // round to nearest even
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}
inline __m512bh ldbh(const uint16_t *p) { return (__m512bh)_mm512_loadu_si512(p); }

// acc[r][t] = sum_k W[r][k] * X[t][k] for R rows and TT tokens (K % 32 == 0).
template <int R, int TT>
inline void dot_tile(const uint16_t *const *w, const uint16_t *const *x, int K, float (&out)[R][TT]) {
  __m512 acc[R][TT];
#pragma GCC unroll 4
  for (int r = 0; r < R; ++r)
#pragma GCC unroll 4
    for (int t = 0; t < TT; ++t) acc[r][t] = _mm512_setzero_ps();
  for (int k = 0; k < K; k += 32) {
    __m512bh xv[TT];
#pragma GCC unroll 4
    for (int t = 0; t < TT; ++t) xv[t] = ldbh(x[t] + k);
#pragma GCC unroll 4
    for (int r = 0; r < R; ++r) {
      const __m512bh wv = ldbh(w[r] + k);
#pragma GCC unroll 4
      for (int t = 0; t < TT; ++t) acc[r][t] = _mm512_dpbf16_ps(acc[r][t], wv, xv[t]);
    }
  }
  for (int r = 0; r < R; ++r)
    for (int t = 0; t < TT; ++t) out[r][t] = _mm512_reduce_add_ps(acc[r][t]);
}

inline float silu(float g) { return g / (1.0f + std::exp(-g)); }

// W13 phase for pairs [i0, i1): h[t][i] = bf16(silu(g.x_t) * (u.x_t))
void phase1(const uint16_t *img, int H, int I, const uint16_t *x, int M, uint16_t *h, int i0, int i1) {
  for (int tb = 0; tb < M; tb += 4) {
    const int tt = std::min(4, M - tb);
    const uint16_t *xp[4];
    for (int t = 0; t < 4; ++t) xp[t] = x + static_cast<size_t>(tb + std::min(t, tt - 1)) * H;
    for (int i = i0; i < i1; i += 2) {
      const int npair = std::min(2, i1 - i);
      const uint16_t *w[4];
      for (int q = 0; q < 2; ++q) {
        const int ii = i + std::min(q, npair - 1);
        const size_t grow = static_cast<size_t>((ii / kIlv) * 2 * kIlv + ii % kIlv);
        w[2 * q] = img + grow * H;
        w[2 * q + 1] = img + (grow + kIlv) * H;
      }
      float o[4][4];
      if (tt == 1) {
        float o1[4][1];
        dot_tile<4, 1>(w, xp, H, o1);
        for (int r = 0; r < 4; ++r) o[r][0] = o1[r][0];
      } else {
        dot_tile<4, 4>(w, xp, H, o);
      }
      for (int q = 0; q < npair; ++q)
        for (int t = 0; t < tt; ++t)
          h[static_cast<size_t>(tb + t) * I + i + q] = f2bf(silu(o[2 * q][t]) * o[2 * q + 1][t]);
    }
  }
}

// W2 phase for output rows [j0, j1): out[t][j] = W2[j] . h[t]
void phase2(const uint16_t *img, int H, int I, const uint16_t *h, int M, float *out, int j0, int j1) {
  const uint16_t *w2 = img + static_cast<size_t>(2) * I * H;
  constexpr int RB = 16;  // weight rows kept hot across token blocks
  for (int jb = j0; jb < j1; jb += RB) {
    const int je = std::min(j1, jb + RB);
    for (int tb = 0; tb < M; tb += 4) {
      const int tt = std::min(4, M - tb);
      const uint16_t *hp[4];
      for (int t = 0; t < 4; ++t) hp[t] = h + static_cast<size_t>(tb + std::min(t, tt - 1)) * I;
      for (int j = jb; j < je; j += 4) {
        const int nr = std::min(4, je - j);
        const uint16_t *w[4];
        for (int r = 0; r < 4; ++r) w[r] = w2 + static_cast<size_t>(j + std::min(r, nr - 1)) * I;
        float o[4][4];
        if (tt == 1) {
          float o1[4][1];
          dot_tile<4, 1>(w, hp, I, o1);
          for (int r = 0; r < 4; ++r) o[r][0] = o1[r][0];
        } else {
          dot_tile<4, 4>(w, hp, I, o);
        }
        for (int r = 0; r < nr; ++r)
          for (int t = 0; t < tt; ++t) out[static_cast<size_t>(tb + t) * H + j + r] = o[r][t];
      }
    }
  }
}

// One token: dot of `n` consecutive rows (stride K) with x, in memory order --
// a single sequential stream per thread, 4 independent accumulators, software
// prefetch a few KB ahead.  This is the decode (host-DRAM-bound) path.
// Software-prefetch distance (elements) and hint; HM_PF_DIST / HM_PF_HINT
// (0 none, 1 T0, 2 T1, 3 NTA) override them for tuning on a new host.
struct PfCfg {  // B200 box host, tools/host_phase_prof.py sweep: L2 hint, 16 KB ahead (64 KB overshot the
                // per-thread chunks of small experts: DeepSeek 1 expert 104 -> 175 GB/s, Mixtral 184-194 -> 206)
  int dist = 8192;
  int hint = 2;
};
PfCfg &pf_cfg() {
  static PfCfg c = [] {
    PfCfg p;
    if (const char *s = std::getenv("HM_PF_DIST")) p.dist = std::atoi(s);
    if (const char *s = std::getenv("HM_PF_HINT")) p.hint = std::atoi(s);
    return p;
  }();
  return c;
}

template <int HINT>
inline void stream_rows_t(const uint16_t *w, int n, int K, const uint16_t *x, float *out, int ahead) {
  for (int r = 0; r < n; ++r) {
    const uint16_t *row = w + static_cast<size_t>(r) * K;
    __m512 a0 = _mm512_setzero_ps(), a1 = _mm512_setzero_ps(), a2 = _mm512_setzero_ps(),
           a3 = _mm512_setzero_ps();
    int k = 0;
    for (; k + 128 <= K; k += 128) {
      if constexpr (HINT != 0) {
        constexpr auto hint = HINT == 1 ? _MM_HINT_T0 : (HINT == 2 ? _MM_HINT_T1 : _MM_HINT_NTA);
        const char *pf = reinterpret_cast<const char *>(row + k + ahead);  // the 4 lines of this step
        _mm_prefetch(pf, hint);
        _mm_prefetch(pf + 64, hint);
        _mm_prefetch(pf + 128, hint);
        _mm_prefetch(pf + 192, hint);
      }
      a0 = _mm512_dpbf16_ps(a0, ldbh(row + k), ldbh(x + k));
      a1 = _mm512_dpbf16_ps(a1, ldbh(row + k + 32), ldbh(x + k + 32));
      a2 = _mm512_dpbf16_ps(a2, ldbh(row + k + 64), ldbh(x + k + 64));
      a3 = _mm512_dpbf16_ps(a3, ldbh(row + k + 96), ldbh(x + k + 96));
    }
    for (; k < K; k += 32) a0 = _mm512_dpbf16_ps(a0, ldbh(row + k), ldbh(x + k));
    out[r] = _mm512_reduce_add_ps(_mm512_add_ps(_mm512_add_ps(a0, a1), _mm512_add_ps(a2, a3)));
  }
}

inline void stream_rows(const uint16_t *w, int n, int K, const uint16_t *x, float *out) {
  const PfCfg &c = pf_cfg();
  switch (c.hint) {
    case 0: stream_rows_t<0>(w, n, K, x, out, c.dist); break;
    case 2: stream_rows_t<2>(w, n, K, x, out, c.dist); break;
    case 3: stream_rows_t<3>(w, n, K, x, out, c.dist); break;
    default: stream_rows_t<1>(w, n, K, x, out, c.dist); break;
  }
}

// Decode phase 1 over whole 128-pair blocks [b0, b1): W13 block b is 128 gate
// rows then 128 up rows, contiguous -- read it front to back.
void phase1_stream(const uint16_t *img, int H, int I, const uint16_t *x, uint16_t *h, int b0, int b1) {
  float gu[2 * kIlv];
  for (int b = b0; b < b1; ++b) {
    stream_rows(img + static_cast<size_t>(b) * 2 * kIlv * H, 2 * kIlv, H, x, gu);
    for (int i = 0; i < kIlv; ++i) h[b * kIlv + i] = f2bf(silu(gu[i]) * gu[kIlv + i]);
  }
}

// Decode phase 1 over pairs [i0, i1) (any range): inside each 128-pair block
// the gate rows of the range, then its up rows -- two sequential streams.
// Pair-granular ranges balance the threads when a layer's experts are small
// (DeepSeek: 11 blocks per expert would leave 16 threads 9 % imbalanced).
void phase1_pairs(const uint16_t *img, int H, int I, const uint16_t *x, uint16_t *h, int i0, int i1) {
  float g[kIlv], u[kIlv];
  while (i0 < i1) {
    const int b = i0 / kIlv, s = i0 % kIlv;
    const int n = std::min(i1, (b + 1) * kIlv) - i0;
    const uint16_t *blk = img + static_cast<size_t>(b) * 2 * kIlv * H;
    stream_rows(blk + static_cast<size_t>(s) * H, n, H, x, g);
    stream_rows(blk + static_cast<size_t>(kIlv + s) * H, n, H, x, u);
    for (int i = 0; i < n; ++i) h[i0 + i] = f2bf(silu(g[i]) * u[i]);
    i0 += n;
  }
}

long steal_kb() {
  static const long v = [] {
    const char *e = std::getenv("HM_STEAL_KB");
    return e ? std::max(1L, std::atol(e)) : 64L;
  }();
  return v;
}

// Decode work split granularity (pairs in phase 1, rows in phase 2); 0 = the
// legacy whole-128-pair-block split.  Process-wide tuning knob.
int &decode_grain() {
  static int g = [] {
    const char *s = std::getenv("HM_DECODE_GRAIN");
    return s ? std::atoi(s) : 16;
  }();
  return g;
}

// Per-thread phase timestamps of the last decode / AMX call (hm_cpu_decode_profile):
// AMX: [0] start, [1] activations packed, [2] phase 1 done, [3] phase 2 done (ns);
// [tid][0] start, [1] phase 1 done, [2] barrier passed, [3] phase 2 done (ns).
static std::vector<int64_t> g_dec_prof;
static bool g_dec_prof_on = false;
// accumulated over decode calls while profiling (hm_cpu_decode_profile_accum):
// calls, sum of [max worker start (tid >= 1), tid-0 start, max phase-1 end,
// barrier passed, max phase-2 end, wall] in ns
static int64_t g_dec_acc[7] = {0, 0, 0, 0, 0, 0, 0};
// worker-start histogram (max over tid >= 1 per call: <= 5, 20, 100, 1000, > 1000 us)
// and the slowest starter's tid
static int64_t g_dec_hist[5] = {0, 0, 0, 0, 0};
static std::vector<int64_t> g_dec_slowest;
static inline int64_t ns_now() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// ------------------------------------------------------------ AMX (prefill)
// Multi-token experts on the AMX tile unit: out^T = W . X^T with A = 16 weight
// rows x 32 K (row-major, loaded straight from the image) and B = 16 token
// pairs x 16 tokens in VNNI order (x and h are repacked once per expert).
// Register blocking: 2 A x 2 B -> 4 fp32 C tiles (tiles 0-3 C, 4-5 A, 6-7 B).
struct alignas(64) TileCfg {
  uint8_t palette = 1;
  uint8_t start_row = 0;
  uint8_t reserved[14] = {};
  uint16_t colsb[16] = {};
  uint8_t rows[16] = {};
};

// exp(x) for 16 floats: 2^n * p(r), |r| <= ln2/2, degree-6 polynomial (rel err ~1e-7).
inline __m512 exp16(__m512 x) {
  x = _mm512_max_ps(_mm512_min_ps(x, _mm512_set1_ps(88.0f)), _mm512_set1_ps(-88.0f));
  const __m512 n = _mm512_roundscale_ps(_mm512_mul_ps(x, _mm512_set1_ps(1.4426950408889634f)), _MM_FROUND_TO_NEAREST_INT);
  const __m512 r = _mm512_fnmadd_ps(n, _mm512_set1_ps(0.6931471805599453f), x);
  __m512 p = _mm512_set1_ps(1.0f / 720.0f);
  p = _mm512_fmadd_ps(p, r, _mm512_set1_ps(1.0f / 120.0f));
  p = _mm512_fmadd_ps(p, r, _mm512_set1_ps(1.0f / 24.0f));
  p = _mm512_fmadd_ps(p, r, _mm512_set1_ps(1.0f / 6.0f));
  p = _mm512_fmadd_ps(p, r, _mm512_set1_ps(0.5f));
  p = _mm512_fmadd_ps(p, r, _mm512_set1_ps(1.0f));
  p = _mm512_fmadd_ps(p, r, _mm512_set1_ps(1.0f));
  return _mm512_scalef_ps(p, n);
}

// silu(g) * u for 16 lanes
inline __m512 silu_mul16(const float *g, const float *u) {
  const __m512 gv = _mm512_loadu_ps(g);
  const __m512 den = _mm512_add_ps(_mm512_set1_ps(1.0f), exp16(_mm512_sub_ps(_mm512_setzero_ps(), gv)));
  return _mm512_mul_ps(_mm512_div_ps(gv, den), _mm512_loadu_ps(u));
}

// two 16-float rows -> 32 bf16 interleaved (a0 b0 a1 b1 ...), round to nearest even
inline __m512i interleave_bf16(__m512 a, __m512 b) {
  const __m512i v = _mm512_inserti64x4(_mm512_castsi256_si512((__m256i)_mm512_cvtneps_pbh(a)),
                                       (__m256i)_mm512_cvtneps_pbh(b), 1);
  const __m512i idx = _mm512_set_epi16(31, 15, 30, 14, 29, 13, 28, 12, 27, 11, 26, 10, 25, 9, 24, 8, 23, 7, 22, 6,
                                       21, 5, 20, 4, 19, 3, 18, 2, 17, 1, 16, 0);
  return _mm512_permutexvar_epi16(idx, v);
}

bool amx_enable() {  // Linux: request the XTILEDATA permission once per process
  static const bool ok = [] {
    if (!__builtin_cpu_supports("amx-bf16")) return false;
    constexpr long kReqPerm = 0x1023, kXtileData = 18;
    return syscall(SYS_arch_prctl, kReqPerm, kXtileData) == 0;
  }();
  return ok;
}

inline void amx_config() {
  static thread_local bool done = false;
  if (done) return;
  TileCfg c;
  for (int t = 0; t < 8; ++t) {
    c.colsb[t] = 64;
    c.rows[t] = 16;
  }
  _tile_loadconfig(&c);
  done = true;
}

// VNNI repack: src [M, K] bf16 rows -> dst [K/2][Mpad][2] (zero-padded tokens),
// i.e. a transpose of the [M][K/2] matrix of 32-bit bf16 pairs.  Rows of
// k-pairs [kp0, kp1) only: every pool thread packs its own slice (the serial
// scalar pack was ~40 % of a 64-token DeepSeek expert); 16 tokens per gather.
void vnni_pack_rows(const uint16_t *src, int M, int K, int Mpad, uint16_t *dst, int kp0, int kp1) {
  const int *s32 = reinterpret_cast<const int *>(src);
  uint32_t *d32 = reinterpret_cast<uint32_t *>(dst);
  const int K2 = K / 2;
  const __m512i iota = _mm512_set_epi32(15, 14, 13, 12, 11, 10, 9, 8, 7, 6, 5, 4, 3, 2, 1, 0);
  for (int tb = 0; tb < Mpad; tb += 16) {
    const int n = M - tb;
    const __mmask16 live = n >= 16 ? 0xFFFF : n > 0 ? static_cast<__mmask16>((1u << n) - 1u) : 0;
    const __m512i idx = _mm512_mullo_epi32(_mm512_add_epi32(_mm512_set1_epi32(tb), iota), _mm512_set1_epi32(K2));
    for (int kp = kp0; kp < kp1; ++kp) {
      const __m512i v = live ? _mm512_mask_i32gather_epi32(_mm512_setzero_si512(), live, idx, s32 + kp, 4)
                             : _mm512_setzero_si512();
      _mm512_storeu_si512(d32 + static_cast<size_t>(kp) * Mpad + tb, v);
    }
  }
}
// this pool thread's share of the pack, then a barrier (inside pool.run)
inline void vnni_pack_par(ThreadPool &pool, int tid, int nt, const uint16_t *src, int M, int K, int Mpad,
                          uint16_t *dst) {
  const int K2 = K / 2;
  vnni_pack_rows(src, M, K, Mpad, dst, static_cast<int>(static_cast<long>(K2) * tid / nt),
                 static_cast<int>(static_cast<long>(K2) * (tid + 1) / nt));
  pool.barrier();
}
// per-thread scratch that persists across calls (a fresh std::vector per call
// page-faulted and zeroed up to 1 MB per thread per expert)
template <class T>
T *tls_buf(std::vector<T> &v, size_t n) {
  if (v.size() < n) v.resize(n);
  return v.data();
}

// C[a][b] (16 rows of A-block a x 16 tokens of B-block b) over the full K for
// two weight row blocks (wa0, wa1; stride ldw bytes) and token blocks tb0, tb0+16.
inline void amx_block(const uint16_t *wa0, const uint16_t *wa1, size_t ldw, const uint16_t *xv, int Mpad, int tb0,
                      bool two_b, int K, float (*c)[16][16]) {
  _tile_zero(0);
  _tile_zero(1);
  _tile_zero(2);
  _tile_zero(3);
  const size_t ldb = static_cast<size_t>(Mpad) * 4;
  for (int k = 0; k < K; k += 32) {
    _tile_loadd(4, wa0 + k, ldw);
    _tile_loadd(5, wa1 + k, ldw);
    const uint16_t *b = xv + (static_cast<size_t>(k >> 1) * Mpad + tb0) * 2;
    _tile_loadd(6, b, ldb);
    _tile_dpbf16ps(0, 4, 6);
    _tile_dpbf16ps(2, 5, 6);
    if (two_b) {
      _tile_loadd(7, b + 32, ldb);
      _tile_dpbf16ps(1, 4, 7);
      _tile_dpbf16ps(3, 5, 7);
    }
  }
  _tile_stored(0, c[0], 64);
  _tile_stored(2, c[2], 64);
  if (two_b) {
    _tile_stored(1, c[1], 64);
    _tile_stored(3, c[3], 64);
  }
}

// Cache-blocked AMX GEMM over weight rows (A, row-major straight from the
// expert image) and tokens (B, VNNI):  for each unit o in [o0, o1) two 16-row
// weight blocks (rowptr(o, 0/1)) times all nbt token blocks over the full K,
// accumulated in C[o - o0][2][nbt][16 x 16] fp32 (cbuf).
// Loop order: units in groups of GO (their C stays in L2) -> K chunks of KC
// (a unit's 2 x 16 x KC weight chunk is loaded from DRAM once and reused
// from L1 for every token-block pair; the chunk of the next unit is software-
// prefetched meanwhile) -> token-block pairs (2 x 2 register blocking: 4 C,
// 2 A, 2 B tiles).  The previous kernel re-read the whole token matrix from
// L2/L3 for every 16-row block and ran at ~3.5 TF/s.
struct AmxCfg {
  int kc = 128;  // K chunk (elements)
  int go = 8;    // units per group
};
AmxCfg &amx_cfg() {
  static AmxCfg c = [] {
    AmxCfg a;
    if (const char *e = std::getenv("HM_AMX_KC")) a.kc = std::max(32, std::atoi(e) / 32 * 32);
    if (const char *e = std::getenv("HM_AMX_GO")) a.go = std::max(1, std::atoi(e));
    return a;
  }();
  return c;
}
// 0 (default): per-unit full-K blocks; 1: cache-blocked; -1: cache-blocked
// from 256 tokens up.  With dynamic unit claims and vector output transposes
// in both, the full-K kernel measured faster at every shape and M <= 256 on
// the box's host (tools/amx_phase_prof.py; Mixtral M=256 11.5 vs 17.6 ms).
int &amx_algo() {
  static int a = [] {
    const char *e = std::getenv("HM_AMX_ALGO");
    return e ? std::atoi(e) : 0;
  }();
  return a;
}

template <class RowPtr>
void amx_gemm_units(RowPtr rowptr, int o0, int o1, size_t lda_bytes, const uint16_t *bv, int Mpad, int K,
                    float *cbuf) {
  const int nbt = Mpad / 16;
  const size_t ldb = static_cast<size_t>(Mpad) * 4;
  const size_t cu = static_cast<size_t>(2) * nbt * 256;  // floats of C per unit
  const int KC = amx_cfg().kc;
  for (int kc = 0; kc < K; kc += KC) {
    const int kend = std::min(K, kc + KC);
    for (int o = o0; o < o1; ++o) {
      const uint16_t *a0 = rowptr(o, 0), *a1 = rowptr(o, 1);
      // prefetch the next unit's chunk (or this unit's next chunk) into L2
      {
        const bool last = o + 1 >= o1;
        const int po = last ? o0 : o + 1;
        const int pk = last ? kend : kc;
        if (pk < K) {
          const uint16_t *p0 = rowptr(po, 0), *p1 = rowptr(po, 1);
          const int pn = std::min(K, pk + KC) - pk;
          for (int r = 0; r < 16; ++r)
            for (int c = 0; c < pn * 2; c += 64) {
              _mm_prefetch(reinterpret_cast<const char *>(p0) + r * lda_bytes + pk * 2 + c, _MM_HINT_T1);
              _mm_prefetch(reinterpret_cast<const char *>(p1) + r * lda_bytes + pk * 2 + c, _MM_HINT_T1);
            }
        }
      }
      float *cb = cbuf + static_cast<size_t>(o - o0) * cu;
      for (int b = 0; b < nbt; b += 2) {
        const bool two = b + 1 < nbt;
        float *c00 = cb + static_cast<size_t>(b) * 256, *c01 = c00 + 256;
        float *c10 = cb + (static_cast<size_t>(nbt) + b) * 256, *c11 = c10 + 256;
        if (kc == 0) {
          _tile_zero(0);
          _tile_zero(1);
          _tile_zero(2);
          _tile_zero(3);
        } else {
          _tile_loadd(0, c00, 64);
          _tile_loadd(2, c10, 64);
          if (two) {
            _tile_loadd(1, c01, 64);
            _tile_loadd(3, c11, 64);
          }
        }
        for (int k = kc; k < kend; k += 32) {
          _tile_loadd(4, a0 + k, lda_bytes);
          _tile_loadd(5, a1 + k, lda_bytes);
          const uint16_t *bp = bv + (static_cast<size_t>(k >> 1) * Mpad + b * 16) * 2;
          _tile_loadd(6, bp, ldb);
          _tile_dpbf16ps(0, 4, 6);
          _tile_dpbf16ps(2, 5, 6);
          if (two) {
            _tile_loadd(7, bp + 32, ldb);
            _tile_dpbf16ps(1, 4, 7);
            _tile_dpbf16ps(3, 5, 7);
          }
        }
        _tile_stored(0, c00, 64);
        _tile_stored(2, c10, 64);
        if (two) {
          _tile_stored(1, c01, 64);
          _tile_stored(3, c11, 64);
        }
      }
    }
  }
}

void cpu_expert_amx2(ThreadPool &pool, const uint16_t *img, int H, int I, const uint16_t *x, int M, float *out,
                     std::vector<uint16_t> &scratch) {
  const int Mpad = (M + 31) / 32 * 32;  // token blocks in pairs
  const int nbt = Mpad / 16;
  scratch.resize(static_cast<size_t>(H) * Mpad + static_cast<size_t>(I) * Mpad);
  uint16_t *xv = scratch.data();
  uint16_t *hv = xv + static_cast<size_t>(H) * Mpad;
  const uint16_t *w2 = img + static_cast<size_t>(2) * I * H;
  const int GO = amx_cfg().go;
  std::atomic<int> next1{0}, next2{0};  // groups of GO units, claimed dynamically
  if (g_dec_prof_on && g_dec_prof.size() < static_cast<size_t>(pool.size()) * 4)
    g_dec_prof.assign(static_cast<size_t>(pool.size()) * 4, 0);
  const int64_t t_call = g_dec_prof_on ? ns_now() : 0;
  pool.run([&](int tid, int nt) {
    int64_t *tp = g_dec_prof_on ? &g_dec_prof[static_cast<size_t>(tid) * 4] : nullptr;
    if (tp) tp[0] = ns_now() - t_call;
    amx_config();
    vnni_pack_par(pool, tid, nt, x, M, H, Mpad, xv);
    if (tp) tp[1] = ns_now() - t_call;
    static thread_local std::vector<float> cvec;
    struct {
      float *p;
      float *data() { return p; }
    } cbuf{tls_buf(cvec, static_cast<size_t>(GO) * 2 * nbt * 256)};
    // phase 1: unit o = 16 gate rows (block 0) + their 16 up rows (block 1)
    const int ob = I / 16;
    auto row1 = [&](int o, int which) {
      const int i0 = o * 16;
      const size_t grow = static_cast<size_t>((i0 / kIlv) * 2 * kIlv + i0 % kIlv);
      return img + (grow + (which ? kIlv : 0)) * H;
    };
    // groups small enough that every thread claims at least two
    const int GO1 = std::max(1, std::min(GO, ob / (2 * nt)));
    for (int gi; (gi = next1.fetch_add(1, std::memory_order_relaxed)) * GO1 < ob;) {
      const int g0 = gi * GO1, g1 = std::min(ob, g0 + GO1);
      amx_gemm_units(row1, g0, g1, static_cast<size_t>(H) * 2, xv, Mpad, H, cbuf.data());
      for (int o = g0; o < g1; ++o) {
        const float *cb = cbuf.data() + static_cast<size_t>(o - g0) * 2 * nbt * 256;
        const int i0 = o * 16;
        for (int b = 0; b < nbt; ++b) {
          const int tok0 = b * 16;
          if (tok0 >= M) {  // padded tokens: zero h
            for (int r = 0; r < 16; r += 2)
              _mm512_storeu_si512(hv + (static_cast<size_t>((i0 + r) >> 1) * Mpad + tok0) * 2, _mm512_setzero_si512());
            continue;
          }
          const __mmask16 live = tok0 + 16 <= M ? 0xFFFF : static_cast<__mmask16>((1u << (M - tok0)) - 1u);
          const float *cg = cb + static_cast<size_t>(b) * 256, *cu = cb + (static_cast<size_t>(nbt) + b) * 256;
          for (int r = 0; r < 16; r += 2) {
            const __m512 h0 = _mm512_maskz_mov_ps(live, silu_mul16(cg + r * 16, cu + r * 16));
            const __m512 h1 = _mm512_maskz_mov_ps(live, silu_mul16(cg + (r + 1) * 16, cu + (r + 1) * 16));
            _mm512_storeu_si512(hv + (static_cast<size_t>((i0 + r) >> 1) * Mpad + tok0) * 2, interleave_bf16(h0, h1));
          }
        }
      }
    }
    if (tp) tp[2] = ns_now() - t_call;
    pool.barrier();
    // phase 2: unit q = W2 rows 32q..32q+15 (block 0) and 32q+16..32q+31 (block 1)
    const int pairs = H / 32;
    auto row2 = [&](int q, int which) { return w2 + static_cast<size_t>(q * 32 + which * 16) * I; };
    const __m512i col = _mm512_set_epi32(240, 224, 208, 192, 176, 160, 144, 128, 112, 96, 80, 64, 48, 32, 16, 0);
    const int GO2 = std::max(1, std::min(GO, pairs / (2 * nt)));
    for (int gi; (gi = next2.fetch_add(1, std::memory_order_relaxed)) * GO2 < pairs;) {
      const int g0 = gi * GO2, g1 = std::min(pairs, g0 + GO2);
      amx_gemm_units(row2, g0, g1, static_cast<size_t>(I) * 2, hv, Mpad, I, cbuf.data());
      for (int q = g0; q < g1; ++q) {
        const float *cb = cbuf.data() + static_cast<size_t>(q - g0) * 2 * nbt * 256;
        for (int a = 0; a < 2; ++a)
          for (int b = 0; b < nbt; ++b) {
            const float *c = cb + (static_cast<size_t>(a) * nbt + b) * 256;
            for (int t = 0; t < 16; ++t) {  // column t of C = token t's 16 outputs
              const int tok = b * 16 + t;
              if (tok >= M) break;
              _mm512_storeu_ps(out + static_cast<size_t>(tok) * H + q * 32 + a * 16, _mm512_i32gather_ps(col, c + t, 4));
            }
          }
      }
    }
    if (tp) tp[3] = ns_now() - t_call;
  });
}

// ------------------------------------------------------------ 4-bit experts
// Image layout and value rule: include/hybrimoe.h (hm_q4_*), oracle/moe_ref.py.
struct Q4View {
  const uint8_t *n13, *n2;
  const uint16_t *s13, *s2;
};
inline Q4View q4_view(const uint8_t *img, int H, int I) {
  const size_t hi = static_cast<size_t>(H) * I;
  Q4View v;
  v.n13 = img;
  v.n2 = img + hi;
  v.s13 = reinterpret_cast<const uint16_t *>(img + hi + hi / 2);
  v.s2 = v.s13 + static_cast<size_t>(2) * I * (H / 128);
  return v;
}

// x (bf16 [K]) for the int4 GEMV: per 128-group g, scale sx = max|x|/127 and
// two int8 digits per element, x ~= sx * (hi + lo/256) (|error| <= sx/512),
// split into even / odd elements so that VNNI (vpdpbusd: u8 x s8, 4 per int32
// lane) multiplies the low nibbles (even elements) and the high nibbles (odd)
// of a weight byte vector with the matching digits.  sq = sum(hi) + sum(lo)/256.
struct Q4X {
  std::vector<int8_t> d;   // [K/128][4][64]: even hi | odd hi | even lo | odd lo
  std::vector<float> sx, sq;
};
inline void q4_alloc_x(int K, Q4X &q) {
  const int ng = K / 128;
  q.d.resize(static_cast<size_t>(ng) * 256);
  q.sx.resize(ng);
  q.sq.resize(ng);
}
// groups [g0, g1) of x (q already sized by q4_alloc_x)
inline void q4_prep_groups(const uint16_t *x, Q4X &q, int g0, int g1) {
  for (int g = g0; g < g1; ++g) {
    float m = 0.f;
    for (int i = 0; i < 128; ++i) m = std::max(m, std::fabs(bf2f(x[g * 128 + i])));
    const float s = m > 0.f ? m / 127.f : 1.f, inv = 1.f / s;
    int sh = 0, sl = 0;
    int8_t *d = q.d.data() + static_cast<size_t>(g) * 256;
    for (int i = 0; i < 128; ++i) {
      const float t = bf2f(x[g * 128 + i]) * inv;
      const float hi = std::nearbyint(t);
      const int lo = std::max(-127, std::min(127, static_cast<int>(std::nearbyint((t - hi) * 256.f))));
      d[(i & 1) * 64 + (i >> 1)] = static_cast<int8_t>(hi);
      d[128 + (i & 1) * 64 + (i >> 1)] = static_cast<int8_t>(lo);
      sh += static_cast<int>(hi);
      sl += lo;
    }
    q.sx[g] = s;
    q.sq[g] = static_cast<float>(sh) + static_cast<float>(sl) * (1.f / 256.f);
  }
}
inline void q4_prep_x(const uint16_t *x, int K, Q4X &q) {
  q4_alloc_x(K, q);
  q4_prep_groups(x, q, 0, K / 128);
}

// Software-prefetch distance of the 4-bit decode stream (HM_Q4_PF bytes, 0 = off).
inline int q4_pf_dist() {
  static const int d = [] {
    const char *e = std::getenv("HM_Q4_PF");
    return e ? std::atoi(e) : 16384;
  }();
  return d;
}

// Up to 4 tokens at once: each 128-group's 64 nibble bytes are split into
// low / high nibble vectors once and multiplied with every token's digits
// (4 vpdpbusd per token and group).  out[t * ldo + r].
template <int MT>
inline void dot_rows_q4_mt(const uint8_t *nib, const uint16_t *sc, int n, int K, const Q4X *const *q, float *out,
                           size_t ldo) {
  const __m512i m15 = _mm512_set1_epi8(15);
  const __m512 inv256 = _mm512_set1_ps(1.f / 256.f);
  const int ng = K / 128;
  for (int r = 0; r < n; ++r) {
    const uint8_t *row = nib + static_cast<size_t>(r) * (K / 2);
    const uint16_t *srow = sc + static_cast<size_t>(r) * (K / 128);
    _mm_prefetch(reinterpret_cast<const char *>(row + 16 * (K / 2)), _MM_HINT_T1);
    __m512 acc[MT];
    float corr[MT];
    for (int t = 0; t < MT; ++t) {
      acc[t] = _mm512_setzero_ps();
      corr[t] = 0.f;
    }
    for (int g = 0; g < ng; ++g) {
      // rows of a unit are contiguous: keep the stream q4_pf_dist() bytes ahead
      _mm_prefetch(reinterpret_cast<const char *>(row + g * 64) + q4_pf_dist(), _MM_HINT_T1);
      const __m512i wb = _mm512_loadu_si512(row + g * 64);
      const __m512i lo = _mm512_and_si512(wb, m15);
      const __m512i hi = _mm512_and_si512(_mm512_srli_epi16(wb, 4), m15);
      const float sw = bf2f(srow[g]);
      for (int t = 0; t < MT; ++t) {
        const int8_t *d = q[t]->d.data() + static_cast<size_t>(g) * 256;
        __m512i ah = _mm512_dpbusd_epi32(_mm512_setzero_si512(), lo, _mm512_loadu_si512(d));
        ah = _mm512_dpbusd_epi32(ah, hi, _mm512_loadu_si512(d + 64));
        __m512i al = _mm512_dpbusd_epi32(_mm512_setzero_si512(), lo, _mm512_loadu_si512(d + 128));
        al = _mm512_dpbusd_epi32(al, hi, _mm512_loadu_si512(d + 192));
        const __m512 f = _mm512_fmadd_ps(_mm512_cvtepi32_ps(al), inv256, _mm512_cvtepi32_ps(ah));
        const float c = sw * q[t]->sx[g];
        acc[t] = _mm512_fmadd_ps(_mm512_set1_ps(c), f, acc[t]);
        corr[t] += c * q[t]->sq[g];
      }
    }
    for (int t = 0; t < MT; ++t) out[static_cast<size_t>(t) * ldo + r] = _mm512_reduce_add_ps(acc[t]) - 8.f * corr[t];
  }
}

inline void dot_rows_q4(const uint8_t *nib, const uint16_t *sc, int n, int K, const Q4X &q, float *out) {
  const Q4X *qp[1] = {&q};
  dot_rows_q4_mt<1>(nib, sc, n, K, qp, out, 0);
}

inline void dot_rows_q4_tokens(const uint8_t *nib, const uint16_t *sc, int n, int K, const Q4X *const *q, int mt,
                               float *out, size_t ldo) {
  switch (mt) {
    case 1: dot_rows_q4_mt<1>(nib, sc, n, K, q, out, ldo); break;
    case 2: dot_rows_q4_mt<2>(nib, sc, n, K, q, out, ldo); break;
    case 3: dot_rows_q4_mt<3>(nib, sc, n, K, q, out, ldo); break;
    default: dot_rows_q4_mt<4>(nib, sc, n, K, q, out, ldo); break;
  }
}

// dequantize n 4-bit rows to bf16 rows (w = bf16((nibble - 8) * scale), as the GPU dequantizer)
inline void dequant_rows_q4(const uint8_t *nib, const uint16_t *sc, int n, int K, uint16_t *dst) {
  const __m512i m15 = _mm512_set1_epi32(15);
  const __m512 eight = _mm512_set1_ps(8.0f);
  for (int r = 0; r < n; ++r)
    for (int g = 0; g < K / 128; ++g) {
      const __m512 s = _mm512_set1_ps(bf2f(sc[static_cast<size_t>(r) * (K / 128) + g]));
      const uint8_t *b = nib + static_cast<size_t>(r) * (K / 2) + g * 64;
      uint16_t *o = dst + static_cast<size_t>(r) * K + g * 128;
      for (int c = 0; c < 4; ++c) {  // 16 bytes -> 32 bf16 (element 2k low nibble, 2k+1 high nibble)
        const __m512i v = _mm512_cvtepu8_epi32(_mm_loadu_si128(reinterpret_cast<const __m128i *>(b + c * 16)));
        const __m512 lo = _mm512_mul_ps(_mm512_sub_ps(_mm512_cvtepi32_ps(_mm512_and_epi32(v, m15)), eight), s);
        const __m512 hi = _mm512_mul_ps(_mm512_sub_ps(_mm512_cvtepi32_ps(_mm512_srli_epi32(v, 4)), eight), s);
        // bf16 pairs (lo_k, hi_k) in each 32-bit lane == memory order; RNE like f2bf
        _mm512_storeu_si512(o + c * 32, interleave_bf16(lo, hi));
      }
    }
}

}  // namespace

void cpu_experts_decode_q4(ThreadPool &pool, const uint8_t *const *imgs, const uint16_t *const *xs, int n, int H,
                           int I, float *const *outs, std::vector<uint16_t> &hbuf,
                           const std::function<void()> *before_self) {
  HM_REQUIRE(H % 128 == 0 && I % 128 == 0, HM_EVALUE, "4-bit host worker needs H, I multiples of 128");
  if (n <= 0) {
    if (before_self) (*before_self)();
    return;
  }
  hbuf.resize(static_cast<size_t>(n) * I);
  uint16_t *h = hbuf.data();
  std::vector<Q4X> qx(n), hx(n);
  for (int e = 0; e < n; ++e) {
    q4_prep_x(xs[e], H, qx[e]);
    q4_alloc_x(I, hx[e]);
  }
  // 16-pair (phase 1) and 16-row (phase 2) units, per-thread contiguous ranges
  // with stealing from the tails (as cpu_experts_decode)
  const int nt0 = pool.size();
  const long nu1 = static_cast<long>(n) * I / 16, nu2 = static_cast<long>(n) * H / 16;
  for (int t = 0; t < nt0; ++t) {
    pool.ranges(0)[t].fb.store((static_cast<uint64_t>(nu1 * t / nt0) << 32) | static_cast<uint64_t>(nu1 * (t + 1) / nt0),
                               std::memory_order_relaxed);
    pool.ranges(1)[t].fb.store((static_cast<uint64_t>(nu2 * t / nt0) << 32) | static_cast<uint64_t>(nu2 * (t + 1) / nt0),
                               std::memory_order_relaxed);
  }
  pool.run([&](int tid, int nt) {
    // phase 1: 16-pair units over the flat (expert, pair) space, gate and up rows
    float g[16], u[16];
    run_ranges(pool.ranges(0), tid, nt, 2, [&](uint32_t q0, uint32_t q1) {
      for (long q = q0; q < static_cast<long>(q1); ++q) {
        const int e = static_cast<int>(q / (I / 16)), i0 = static_cast<int>(q % (I / 16)) * 16;
        const Q4View v = q4_view(imgs[e], H, I);
        const size_t grow = static_cast<size_t>((i0 / kIlv) * 2 * kIlv + i0 % kIlv);
        dot_rows_q4(v.n13 + grow * (H / 2), v.s13 + grow * (H / 128), 16, H, qx[e], g);
        dot_rows_q4(v.n13 + (grow + kIlv) * (H / 2), v.s13 + (grow + kIlv) * (H / 128), 16, H, qx[e], u);
        for (int i = 0; i < 16; ++i) h[static_cast<size_t>(e) * I + i0 + i] = f2bf(silu(g[i]) * u[i]);
      }
    });
    pool.barrier();
    {  // h -> int8 digits, groups split over the threads (once, not per thread)
      const long ng = static_cast<long>(n) * (I / 128);
      for (long q = ng * tid / nt; q < ng * (tid + 1) / nt; ++q) {
        const int e = static_cast<int>(q / (I / 128)), gq = static_cast<int>(q % (I / 128));
        q4_prep_groups(h + static_cast<size_t>(e) * I, hx[e], gq, gq + 1);
      }
    }
    pool.barrier();
    run_ranges(pool.ranges(1), tid, nt, 2, [&](uint32_t q0, uint32_t q1) {
      for (long q = q0; q < static_cast<long>(q1); ++q) {
        const int e = static_cast<int>(q / (H / 16)), j0 = static_cast<int>(q % (H / 16)) * 16;
        const Q4View v = q4_view(imgs[e], H, I);
        dot_rows_q4(v.n2 + static_cast<size_t>(j0) * (I / 2), v.s2 + static_cast<size_t>(j0) * (I / 128), 16, I,
                    hx[e], outs[e] + j0);
      }
    });
  }, before_self);
}

void cpu_expert_q4(ThreadPool &pool, const uint8_t *img, int H, int I, const uint16_t *x, int M, float *out,
                   std::vector<uint16_t> &scratch) {
  HM_REQUIRE(H % 128 == 0 && I % 128 == 0, HM_EVALUE, "4-bit host worker needs H, I multiples of 128");
  if (M <= 0) return;
  if (M == 1) {
    const uint8_t *imgs[1] = {img};
    const uint16_t *xs[1] = {x};
    float *outs[1] = {out};
    cpu_experts_decode_q4(pool, imgs, xs, 1, H, I, outs, scratch);
    return;
  }
  if (M <= 4) {  // few tokens: stream the nibbles once, decode each group once for all tokens
    std::vector<Q4X> qx(M);
    const Q4X *qp[4];
    for (int t = 0; t < M; ++t) {
      q4_prep_x(x + static_cast<size_t>(t) * H, H, qx[t]);
      qp[t] = &qx[t];
    }
    scratch.resize(static_cast<size_t>(M) * I);
    uint16_t *hh = scratch.data();
    std::vector<Q4X> hxs(M);
    for (int t = 0; t < M; ++t) q4_alloc_x(I, hxs[t]);
    const Q4View v = q4_view(img, H, I);
    pool.run([&](int tid, int nt) {
      const int nu = I / 16;
      float g[4 * 16], u[4 * 16];
      for (int q = nu * tid / nt; q < nu * (tid + 1) / nt; ++q) {
        const int i0 = q * 16;
        const size_t grow = static_cast<size_t>((i0 / kIlv) * 2 * kIlv + i0 % kIlv);
        dot_rows_q4_tokens(v.n13 + grow * (H / 2), v.s13 + grow * (H / 128), 16, H, qp, M, g, 16);
        dot_rows_q4_tokens(v.n13 + (grow + kIlv) * (H / 2), v.s13 + (grow + kIlv) * (H / 128), 16, H, qp, M, u, 16);
        for (int t = 0; t < M; ++t)
          for (int i = 0; i < 16; ++i) hh[static_cast<size_t>(t) * I + i0 + i] = f2bf(silu(g[t * 16 + i]) * u[t * 16 + i]);
      }
      pool.barrier();
      const long ng = static_cast<long>(M) * (I / 128);
      for (long q = ng * tid / nt; q < ng * (tid + 1) / nt; ++q) {
        const int t = static_cast<int>(q / (I / 128)), gq = static_cast<int>(q % (I / 128));
        q4_prep_groups(hh + static_cast<size_t>(t) * I, hxs[t], gq, gq + 1);
      }
      pool.barrier();
      const Q4X *hp[4];
      for (int t = 0; t < M; ++t) hp[t] = &hxs[t];
      const int nr = H / 16;
      for (int q = nr * tid / nt; q < nr * (tid + 1) / nt; ++q)
        dot_rows_q4_tokens(v.n2 + static_cast<size_t>(q * 16) * (I / 2), v.s2 + static_cast<size_t>(q * 16) * (I / 128),
                           16, I, hp, M, out + q * 16, static_cast<size_t>(H));
    });
    return;
  }
  HM_REQUIRE(amx_enable(), HM_ERUNTIME, "4-bit prefill on the host needs AMX");
  // multi-token groups: each 32-row unit is dequantized to bf16 in a per-thread
  // buffer (L2-resident) and multiplied on the AMX tiles like a bf16 expert
  const int Mpad = (M + 31) / 32 * 32, nbt = Mpad / 16;
  scratch.resize(static_cast<size_t>(H) * Mpad + static_cast<size_t>(I) * Mpad);
  uint16_t *xv = scratch.data();
  uint16_t *hv = xv + static_cast<size_t>(H) * Mpad;
  const Q4View v = q4_view(img, H, I);
  std::atomic<int> next1{0}, next2{0};  // units claimed dynamically
  pool.run([&](int tid, int nt) {
    amx_config();
    vnni_pack_par(pool, tid, nt, x, M, H, Mpad, xv);
    static thread_local std::vector<float> cvec;
    static thread_local std::vector<uint16_t> wvec;
    struct {
      float *p;
      float *data() { return p; }
    } cbuf{tls_buf(cvec, static_cast<size_t>(2) * nbt * 256)};
    struct {
      uint16_t *p;
      uint16_t *data() { return p; }
    } wbuf{tls_buf(wvec, static_cast<size_t>(32) * std::max(H, I))};
    const int ob = I / 16;
    for (int o; (o = next1.fetch_add(1, std::memory_order_relaxed)) < ob;) {
      const int i0 = o * 16;
      const size_t grow = static_cast<size_t>((i0 / kIlv) * 2 * kIlv + i0 % kIlv);
      dequant_rows_q4(v.n13 + grow * (H / 2), v.s13 + grow * (H / 128), 16, H, wbuf.data());
      dequant_rows_q4(v.n13 + (grow + kIlv) * (H / 2), v.s13 + (grow + kIlv) * (H / 128), 16, H,
                      wbuf.data() + static_cast<size_t>(16) * H);
      auto rowp = [&](int, int which) { return wbuf.data() + static_cast<size_t>(which) * 16 * H; };
      amx_gemm_units(rowp, 0, 1, static_cast<size_t>(H) * 2, xv, Mpad, H, cbuf.data());
      for (int b = 0; b < nbt; ++b) {
        const int tok0 = b * 16;
        if (tok0 >= M) {
          for (int r = 0; r < 16; r += 2)
            _mm512_storeu_si512(hv + (static_cast<size_t>((i0 + r) >> 1) * Mpad + tok0) * 2, _mm512_setzero_si512());
          continue;
        }
        const __mmask16 live = tok0 + 16 <= M ? 0xFFFF : static_cast<__mmask16>((1u << (M - tok0)) - 1u);
        const float *cg = cbuf.data() + static_cast<size_t>(b) * 256;
        const float *cu = cbuf.data() + (static_cast<size_t>(nbt) + b) * 256;
        for (int r = 0; r < 16; r += 2) {
          const __m512 h0 = _mm512_maskz_mov_ps(live, silu_mul16(cg + r * 16, cu + r * 16));
          const __m512 h1 = _mm512_maskz_mov_ps(live, silu_mul16(cg + (r + 1) * 16, cu + (r + 1) * 16));
          _mm512_storeu_si512(hv + (static_cast<size_t>((i0 + r) >> 1) * Mpad + tok0) * 2, interleave_bf16(h0, h1));
        }
      }
    }
    pool.barrier();
    const int pairs = H / 32;
    const __m512i col = _mm512_set_epi32(240, 224, 208, 192, 176, 160, 144, 128, 112, 96, 80, 64, 48, 32, 16, 0);
    for (int q; (q = next2.fetch_add(1, std::memory_order_relaxed)) < pairs;) {
      dequant_rows_q4(v.n2 + static_cast<size_t>(q * 32) * (I / 2), v.s2 + static_cast<size_t>(q * 32) * (I / 128),
                      32, I, wbuf.data());
      auto rowp = [&](int, int which) { return wbuf.data() + static_cast<size_t>(which) * 16 * I; };
      amx_gemm_units(rowp, 0, 1, static_cast<size_t>(I) * 2, hv, Mpad, I, cbuf.data());
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < nbt; ++b) {
          const float *c = cbuf.data() + (static_cast<size_t>(a) * nbt + b) * 256;
          for (int t = 0; t < 16; ++t) {  // column t of C = token t's 16 outputs
            const int tok = b * 16 + t;
            if (tok >= M) break;
            _mm512_storeu_ps(out + static_cast<size_t>(tok) * H + q * 32 + a * 16, _mm512_i32gather_ps(col, c + t, 4));
          }
        }
    }
  });
}

bool amx_available() { return amx_enable(); }

void cpu_expert_amx(ThreadPool &pool, const uint16_t *img, int H, int I, const uint16_t *x, int M, float *out,
                    std::vector<uint16_t> &scratch) {
  if ((amx_algo() == 1 || (amx_algo() < 0 && M >= 256)) && H % 32 == 0) {
    cpu_expert_amx2(pool, img, H, I, x, M, out, scratch);
    return;
  }
  const int Mpad = (M + 15) / 16 * 16;
  scratch.resize(static_cast<size_t>(H) * Mpad + static_cast<size_t>(I) * Mpad);
  uint16_t *xv = scratch.data();
  uint16_t *hv = xv + static_cast<size_t>(H) * Mpad;
  // (phase 1 writes every (pair, token block) of hv, padded tokens as zeros)
  const uint16_t *w2 = img + static_cast<size_t>(2) * I * H;
  const int nb = Mpad / 16;
  if (g_dec_prof_on && g_dec_prof.size() < static_cast<size_t>(pool.size()) * 4)
    g_dec_prof.assign(static_cast<size_t>(pool.size()) * 4, 0);
  const int64_t t_call = g_dec_prof_on ? ns_now() : 0;
  // units are claimed dynamically: with static splits one slowed core held
  // each phase barrier (measured: phase-1 max 2.5x the median thread)
  std::atomic<int> next1{0}, next2{0};
  pool.run([&](int tid, int nt) {
    int64_t *tp = g_dec_prof_on ? &g_dec_prof[static_cast<size_t>(tid) * 4] : nullptr;
    if (tp) tp[0] = ns_now() - t_call;
    amx_config();
    vnni_pack_par(pool, tid, nt, x, M, H, Mpad, xv);
    if (tp) tp[1] = ns_now() - t_call;
    float c[4][16][16];
    // phase 1: 16-output blocks of gate rows with their up rows (128-row interleave)
    const int ob = I / 16;
    for (int o; (o = next1.fetch_add(1, std::memory_order_relaxed)) < ob;) {
      const int i0 = o * 16;
      const size_t grow = static_cast<size_t>((i0 / kIlv) * 2 * kIlv + i0 % kIlv);
      const uint16_t *wg = img + grow * H, *wu = img + (grow + kIlv) * H;
      for (int b = 0; b < nb; b += 2) {
        const bool two = b + 1 < nb;
        amx_block(wg, wu, static_cast<size_t>(H) * 2, xv, Mpad, b * 16, two, H, c);
        for (int bb = 0; bb < (two ? 2 : 1); ++bb) {
          const int tok0 = (b + bb) * 16;
          const __mmask16 live = tok0 + 16 <= M ? 0xFFFF : static_cast<__mmask16>((1u << (M - tok0)) - 1u);
          for (int r = 0; r < 16; r += 2) {  // rows r, r+1 -> one 64-byte VNNI row of hv
            const __m512 h0 = _mm512_maskz_mov_ps(live, silu_mul16(c[bb][r], c[2 + bb][r]));
            const __m512 h1 = _mm512_maskz_mov_ps(live, silu_mul16(c[bb][r + 1], c[2 + bb][r + 1]));
            _mm512_storeu_si512(hv + (static_cast<size_t>((i0 + r) >> 1) * Mpad + tok0) * 2, interleave_bf16(h0, h1));
          }
        }
      }
    }
    if (tp) tp[2] = ns_now() - t_call;
    pool.barrier();
    // phase 2: pairs of 16-row blocks of W2
    const int rb = H / 16;
    const int pairs = (rb + 1) / 2;
    const __m512i col = _mm512_set_epi32(240, 224, 208, 192, 176, 160, 144, 128, 112, 96, 80, 64, 48, 32, 16, 0);
    for (int q; (q = next2.fetch_add(1, std::memory_order_relaxed)) < pairs;) {
      const int j0 = q * 32;
      const bool second = j0 + 16 < H;
      const uint16_t *wa0 = w2 + static_cast<size_t>(j0) * I;
      const uint16_t *wa1 = second ? wa0 + static_cast<size_t>(16) * I : wa0;
      for (int b = 0; b < nb; b += 2) {
        const bool two = b + 1 < nb;
        amx_block(wa0, wa1, static_cast<size_t>(I) * 2, hv, Mpad, b * 16, two, I, c);
        // C is [weight row][token]: token t's 16 outputs are column t -- one
        // gather and one 64-byte store per token (was 16 scalar stores)
        for (int a = 0; a < (second ? 2 : 1); ++a)
          for (int bb = 0; bb < (two ? 2 : 1); ++bb)
            for (int t = 0; t < 16; ++t) {
              const int tok = (b + bb) * 16 + t;
              if (tok >= M) break;
              _mm512_storeu_ps(out + static_cast<size_t>(tok) * H + j0 + a * 16,
                               _mm512_i32gather_ps(col, &c[a * 2 + bb][0][t], 4));
            }
      }
    }
    if (tp) tp[3] = ns_now() - t_call;
  });
}

// A layer's multi-token CPU experts (prefill) in ONE pool run: activations of
// every expert VNNI-packed in parallel, then phase 1 over every (expert, 16-pair
// unit) and phase 2 over every (expert, 32-row unit), claimed dynamically across
// experts -- one wake-up and two barriers per layer instead of per expert, and
// the units of all experts fill each other's tails.  Per unit the arithmetic is
// cpu_expert_amx's (bit-identical outputs).
void cpu_experts_amx(ThreadPool &pool, const uint16_t *const *imgs, const uint16_t *const *xs, const int *Ms, int n,
                     int H, int I, float *const *outs, std::vector<uint16_t> &scratch,
                     const std::function<void()> *before_self) {
  HM_REQUIRE(H % 32 == 0 && I % kIlv == 0, HM_EVALUE, "host worker needs H % 32 == 0 and I % 128 == 0");
  HM_REQUIRE(amx_enable(), HM_ERUNTIME, "multi-token host experts need AMX");
  if (n <= 0) {
    if (before_self) (*before_self)();
    return;
  }
  std::vector<size_t> off_x(n), off_h(n);
  std::vector<int> mpad(n);
  size_t total = 0;
  for (int e = 0; e < n; ++e) {
    HM_REQUIRE(Ms[e] >= 1, HM_EVALUE, "every batched expert needs at least one token");
    mpad[e] = (Ms[e] + 15) / 16 * 16;
    off_x[e] = total;
    total += static_cast<size_t>(H) * mpad[e];
    off_h[e] = total;
    total += static_cast<size_t>(I) * mpad[e];
  }
  scratch.resize(total);
  uint16_t *base = scratch.data();
  const int K2 = H / 2, pk = 64;              // pack units: 64 k-pairs of one expert
  const int npk = (K2 + pk - 1) / pk;
  const int ob = I / 16, pairs = (H / 16 + 1) / 2;
  std::atomic<int> next0{0}, next1{0}, next2{0};
  pool.run([&](int tid, int nt) {
    amx_config();
    for (int u; (u = next0.fetch_add(1, std::memory_order_relaxed)) < n * npk;) {
      const int e = u / npk, k0 = (u % npk) * pk;
      vnni_pack_rows(xs[e], Ms[e], H, mpad[e], base + off_x[e], k0, std::min(K2, k0 + pk));
    }
    pool.barrier();
    float c[4][16][16];
    for (int u; (u = next1.fetch_add(1, std::memory_order_relaxed)) < n * ob;) {
      const int e = u / ob, o = u % ob, M = Ms[e], Mpad = mpad[e], nb = Mpad / 16;
      const uint16_t *img = imgs[e], *xv = base + off_x[e];
      uint16_t *hv = base + off_h[e];
      const int i0 = o * 16;
      const size_t grow = static_cast<size_t>((i0 / kIlv) * 2 * kIlv + i0 % kIlv);
      const uint16_t *wg = img + grow * H, *wu = img + (grow + kIlv) * H;
      for (int b = 0; b < nb; b += 2) {
        const bool two = b + 1 < nb;
        amx_block(wg, wu, static_cast<size_t>(H) * 2, xv, Mpad, b * 16, two, H, c);
        for (int bb = 0; bb < (two ? 2 : 1); ++bb) {
          const int tok0 = (b + bb) * 16;
          const __mmask16 live = tok0 + 16 <= M ? 0xFFFF : static_cast<__mmask16>((1u << (M - tok0)) - 1u);
          for (int r = 0; r < 16; r += 2) {
            const __m512 h0 = _mm512_maskz_mov_ps(live, silu_mul16(c[bb][r], c[2 + bb][r]));
            const __m512 h1 = _mm512_maskz_mov_ps(live, silu_mul16(c[bb][r + 1], c[2 + bb][r + 1]));
            _mm512_storeu_si512(hv + (static_cast<size_t>((i0 + r) >> 1) * Mpad + tok0) * 2, interleave_bf16(h0, h1));
          }
        }
      }
    }
    pool.barrier();
    const __m512i col = _mm512_set_epi32(240, 224, 208, 192, 176, 160, 144, 128, 112, 96, 80, 64, 48, 32, 16, 0);
    for (int u; (u = next2.fetch_add(1, std::memory_order_relaxed)) < n * pairs;) {
      const int e = u / pairs, q = u % pairs, M = Ms[e], Mpad = mpad[e], nb = Mpad / 16;
      const uint16_t *w2 = imgs[e] + static_cast<size_t>(2) * I * H, *hv = base + off_h[e];
      float *out = outs[e];
      const int j0 = q * 32;
      const bool second = j0 + 16 < H;
      const uint16_t *wa0 = w2 + static_cast<size_t>(j0) * I;
      const uint16_t *wa1 = second ? wa0 + static_cast<size_t>(16) * I : wa0;
      for (int b = 0; b < nb; b += 2) {
        const bool two = b + 1 < nb;
        amx_block(wa0, wa1, static_cast<size_t>(I) * 2, hv, Mpad, b * 16, two, I, c);
        for (int a = 0; a < (second ? 2 : 1); ++a)
          for (int bb = 0; bb < (two ? 2 : 1); ++bb)
            for (int t = 0; t < 16; ++t) {
              const int tok = (b + bb) * 16 + t;
              if (tok >= M) break;
              _mm512_storeu_ps(out + static_cast<size_t>(tok) * H + j0 + a * 16,
                               _mm512_i32gather_ps(col, &c[a * 2 + bb][0][t], 4));
            }
      }
    }
  }, before_self);
}

void cpu_experts_decode(ThreadPool &pool, const uint16_t *const *imgs, const uint16_t *const *xs, int n, int H,
                        int I, float *const *outs, std::vector<uint16_t> &hbuf,
                        const std::function<void()> *before_self) {
  if (g_dec_prof_on && g_dec_prof.size() < static_cast<size_t>(pool.size()) * 4)
    g_dec_prof.assign(static_cast<size_t>(pool.size()) * 4, 0);
  // All single-token experts of a layer in one pool run: phase 1 over every
  // (expert, 128-pair block), one barrier, phase 2 over every (expert, row).
  HM_REQUIRE(H % 32 == 0 && I % kIlv == 0, HM_EVALUE, "host worker needs H % 32 == 0 and I % 128 == 0");
  if (n <= 0) {
    if (before_self) (*before_self)();
    return;
  }
  hbuf.resize(static_cast<size_t>(n) * I);
  uint16_t *h = hbuf.data();
  const int grain = decode_grain();
  const int64_t t_call = g_dec_prof_on ? ns_now() : 0;
  // per-thread contiguous ranges (phase 1: pairs in grain units, phase 2:
  // rows) with stealing from the tails
  const int nt0 = pool.size();
  const long np1 = static_cast<long>(n) * I, np2 = static_cast<long>(n) * H;
  const int g1 = grain > 0 ? grain : kIlv;
  {
    const long nu = (np1 + g1 - 1) / g1;
    ThreadPool::Range *r1 = pool.ranges(0), *r2 = pool.ranges(1);
    for (int t = 0; t < nt0; ++t) {
      const uint64_t f1 = static_cast<uint64_t>(std::min(np1, nu * t / nt0 * g1));
      const uint64_t b1 = static_cast<uint64_t>(std::min(np1, nu * (t + 1) / nt0 * g1));
      r1[t].fb.store((f1 << 32) | b1, std::memory_order_relaxed);
      const uint64_t f2 = static_cast<uint64_t>(np2 * t / nt0), b2 = static_cast<uint64_t>(np2 * (t + 1) / nt0);
      r2[t].fb.store((f2 << 32) | b2, std::memory_order_relaxed);
    }
  }
  // the owner takes grain-aligned runs of >= ~64 KB from its front; thieves take
  // ~steal_kb() KB (HM_STEAL_KB, default 64) from the others' backs
  const long skb = steal_kb();
  const uint32_t c1 = static_cast<uint32_t>(std::max<long>(g1, (64L << 10) / (4L * H) / g1 * g1));
  const uint32_t s1 = static_cast<uint32_t>(std::max<long>(1, (skb << 10) / (4L * H)));
  const uint32_t c2 = static_cast<uint32_t>(std::max<long>(1, (64L << 10) / (2L * I)));
  const uint32_t s2 = static_cast<uint32_t>(std::max<long>(1, (skb << 10) / (2L * I)));
  pool.run([&](int tid, int nt) {
    int64_t *tp = g_dec_prof_on ? &g_dec_prof[static_cast<size_t>(tid) * 4] : nullptr;
    if (tp) tp[0] = ns_now() - t_call;
    run_ranges(pool.ranges(0), tid, nt, c1, [&](uint32_t q0, uint32_t q1) {
      for (long q = q0; q < static_cast<long>(q1);) {
        const int e = static_cast<int>(q / I), i0 = static_cast<int>(q % I);
        const int i1 = static_cast<int>(std::min<long>(I, i0 + (static_cast<long>(q1) - q)));
        phase1_pairs(imgs[e], H, I, xs[e], h + static_cast<size_t>(e) * I, i0, i1);
        q += i1 - i0;
      }
    }, s1);
    if (tp) tp[1] = ns_now() - t_call;
    pool.barrier();
    if (tp) tp[2] = ns_now() - t_call;
    run_ranges(pool.ranges(1), tid, nt, c2, [&](uint32_t u0, uint32_t u1) {
      for (long u = u0; u < static_cast<long>(u1);) {
        const int e = static_cast<int>(u / H), j0 = static_cast<int>(u % H);
        const int j1 = static_cast<int>(std::min<long>(H, j0 + (static_cast<long>(u1) - u)));
        const uint16_t *w2 = imgs[e] + static_cast<size_t>(2) * I * H;
        stream_rows(w2 + static_cast<size_t>(j0) * I, j1 - j0, I, h + static_cast<size_t>(e) * I, outs[e] + j0);
        u += j1 - j0;
      }
    }, s2);
    if (tp) tp[3] = ns_now() - t_call;
  }, before_self);
  if (g_dec_prof_on) {
    int64_t mx[4] = {0, 0, 0, 0};
    for (int t = 0; t < nt0; ++t)
      for (int k = 0; k < 4; ++k)
        if (t > 0 || k > 0) mx[k] = std::max(mx[k], g_dec_prof[static_cast<size_t>(t) * 4 + k]);
    g_dec_acc[0] += 1;
    g_dec_acc[1] += mx[0];
    const int64_t us = mx[0] / 1000;
    ++g_dec_hist[us <= 5 ? 0 : us <= 20 ? 1 : us <= 100 ? 2 : us <= 1000 ? 3 : 4];
    if (static_cast<int>(g_dec_slowest.size()) < nt0) g_dec_slowest.assign(nt0, 0);
    int slow = 1;
    for (int t = 1; t < nt0; ++t)
      if (g_dec_prof[static_cast<size_t>(t) * 4] > g_dec_prof[static_cast<size_t>(slow) * 4]) slow = t;
    ++g_dec_slowest[slow];
    g_dec_acc[2] += g_dec_prof[0];
    g_dec_acc[3] += mx[1];
    g_dec_acc[4] += mx[2];
    g_dec_acc[5] += mx[3];
    g_dec_acc[6] += ns_now() - t_call;
  }
}

void cpu_expert(ThreadPool &pool, const uint16_t *img, int H, int I, const uint16_t *x, int M, float *out,
                std::vector<uint16_t> &hbuf) {
  HM_REQUIRE(H % 32 == 0 && I % kIlv == 0, HM_EVALUE, "host worker needs H % 32 == 0 and I % 128 == 0");
  if (M <= 0) return;
  hbuf.resize(static_cast<size_t>(M) * I);
  uint16_t *h = hbuf.data();
  if (M == 1) {  // decode: one sequential stream per thread in both phases
    const int nblk = I / kIlv;
    const uint16_t *w2 = img + static_cast<size_t>(2) * I * H;
    pool.run([&](int tid, int nt) {
      const int b0 = static_cast<int>(static_cast<long>(nblk) * tid / nt);
      const int b1 = static_cast<int>(static_cast<long>(nblk) * (tid + 1) / nt);
      if (b0 < b1) phase1_stream(img, H, I, x, h, b0, b1);
      pool.barrier();  // h complete
      const int j0 = static_cast<int>(static_cast<long>(H) * tid / nt);
      const int j1 = static_cast<int>(static_cast<long>(H) * (tid + 1) / nt);
      if (j0 < j1) stream_rows(w2 + static_cast<size_t>(j0) * I, j1 - j0, I, h, out + j0);
    });
    return;
  }
  if (M >= 8 && amx_available()) {  // prefill-sized token groups: AMX tiles
    cpu_expert_amx(pool, img, H, I, x, M, out, hbuf);
    return;
  }
  pool.run([&](int tid, int nt) {
    // pairs in multiples of 16 per thread keep each thread on contiguous rows
    const int per = ((I + nt - 1) / nt + 15) / 16 * 16;
    const int i0 = std::min(I, tid * per), i1 = std::min(I, i0 + per);
    if (i0 < i1) phase1(img, H, I, x, M, h, i0, i1);
  });
  pool.run([&](int tid, int nt) {
    const int per = ((H + nt - 1) / nt + 3) / 4 * 4;
    const int j0 = std::min(H, tid * per), j1 = std::min(H, j0 + per);
    if (j0 < j1) phase2(img, H, I, h, M, out, j0, j1);
  });
}

}  // namespace hm

extern "C" {

struct hm_cpu_pool;

int hm_cpu_pool_create(int nthreads, hm_cpu_pool **out) {
  HM_API_BEGIN
  if (nthreads <= 0) nthreads = static_cast<int>(std::thread::hardware_concurrency());
  *out = reinterpret_cast<hm_cpu_pool *>(new hm::ThreadPool(nthreads));
  HM_API_END
}

void hm_cpu_pool_destroy(hm_cpu_pool *p) { delete reinterpret_cast<hm::ThreadPool *>(p); }

int hm_cpu_expert(hm_cpu_pool *pool, const uint16_t *img, int H, int I, const uint16_t *x, int M, float *out) {
  HM_API_BEGIN
  std::vector<uint16_t> hbuf;
  hm::cpu_expert(*reinterpret_cast<hm::ThreadPool *>(pool), img, H, I, x, M, out, hbuf);
  HM_API_END
}

int hm_cpu_experts_amx(hm_cpu_pool *pool, const uint16_t *const *imgs, const uint16_t *const *xs, const int *Ms,
                       int n, int H, int I, float *const *outs) {
  HM_API_BEGIN
  std::vector<uint16_t> scratch;
  hm::cpu_experts_amx(*reinterpret_cast<hm::ThreadPool *>(pool), imgs, xs, Ms, n, H, I, outs, scratch);
  HM_API_END
}

int hm_cpu_experts_decode(hm_cpu_pool *pool, const uint16_t *const *imgs, const uint16_t *const *xs, int n, int H,
                          int I, float *const *outs) {
  HM_API_BEGIN
  std::vector<uint16_t> hbuf;
  hm::cpu_experts_decode(*reinterpret_cast<hm::ThreadPool *>(pool), imgs, xs, n, H, I, outs, hbuf);
  HM_API_END
}

int hm_cpu_expert_q4(hm_cpu_pool *pool, const uint8_t *img, int H, int I, const uint16_t *x, int M, float *out) {
  HM_API_BEGIN
  std::vector<uint16_t> hbuf;
  hm::cpu_expert_q4(*reinterpret_cast<hm::ThreadPool *>(pool), img, H, I, x, M, out, hbuf);
  HM_API_END
}

int hm_cpu_experts_decode_q4(hm_cpu_pool *pool, const uint8_t *const *imgs, const uint16_t *const *xs, int n, int H,
                             int I, float *const *outs) {
  HM_API_BEGIN
  std::vector<uint16_t> hbuf;
  hm::cpu_experts_decode_q4(*reinterpret_cast<hm::ThreadPool *>(pool), imgs, xs, n, H, I, outs, hbuf);
  HM_API_END
}

int hm_cpu_has_avx512bf16(void) { return __builtin_cpu_supports("avx512bf16") ? 1 : 0; }

int hm_cpu_has_amx_bf16(void) { return hm::amx_available() ? 1 : 0; }

// Tuning knob for the decode stream: software-prefetch distance (bf16
// elements) and hint (0 none, 1 T0, 2 T1, 3 NTA).  Process-wide.
int hm_cpu_set_prefetch(int dist, int hint) {
  HM_API_BEGIN
  HM_REQUIRE(dist >= 0 && hint >= 0 && hint <= 3, HM_EVALUE, "bad prefetch setting");
  hm::pf_cfg().dist = dist;
  hm::pf_cfg().hint = hint;
  HM_API_END
}

// Tuning knob for the decode split granularity (pairs; 0 = whole 128-pair blocks).
int hm_cpu_decode_profile(int enable, int64_t *out, int n_threads) {
  HM_API_BEGIN
  hm::g_dec_prof_on = enable != 0;
  if (out)
    for (int i = 0; i < n_threads * 4 && i < static_cast<int>(hm::g_dec_prof.size()); ++i) out[i] = hm::g_dec_prof[i];
  HM_API_END
}

int hm_cpu_decode_profile_accum(int64_t *out7, int reset) {
  HM_API_BEGIN
  if (out7)
    for (int i = 0; i < 7; ++i) out7[i] = hm::g_dec_acc[i];
  if (reset) {
    for (auto &v : hm::g_dec_acc) v = 0;
    for (auto &v : hm::g_dec_hist) v = 0;
    hm::g_dec_slowest.clear();
  }
  HM_API_END
}

int hm_cpu_decode_profile_hist(int64_t *out5, int64_t *slowest, int n_threads) {
  HM_API_BEGIN
  for (int i = 0; i < 5; ++i) out5[i] = hm::g_dec_hist[i];
  if (slowest)
    for (int t = 0; t < n_threads; ++t)
      slowest[t] = t < static_cast<int>(hm::g_dec_slowest.size()) ? hm::g_dec_slowest[t] : 0;
  HM_API_END
}

int hm_cpu_set_decode_steal(int on) {
  HM_API_BEGIN
  hm::decode_steal() = on != 0;
  HM_API_END
}

int hm_cpu_set_decode_grain(int grain) {
  HM_API_BEGIN
  HM_REQUIRE(grain >= 0, HM_EVALUE, "bad decode grain");
  hm::decode_grain() = grain;
  HM_API_END
}

// Host DRAM read bandwidth with the worker pool (the host roofline denominator).
int hm_host_read_bw(hm_cpu_pool *pool, const void *p, size_t bytes, int reps, double *gbs) {
  HM_API_BEGIN
  auto &tp = *reinterpret_cast<hm::ThreadPool *>(pool);
  const size_t n64 = bytes / 64;
  const char *base = static_cast<const char *>(p);
  std::vector<double> sink(static_cast<size_t>(tp.size()), 0.0);
  double best = 0.0;
  for (int r = 0; r < reps; ++r) {
    const auto t0 = std::chrono::steady_clock::now();
    tp.run([&](int tid, int nt) {
      const size_t per = (n64 + nt - 1) / nt;
      const size_t a = std::min(n64, static_cast<size_t>(tid) * per), b = std::min(n64, a + per);
      __m512i acc0 = _mm512_setzero_si512(), acc1 = _mm512_setzero_si512();
      size_t i = a;
      for (; i + 1 < b; i += 2) {
        acc0 = _mm512_xor_si512(acc0, _mm512_load_si512(base + i * 64));
        acc1 = _mm512_xor_si512(acc1, _mm512_load_si512(base + (i + 1) * 64));
      }
      if (i < b) acc0 = _mm512_xor_si512(acc0, _mm512_load_si512(base + i * 64));
      sink[tid] += static_cast<double>(_mm512_reduce_add_epi64(_mm512_xor_si512(acc0, acc1)) & 1);
    });
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    best = std::max(best, static_cast<double>(n64 * 64) / s / 1e9);
  }
  *gbs = best + 0.0 * sink[0];
  HM_API_END
}

}  // extern "C"
