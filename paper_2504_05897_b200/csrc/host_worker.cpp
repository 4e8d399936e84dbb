// Host worker: executes the experts the schedule assigns to the CPU
// (the CPU timeline of scheduling.py:257-268).  bf16 expert
// images are read straight from the pinned host master store in the slot
// layout (include/hybrimoe.h, hm_group); arithmetic is AVX-512 BF16
// (vdpbf16ps: bf16 pairs, fp32 accumulate), the intermediate h is rounded to
// bf16 exactly like the GPU path, outputs are fp32 rows in permuted order.
// Decode (1 token) is a DRAM-bandwidth-bound GEMV split over all threads;
// prefill blocks 16 weight rows x 4 tokens so weights are reused from L2.
#include <immintrin.h>

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

ThreadPool::ThreadPool(int n, int spin_us) : n_(std::max(1, n)), spin_us_(spin_us) {
  for (int t = 1; t < n_; ++t) threads_.emplace_back([this, t] { loop(t); });
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

void ThreadPool::run(const std::function<void(int, int)> &fn) {
  if (n_ == 1) {
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
  fn(0, n_);
  wait_until([&] { return pending_.load(std::memory_order_acquire) == 0; });
}

void ThreadPool::barrier() {
  const uint32_t sense = bar_sense_.load(std::memory_order_acquire);
  if (bar_count_.fetch_add(1, std::memory_order_acq_rel) == n_ - 1) {
    bar_count_.store(0, std::memory_order_relaxed);
    bar_sense_.store(sense + 1, std::memory_order_release);
  } else {
    wait_until([&] { return bar_sense_.load(std::memory_order_acquire) != sense; });
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
struct PfCfg {  // tuned on the B200 box's host (tools/host_bench.py): L2 hint, 32 KB ahead
  int dist = 16384;
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

}  // namespace

void cpu_experts_decode(ThreadPool &pool, const uint16_t *const *imgs, const uint16_t *const *xs, int n, int H,
                        int I, float *const *outs, std::vector<uint16_t> &hbuf) {
  // All single-token experts of a layer in one pool run: phase 1 over every
  // (expert, 128-pair block), one barrier, phase 2 over every (expert, row).
  HM_REQUIRE(H % 32 == 0 && I % kIlv == 0, HM_EVALUE, "host worker needs H % 32 == 0 and I % 128 == 0");
  if (n <= 0) return;
  hbuf.resize(static_cast<size_t>(n) * I);
  uint16_t *h = hbuf.data();
  const int nblk = I / kIlv;
  pool.run([&](int tid, int nt) {
    const long u1 = static_cast<long>(n) * nblk;
    for (long u = u1 * tid / nt; u < u1 * (tid + 1) / nt;) {
      const int e = static_cast<int>(u / nblk), b0 = static_cast<int>(u % nblk);
      const int b1 = static_cast<int>(std::min<long>(nblk, b0 + (u1 * (tid + 1) / nt - u)));
      phase1_stream(imgs[e], H, I, xs[e], h + static_cast<size_t>(e) * I, b0, b1);
      u += b1 - b0;
    }
    pool.barrier();
    const long r1 = static_cast<long>(n) * H;
    for (long u = r1 * tid / nt; u < r1 * (tid + 1) / nt;) {
      const int e = static_cast<int>(u / H), j0 = static_cast<int>(u % H);
      const int j1 = static_cast<int>(std::min<long>(H, j0 + (r1 * (tid + 1) / nt - u)));
      const uint16_t *w2 = imgs[e] + static_cast<size_t>(2) * I * H;
      stream_rows(w2 + static_cast<size_t>(j0) * I, j1 - j0, I, h + static_cast<size_t>(e) * I, outs[e] + j0);
      u += j1 - j0;
    }
  });
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

int hm_cpu_experts_decode(hm_cpu_pool *pool, const uint16_t *const *imgs, const uint16_t *const *xs, int n, int H,
                          int I, float *const *outs) {
  HM_API_BEGIN
  std::vector<uint16_t> hbuf;
  hm::cpu_experts_decode(*reinterpret_cast<hm::ThreadPool *>(pool), imgs, xs, n, H, I, outs, hbuf);
  HM_API_END
}

int hm_cpu_has_avx512bf16(void) { return __builtin_cpu_supports("avx512bf16") ? 1 : 0; }

// Tuning knob for the decode stream: software-prefetch distance (bf16
// elements) and hint (0 none, 1 T0, 2 T1, 3 NTA).  Process-wide.
int hm_cpu_set_prefetch(int dist, int hint) {
  HM_API_BEGIN
  HM_REQUIRE(dist >= 0 && hint >= 0 && hint <= 3, HM_EVALUE, "bad prefetch setting");
  hm::pf_cfg().dist = dist;
  hm::pf_cfg().hint = hint;
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
