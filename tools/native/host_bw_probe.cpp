// Host DRAM read-bandwidth probe: which access pattern saturates this host's
// memory system with 16 threads?  Variants: plain 64-byte loads; + software
// prefetch (T0 / T1 / NTA) d bytes ahead; S interleaved streams per thread.
// g++ -O2 -mavx512f -pthread tools/native/host_bw_probe.cpp -o /tmp/host_bw_probe
#include <immintrin.h>
#include <sys/mman.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static char *buf;
static size_t total;

template <int HINT>
static double run(int nt, int streams, size_t pf, size_t bytes_per_call, int calls) {
  std::atomic<int> go{0};
  std::vector<double> sink(nt * 8);
  std::vector<std::thread> th;
  auto t0 = std::chrono::steady_clock::now();
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      __m512i acc = _mm512_setzero_si512();
      for (int c = 0; c < calls; ++c) {
        // call c reads [base, base + bytes_per_call), thread t its slice, as `streams` sub-streams
        const size_t base = (static_cast<size_t>(c) * bytes_per_call * 7) % (total - bytes_per_call);
        const size_t per = bytes_per_call / nt / 64 * 64;
        const char *p = buf + base + per * t;
        const size_t sub = per / streams / 64 * 64;
        for (size_t o = 0; o < sub; o += 64) {
          for (int s = 0; s < streams; ++s) {
            const char *q = p + s * sub + o;
            if (HINT >= 0 && pf) _mm_prefetch(q + pf, static_cast<_mm_hint>(HINT));
            acc = _mm512_xor_si512(acc, _mm512_load_si512(q));
          }
        }
      }
      sink[t * 8] = static_cast<double>(_mm512_reduce_add_epi64(acc) & 1);
    });
  for (auto &x : th) x.join();
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return static_cast<double>(bytes_per_call) * calls / s / 1e9 + 0 * sink[0];
}

int main(int argc, char **argv) {
  const int nt = argc > 1 ? std::atoi(argv[1]) : 16;
  total = static_cast<size_t>(16) << 30;
  buf = static_cast<char *>(aligned_alloc(2 << 20, total));
  madvise(buf, total, MADV_NOHUGEPAGE);
  std::memset(buf, 1, total);
  const size_t call = 352u << 20;  // one Mixtral expert
  const int calls = 12;
  std::printf("threads %d, %zu MB per call\n", nt, call >> 20);
  for (int streams : {1, 2, 4}) {
    std::printf("streams %d: plain %.1f GB/s", streams, run<-1>(nt, streams, 0, call, calls));
    for (size_t pf : {2048, 8192, 16384, 65536}) {
      std::printf(" | T0 %zuK %.1f", pf >> 10, run<_MM_HINT_T0>(nt, streams, pf, call, calls));
      std::printf(" T1 %zuK %.1f", pf >> 10, run<_MM_HINT_T1>(nt, streams, pf, call, calls));
    }
    std::printf(" | NTA 8K %.1f\n", run<_MM_HINT_NTA>(nt, streams, 8192, call, calls));
  }
}
