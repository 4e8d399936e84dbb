// AMX-BF16 throughput probe on the host (one thread per core, all cores):
//  peak:  4 independent C tiles, A/B tiles resident (no loads in the loop)
//  l1:    2 A + 2 B tile loads per step from a 4 KB L1-resident block
//  l2:    the same from a 1 MB per-thread buffer (L2-resident), strided like weight rows
// g++ -O2 -mamx-tile -mamx-bf16 -mavx512f -pthread tools/native/amx_probe.cpp -o /tmp/amx_probe
#include <immintrin.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

struct alignas(64) Cfg {
  uint8_t palette = 1, start = 0, res[14] = {};
  uint16_t colsb[16] = {};
  uint8_t rows[16] = {};
};

static double run(int mode, int nthreads, long iters) {
  std::atomic<int> go{0};
  std::vector<double> dt(nthreads);
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t)
    th.emplace_back([&, t] {
      Cfg c;
      for (int i = 0; i < 8; ++i) {
        c.colsb[i] = 64;
        c.rows[i] = 16;
      }
      _tile_loadconfig(&c);
      const size_t nb = mode == 2 ? (1 << 20) : 8192;
      uint16_t *buf = static_cast<uint16_t *>(aligned_alloc(64, nb));
      for (size_t i = 0; i < nb / 2; ++i) buf[i] = 0x3f80;
      float cst[256];
      _tile_zero(0); _tile_zero(1); _tile_zero(2); _tile_zero(3);
      _tile_loadd(4, buf, 64); _tile_loadd(5, buf, 64); _tile_loadd(6, buf, 64); _tile_loadd(7, buf, 64);
      while (!go.load()) {}
      auto t0 = std::chrono::steady_clock::now();
      if (mode == 0) {
        for (long i = 0; i < iters; ++i) {
          _tile_dpbf16ps(0, 4, 6); _tile_dpbf16ps(1, 4, 7); _tile_dpbf16ps(2, 5, 6); _tile_dpbf16ps(3, 5, 7);
        }
      } else if (mode == 1) {
        for (long i = 0; i < iters; ++i) {
          _tile_loadd(4, buf, 64); _tile_loadd(5, buf + 512, 64); _tile_loadd(6, buf + 1024, 64); _tile_loadd(7, buf + 1536, 64);
          _tile_dpbf16ps(0, 4, 6); _tile_dpbf16ps(1, 4, 7); _tile_dpbf16ps(2, 5, 6); _tile_dpbf16ps(3, 5, 7);
        }
      } else {
        // A: 2 x 16 rows of a [32 rows][8 KB] block (stride 8 KB), B: contiguous 1 KB tiles
        const size_t lda = 8192;
        const char *a = reinterpret_cast<const char *>(buf);
        const char *b = a + 32 * lda;
        for (long i = 0; i < iters; ++i) {
          const int k = static_cast<int>(i % 128) * 64;
          _tile_loadd(4, a + k, lda); _tile_loadd(5, a + 16 * lda + k, lda);
          _tile_loadd(6, b + (i % 128) * 2048, 64); _tile_loadd(7, b + (i % 128) * 2048 + 1024, 64);
          _tile_dpbf16ps(0, 4, 6); _tile_dpbf16ps(1, 4, 7); _tile_dpbf16ps(2, 5, 6); _tile_dpbf16ps(3, 5, 7);
        }
      }
      _tile_stored(0, cst, 64);
      dt[t] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      free(buf);
    });
  go = 1;
  for (auto &x : th) x.join();
  double mx = 0;
  for (double d : dt) mx = mx > d ? mx : d;
  return 4.0 * 16 * 16 * 32 * 2 * iters * nthreads / mx / 1e12;
}

int main(int argc, char **argv) {
  if (syscall(SYS_arch_prctl, 0x1023, 18) != 0) { std::puts("no AMX permission"); return 1; }
  const int nt = argc > 1 ? std::atoi(argv[1]) : static_cast<int>(std::thread::hardware_concurrency());
  const long iters = 2000000;
  for (int mode = 0; mode < 3; ++mode) {
    const char *name[] = {"peak(no loads)", "L1 loads", "L2 strided A"};
    std::printf("%-16s 1 thread: %6.2f TF/s   %d threads: %6.2f TF/s\n", name[mode], run(mode, 1, iters),
                nt, run(mode, nt, iters));
  }
}
