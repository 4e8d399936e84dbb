/* ORACLE -- test infrastructure only (tests/, __graft_entry__.smoke(), bench.py's
 * reference arm and cpu_baseline leg).  Not linked into, loaded by or called
 * from the product package.
 *
 * Plain-C restatement of the reference's CPU path for one MoE expert
 * evaluation (the paper's CPU expert, Eq. 1):
 *     out[m] = W2 ( silu(Wg x[m]) * (Wu x[m]) )
 * bf16 weights and activations, fp32 accumulation, h rounded to bf16, the
 * expert image layout of this oracle: W13 rows [gate 0..I-1 | up 0..I-1] x H,
 * then W2 [H][I].  OpenMP over output rows on all host threads; the inner
 * loops keep 16 independent fp32 partial sums so the compiler vectorises them
 * without reassociating a single accumulator.  It exists so the reference arm
 * is the reference's CPU path at full host bandwidth, not a slow library call
 * (torch CPU's bf16 GEMV streams at 20-40 GB/s on these hosts).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

static inline float bf2f(uint16_t v) {
  uint32_t u = (uint32_t)v << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static inline uint16_t f2bf(float f) { /* round to nearest even (finite inputs) */
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

static inline float dot_bf16(const uint16_t *w, const float *x, int n) {
  float acc[16] = {0};
  int c = 0;
  for (; c + 16 <= n; c += 16)
    for (int v = 0; v < 16; ++v) acc[v] += bf2f(w[c + v]) * x[c + v];
  float s = 0.f;
  for (int v = 0; v < 16; ++v) s += acc[v];
  for (; c < n; ++c) s += bf2f(w[c]) * x[c];
  return s;
}

/* x: M rows of H bf16; out: M rows of H fp32; scratch: (H + I) * M floats. */
int oc_expert(const uint16_t *w13, const uint16_t *w2, int H, int I, const uint16_t *x, int M, float *out,
              float *scratch) {
  if (H <= 0 || I <= 0 || M < 0) return 1;
  float *xf = scratch;             /* [M][H] */
  float *hf = scratch + (size_t)M * H; /* [M][I] */
  for (size_t i = 0; i < (size_t)M * H; ++i) xf[i] = bf2f(x[i]);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < I; ++i) {
    const uint16_t *wg = w13 + (size_t)i * H, *wu = w13 + (size_t)(I + i) * H;
    for (int m = 0; m < M; ++m) {
      const float g = dot_bf16(wg, xf + (size_t)m * H, H);
      const float u = dot_bf16(wu, xf + (size_t)m * H, H);
      hf[(size_t)m * I + i] = bf2f(f2bf(g / (1.f + expf(-g)) * u));
    }
  }
#pragma omp parallel for schedule(static)
  for (int j = 0; j < H; ++j)
    for (int m = 0; m < M; ++m) out[(size_t)m * H + j] = dot_bf16(w2 + (size_t)j * I, hf + (size_t)m * I, I);
  return 0;
}

int oc_threads(void);
#ifdef _OPENMP
#include <omp.h>
int oc_threads(void) { return omp_get_max_threads(); }
#else
int oc_threads(void) { return 1; }
#endif
