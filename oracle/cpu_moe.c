/* ORACLE -- test infrastructure only (tests/, __graft_entry__.smoke(), bench.py's
 * reference arm and cpu_baseline leg).  Not linked into, loaded by or called
 * from the product package.
 *
 * Plain-C restatement of the reference's CPU path for one MoE expert
 * evaluation (the paper's CPU expert, Eq. 1):
 *     out[m] = W2 ( silu(Wg x[m]) * (Wu x[m]) )
 * bf16 weights and activations, fp32 accumulation, h rounded to bf16, the
 * expert image layout of this oracle: W13 rows [gate 0..I-1 | up 0..I-1] x H,
 * then W2 [H][I].  OpenMP over output rows on all host threads; the dot
 * products use AVX-512 BF16 (vdpbf16ps) where the host has it, else 16
 * independent fp32 partial sums.  It exists so the reference arm is the
 * reference's CPU path at full host bandwidth, not a slow library call
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

#ifdef __AVX512BF16__
#include <immintrin.h>
/* bf16 . bf16 with fp32 accumulation: vdpbf16ps (pairs of exact products
 * summed into 16 fp32 lanes), 64 elements per step in two chains. */
static inline float dot_bf16(const uint16_t *w, const uint16_t *x, int n) {
  __m512 a0 = _mm512_setzero_ps(), a1 = _mm512_setzero_ps();
  int c = 0;
  for (; c + 64 <= n; c += 64) {
    a0 = _mm512_dpbf16_ps(a0, (__m512bh)_mm512_loadu_si512(w + c), (__m512bh)_mm512_loadu_si512(x + c));
    a1 = _mm512_dpbf16_ps(a1, (__m512bh)_mm512_loadu_si512(w + c + 32), (__m512bh)_mm512_loadu_si512(x + c + 32));
  }
  float s = _mm512_reduce_add_ps(_mm512_add_ps(a0, a1));
  for (; c < n; ++c) s += bf2f(w[c]) * bf2f(x[c]);
  return s;
}
#else
static inline float dot_bf16(const uint16_t *w, const uint16_t *x, int n) {
  float acc[16] = {0};
  int c = 0;
  for (; c + 16 <= n; c += 16)
    for (int v = 0; v < 16; ++v) acc[v] += bf2f(w[c + v]) * bf2f(x[c + v]);
  float s = 0.f;
  for (int v = 0; v < 16; ++v) s += acc[v];
  for (; c < n; ++c) s += bf2f(w[c]) * bf2f(x[c]);
  return s;
}
#endif

/* x: M rows of H bf16; out: M rows of H fp32; scratch: >= I * M / 2 + 16 floats (h as bf16). */
int oc_expert(const uint16_t *w13, const uint16_t *w2, int H, int I, const uint16_t *x, int M, float *out,
              float *scratch) {
  if (H <= 0 || I <= 0 || M < 0) return 1;
  uint16_t *hb = (uint16_t *)scratch; /* [M][I] bf16 */
#pragma omp parallel for schedule(static)
  for (int i = 0; i < I; ++i) {
    const uint16_t *wg = w13 + (size_t)i * H, *wu = w13 + (size_t)(I + i) * H;
    for (int m = 0; m < M; ++m) {
      const float g = dot_bf16(wg, x + (size_t)m * H, H);
      const float u = dot_bf16(wu, x + (size_t)m * H, H);
      hb[(size_t)m * I + i] = f2bf(g / (1.f + expf(-g)) * u);
    }
  }
#pragma omp parallel for schedule(static)
  for (int j = 0; j < H; ++j)
    for (int m = 0; m < M; ++m) out[(size_t)m * H + j] = dot_bf16(w2 + (size_t)j * I, hb + (size_t)m * I, I);
  return 0;
}

int oc_threads(void);
#ifdef _OPENMP
#include <omp.h>
int oc_threads(void) { return omp_get_max_threads(); }
#else
int oc_threads(void) { return 1; }
#endif
