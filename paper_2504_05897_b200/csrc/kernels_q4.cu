// 4-bit expert weights (the paper runs Marlin 4-bit
// experts; the reference's default bytes_per_weight is 0.5,
// core.py:55).  Weight-only int4, symmetric, one bf16 scale per 128 weights
// of a row:  w = (nibble - 8) * scale.
//
// Expert image (bytes), rows in the same order as the bf16 image (W13 with
// gate/up rows interleaved in 128-row blocks, then W2):
//   [0, HI)                 W13 nibbles  [2I rows][H/2]   (element 2k: low nibble of byte k)
//   [HI, 3HI/2)             W2 nibbles   [H rows][I/2]
//   [3HI/2, +2I*H/64)       W13 scales   [2I rows][H/128] bf16
//   [.., +H*I/64)           W2 scales    [H rows][I/128]  bf16
// = 3HI/2 + 3HI/64 bytes (expert_bytes at bytes_per_weight 0.5, plus 3.1 % scales).
//
// Kernels: quantize (bf16 image -> q4 image), dequantize (q4 -> bf16 image,
// feeding the tcgen05 GEMM for prefill-sized groups), and the decode GEMV on
// the q4 image: activations staged per 32-element block as two int8 digits
// (x ~= sx * (hi + lo/256)), nibble words masked into bytes and multiplied
// with DP4A (4 MACs per instruction, exact int32), fp32 across blocks.
#include <cstdlib>
#include <vector>

#include "device.cuh"

namespace hm {
namespace {

constexpr int kQG = 128;  // weights per scale
constexpr int kQ4MaxGroups = 96;
constexpr int kIlvQ = 128;

struct Q4Layout {
  size_t w2_off, s13_off, s2_off, bytes;
};
__host__ __device__ inline Q4Layout q4_layout(int H, int I) {
  const size_t hi = static_cast<size_t>(H) * I;
  Q4Layout l;
  l.w2_off = hi;
  l.s13_off = hi + hi / 2;
  l.s2_off = l.s13_off + static_cast<size_t>(2) * I * (H / kQG) * 2;
  l.bytes = l.s2_off + static_cast<size_t>(H) * (I / kQG) * 2;
  return l;
}

// one thread per (row, 128-group) of W13 then W2
__global__ void q4_quantize_kernel(const uint16_t *__restrict__ img, int H, int I, uint8_t *__restrict__ q) {
  const Q4Layout L = q4_layout(H, I);
  const long g13 = static_cast<long>(2) * I * (H / kQG), g2 = static_cast<long>(H) * (I / kQG);
  const long t = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= g13 + g2) return;
  const bool w13 = t < g13;
  const long tt = w13 ? t : t - g13;
  const int K = w13 ? H : I, gpr = K / kQG;
  const long row = tt / gpr, grp = tt % gpr;
  const uint16_t *src = img + (w13 ? 0 : static_cast<size_t>(2) * I * H) + row * K + grp * kQG;
  float mx = 0.f;
  for (int i = 0; i < kQG; ++i) mx = fmaxf(mx, fabsf(dev::bf2f(src[i])));
  const uint16_t sb = dev::f2bf(mx / 7.0f);
  const float s = dev::bf2f(sb);
  uint8_t *dst = q + (w13 ? 0 : L.w2_off) + row * (K / 2) + grp * (kQG / 2);
  for (int i = 0; i < kQG; i += 2) {
    int a = 8, b = 8;
    if (s > 0.f) {
      a = 8 + max(-8, min(7, __float2int_rn(dev::bf2f(src[i]) / s)));
      b = 8 + max(-8, min(7, __float2int_rn(dev::bf2f(src[i + 1]) / s)));
    }
    dst[i / 2] = static_cast<uint8_t>(a | (b << 4));
  }
  reinterpret_cast<uint16_t *>(q + (w13 ? L.s13_off : L.s2_off))[row * gpr + grp] = sb;
}

__global__ void q4_dequantize_kernel(const uint8_t *__restrict__ q, int H, int I, uint16_t *__restrict__ img) {
  const Q4Layout L = q4_layout(H, I);
  const long g13 = static_cast<long>(2) * I * (H / kQG), g2 = static_cast<long>(H) * (I / kQG);
  const long t = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= g13 + g2) return;
  const bool w13 = t < g13;
  const long tt = w13 ? t : t - g13;
  const int K = w13 ? H : I, gpr = K / kQG;
  const long row = tt / gpr, grp = tt % gpr;
  const float s = dev::bf2f(reinterpret_cast<const uint16_t *>(q + (w13 ? L.s13_off : L.s2_off))[row * gpr + grp]);
  const uint8_t *src = q + (w13 ? 0 : L.w2_off) + row * (K / 2) + grp * (kQG / 2);
  uint16_t *dst = img + (w13 ? 0 : static_cast<size_t>(2) * I * H) + row * K + grp * kQG;
  for (int i = 0; i < kQG / 2; ++i) {
    const uint8_t b = src[i];
    dst[2 * i] = dev::f2bf(static_cast<float>((b & 15) - 8) * s);
    dst[2 * i + 1] = dev::f2bf(static_cast<float>((b >> 4) - 8) * s);
  }
}

// Activations for the int4 GEMV: per 32-element block b, scale sx = max|x|/127
// and two int8 digits per element, x ~= sx * (hi + lo/256) (|error| <= sx/512,
// i.e. ~1e-5 of the block max), split into even / odd elements so that the
// DP4A against a nibble word's low (even elements) and high (odd) nibbles
// multiplies matching pairs.  Shared memory: four planes of 16 int8 per block
// (even hi | odd hi | even lo | odd lo, each plane [nb][16]), then sx[nb] and
// sq[nb] = sum(hi) + sum(lo)/256.  Lane L reads block j*32 + L of each plane:
// consecutive lanes, consecutive 16-byte words (a [nb][64] layout put lanes
// 64 B apart and cost 4-way bank conflicts on every load).
__host__ __device__ inline int q4_pad(int K) { return (K + 1023) / 1024 * 1024; }
__host__ __device__ inline int q4_stage_bytes(int K) { return q4_pad(K) / 32 * 72; }

__device__ void stage_x_q8(const uint16_t *__restrict__ x, int K, uint8_t *st) {
  const int nb = q4_pad(K) / 32;
  int4 *planes = reinterpret_cast<int4 *>(st);  // plane p, block b: planes[p * nb + b]
  float *sx = reinterpret_cast<float *>(st + static_cast<size_t>(nb) * 64);
  float *sq = sx + nb;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    if (b * 32 >= K) {  // padding block: zeros
      const int4 z = make_int4(0, 0, 0, 0);
      planes[b] = planes[nb + b] = planes[2 * nb + b] = planes[3 * nb + b] = z;
      sx[b] = 0.f;
      sq[b] = 0.f;
      continue;
    }
    float v[32], m = 0.f;
    const uint4 *src = reinterpret_cast<const uint4 *>(x + static_cast<size_t>(b) * 32);
#pragma unroll
    for (int c = 0; c < 4; ++c) {  // 4 x 16-byte loads = 32 bf16
      const uint4 u = src[c];
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        v[c * 8 + 2 * j] = dev::bf_lo(w[j]);
        v[c * 8 + 2 * j + 1] = dev::bf_hi(w[j]);
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) m = fmaxf(m, fabsf(v[i]));
    const float s = m > 0.f ? m / 127.f : 1.f, inv = 1.f / s;
    uint32_t pk[4][4];  // [plane][word]
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int w = 0; w < 4; ++w) pk[p][w] = 0u;
    int sh = 0, sl = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float t = v[i] * inv;
      const float hi = rintf(t);
      const int lo = max(-127, min(127, __float2int_rn((t - hi) * 256.f)));
      const int hq = static_cast<int>(hi);
      const int k = i >> 1, word = k >> 2, sh8 = (k & 3) * 8;  // byte k of the plane
      pk[i & 1][word] |= (static_cast<uint32_t>(hq) & 0xFFu) << sh8;        // even / odd hi
      pk[2 + (i & 1)][word] |= (static_cast<uint32_t>(lo) & 0xFFu) << sh8;  // even / odd lo
      sh += hq;
      sl += lo;
    }
#pragma unroll
    for (int p = 0; p < 4; ++p)
      planes[p * nb + b] = make_int4(static_cast<int>(pk[p][0]), static_cast<int>(pk[p][1]),
                                     static_cast<int>(pk[p][2]), static_cast<int>(pk[p][3]));
    sx[b] = s;
    sq[b] = static_cast<float>(sh) + static_cast<float>(sl) * (1.f / 256.f);
  }
}

// One staged 32-element activation block: the four digit planes + scales.
struct XChunk {
  int eh[4], oh[4], el[4], ol[4];
  float sx, sq;
};
__device__ __forceinline__ XChunk load_xchunk(const uint8_t *st, int nb, int b) {
  const int4 *pl = reinterpret_cast<const int4 *>(st) + b;
  const int4 eh = pl[0], oh = pl[nb], el = pl[2 * nb], ol = pl[3 * nb];
  const float *f = reinterpret_cast<const float *>(st + static_cast<size_t>(nb) * 64);
  return XChunk{{eh.x, eh.y, eh.z, eh.w}, {oh.x, oh.y, oh.z, oh.w}, {el.x, el.y, el.z, el.w},
                {ol.x, ol.y, ol.z, ol.w}, f[b], f[nb + b]};
}

// 32 weights (one 16-byte nibble load) of a row against a staged block ->
// sum_k (n_k - 8) x_k in fp32
__device__ __forceinline__ float q4_dot32(const uint4 w, const XChunk &x) {
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
  int ah = 0, al = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int lo = static_cast<int>(ws[q] & 0x0F0F0F0Fu);         // elements 8q + 0, 2, 4, 6
    const int hi = static_cast<int>((ws[q] >> 4) & 0x0F0F0F0Fu);  // elements 8q + 1, 3, 5, 7
    ah = __dp4a(lo, x.eh[q], ah);
    ah = __dp4a(hi, x.oh[q], ah);
    al = __dp4a(lo, x.el[q], al);
    al = __dp4a(hi, x.ol[q], al);
  }
  return x.sx * (static_cast<float>(ah) + static_cast<float>(al) * (1.f / 256.f) - 8.f * x.sq);
}

// NR rows (sharing x) dotted with the M staged activation rows; each lane
// handles 32-weight chunks lane*32 + 1024*j, U chunks per row loaded before
// any is consumed.  Every weight byte is loaded once for all M rows, and every
// staged activation block once for all NR rows: shared-memory traffic per
// weight byte is 4M/NR (it was 4 per row and token -- the kernel was bound by
// it, not by HBM).  Returns the lane's partials acc[m][r].
template <int MR, int NR, int U>
__device__ __forceinline__ void q4_rows_dot(const uint8_t *const (&rows)[NR], const uint16_t *const (&sc)[NR],
                                            const bool (&live)[NR], const uint8_t *st, int stage_bytes, int M, int K,
                                            int lane, float (&acc)[MR][NR]) {
  const int nb = q4_pad(K) / 32;
#pragma unroll
  for (int m = 0; m < MR; ++m)
#pragma unroll
    for (int r = 0; r < NR; ++r) acc[m][r] = 0.f;
  for (int c0 = lane * 32; c0 < K; c0 += 1024 * U) {
    uint4 w[NR][U];
    float s[NR][U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u * 1024;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        if (c < K && live[r]) {
          w[r][u] = dev::ld_stream(rows[r] + c / 2);
          s[r][u] = dev::bf2f(sc[r][c / kQG]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u * 1024;
      if (c < K) {
#pragma unroll
        for (int m = 0; m < MR; ++m) {
          if (m < M) {
            const XChunk x = load_xchunk(st + m * stage_bytes, nb, c / 32);
#pragma unroll
            for (int r = 0; r < NR; ++r)
              if (live[r]) acc[m][r] = fmaf(s[r][u], q4_dot32(w[r][u], x), acc[m][r]);
          }
        }
      }
    }
  }
}

struct Q4GemvParams {
  const uint8_t *pool;
  size_t slot_bytes;
  int H, I, n_groups, bpg, chunk;
  const uint16_t *xp;
  uint16_t *h;
  float *out;
  int32_t slot[kQ4MaxGroups], row_begin[kQ4MaxGroups], row_count[kQ4MaxGroups];
};

// two (gate, up) pairs per warp at a time (pairs i and i + nw): four rows
// share every staged activation block
template <int MR>
__global__ void __launch_bounds__(256, MR == 1 ? 3 : 2) ffn1_q4_kernel(const __grid_constant__ Q4GemvParams p) {
  extern __shared__ __align__(16) uint8_t xs1[];  // [MR][q4_stage_bytes(H)]
  const int g = blockIdx.x / p.bpg, cid = blockIdx.x % p.bpg;
  const int M = p.row_count[g], rb = p.row_begin[g], H = p.H, I = p.I;
  const int Hs = q4_stage_bytes(H);
  for (int m = 0; m < M; ++m) stage_x_q8(p.xp + static_cast<size_t>(rb + m) * H, H, xs1 + m * Hs);
  __syncthreads();
  const Q4Layout L = q4_layout(H, I);
  const uint8_t *img = p.pool + static_cast<size_t>(p.slot[g]) * p.slot_bytes;
  const uint16_t *s13 = reinterpret_cast<const uint16_t *>(img + L.s13_off);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int i_end = min(I, (cid + 1) * p.chunk);
  for (int i0 = cid * p.chunk + wid; i0 < i_end; i0 += 2 * nw) {
    const uint8_t *rows[4];
    const uint16_t *scs[4];
    bool live[4];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int i = i0 + q * nw;
      const int ii = i < i_end ? i : i0;
      const size_t grow = static_cast<size_t>((ii / kIlvQ) * 2 * kIlvQ + (ii % kIlvQ));
      rows[2 * q] = img + grow * (H / 2);
      rows[2 * q + 1] = rows[2 * q] + static_cast<size_t>(kIlvQ) * (H / 2);
      scs[2 * q] = s13 + grow * (H / kQG);
      scs[2 * q + 1] = scs[2 * q] + static_cast<size_t>(kIlvQ) * (H / kQG);
      live[2 * q] = live[2 * q + 1] = i < i_end;
    }
    float a[MR][4];
    q4_rows_dot<MR, 4, 2>(rows, scs, live, xs1, Hs, M, H, lane, a);
#pragma unroll
    for (int m = 0; m < MR; ++m) {
      if (m < M) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (!live[2 * q]) continue;
          const float gs = dev::warp_sum(a[m][2 * q]);
          const float us = dev::warp_sum(a[m][2 * q + 1]);
          if (lane == 0) p.h[static_cast<size_t>(rb + m) * I + i0 + q * nw] = dev::f2bf(dev::silu(gs) * us);
        }
      }
    }
  }
}

// NR W2 rows per warp at a time (j, j + nw, ..): NR = 4 when the layer has
// rows to spare (every staged block shared by four rows), fewer when a single
// expert's H rows would leave most warps idle (Mixtral, 1 expert: NR = 1)
template <int MR, int NR>
__global__ void __launch_bounds__(256, MR == 1 ? 3 : 2) ffn2_q4_kernel(const __grid_constant__ Q4GemvParams p) {
  extern __shared__ __align__(16) uint8_t hs2[];  // [MR][q4_stage_bytes(I)]
  const int g = blockIdx.x / p.bpg, cid = blockIdx.x % p.bpg;
  const int M = p.row_count[g], rb = p.row_begin[g], H = p.H, I = p.I;
  const int Is = q4_stage_bytes(I);
  for (int m = 0; m < M; ++m) stage_x_q8(p.h + static_cast<size_t>(rb + m) * I, I, hs2 + m * Is);
  __syncthreads();
  const Q4Layout L = q4_layout(H, I);
  const uint8_t *img = p.pool + static_cast<size_t>(p.slot[g]) * p.slot_bytes;
  const uint8_t *w2 = img + L.w2_off;
  const uint16_t *s2 = reinterpret_cast<const uint16_t *>(img + L.s2_off);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int j_end = min(H, (cid + 1) * p.chunk);
  constexpr int U = NR == 1 ? 4 : 2;
  for (int j0 = cid * p.chunk + wid; j0 < j_end; j0 += NR * nw) {
    const uint8_t *rows[NR];
    const uint16_t *scs[NR];
    bool live[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int j = j0 + q * nw;
      live[q] = j < j_end;
      const int jj = live[q] ? j : j0;
      rows[q] = w2 + static_cast<size_t>(jj) * (I / 2);
      scs[q] = s2 + static_cast<size_t>(jj) * (I / kQG);
    }
    float a[MR][NR];
    q4_rows_dot<MR, NR, U>(rows, scs, live, hs2, Is, M, I, lane, a);
#pragma unroll
    for (int m = 0; m < MR; ++m) {
      if (m < M) {
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          if (!live[q]) continue;
          const float s = dev::warp_sum(a[m][q]);
          if (lane == 0) p.out[static_cast<size_t>(rb + m) * H + j0 + q * nw] = s;
        }
      }
    }
  }
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <typename K>
void q4_smem(K kernel, int bytes) {
  if (bytes > 48 * 1024) HM_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

void launch_q4_gemv(const uint8_t *pool, size_t slot_bytes, int H, int I, const std::vector<hm_group> &gs,
                    const uint16_t *xp, uint16_t *h, float *out, cudaStream_t st) {
  if (gs.empty()) return;
  Q4GemvParams p{};
  p.pool = pool;
  p.slot_bytes = slot_bytes;
  p.H = H;
  p.I = I;
  p.n_groups = static_cast<int>(gs.size());
  p.xp = xp;
  p.h = h;
  p.out = out;
  int mr = 1;
  for (size_t g = 0; g < gs.size(); ++g) {
    p.slot[g] = gs[g].slot;
    p.row_begin[g] = gs[g].row_begin;
    p.row_count[g] = gs[g].row_count;
    mr = std::max(mr, gs[g].row_count);
  }
  const int target = sm_count() * 3, G = p.n_groups;  // 3 resident blocks per SM (80 registers)
  static const int c1 = [] { const char *e = std::getenv("HM_Q4_CHUNK1"); return e ? std::atoi(e) : 8; }();
  static const int c2 = [] { const char *e = std::getenv("HM_Q4_CHUNK2"); return e ? std::atoi(e) : 0; }();
  p.chunk = std::max(c1, static_cast<int>((static_cast<long>(G) * I + target - 1) / target + 7) / 8 * 8);
  p.bpg = (I + p.chunk - 1) / p.chunk;
  int smem = mr * q4_stage_bytes(H);
  switch (mr) {
    case 1: q4_smem(ffn1_q4_kernel<1>, smem); ffn1_q4_kernel<1><<<G * p.bpg, 256, smem, st>>>(p); break;
    case 2: q4_smem(ffn1_q4_kernel<2>, smem); ffn1_q4_kernel<2><<<G * p.bpg, 256, smem, st>>>(p); break;
    default: q4_smem(ffn1_q4_kernel<4>, smem); ffn1_q4_kernel<4><<<G * p.bpg, 256, smem, st>>>(p); break;
  }
  HM_LAUNCH_CHECK();
  // ffn2: rows per warp-iteration from the rows available per resident warp
  const long rows2 = static_cast<long>(G) * H, warps = static_cast<long>(target) * 8;
  const int nr = rows2 >= 3 * warps ? 4 : rows2 >= 3 * warps / 2 ? 2 : 1;
  p.chunk = std::max(c2 > 8 ? c2 : nr, static_cast<int>((rows2 + target - 1) / target + nr - 1) / nr * nr);
  p.bpg = (H + p.chunk - 1) / p.chunk;
  smem = mr * q4_stage_bytes(I);
#define HM_Q4_FFN2(MRV, NRV)                                            \
  q4_smem(ffn2_q4_kernel<MRV, NRV>, smem);                              \
  ffn2_q4_kernel<MRV, NRV><<<G * p.bpg, 256, smem, st>>>(p)
  const int sel = (mr == 1 ? 0 : mr == 2 ? 1 : 2) * 3 + (nr == 4 ? 0 : nr == 2 ? 1 : 2);
  switch (sel) {
    case 0: HM_Q4_FFN2(1, 4); break;
    case 1: HM_Q4_FFN2(1, 2); break;
    case 2: HM_Q4_FFN2(1, 1); break;
    case 3: HM_Q4_FFN2(2, 4); break;
    case 4: HM_Q4_FFN2(2, 2); break;
    case 5: HM_Q4_FFN2(2, 1); break;
    case 6: HM_Q4_FFN2(4, 4); break;
    case 7: HM_Q4_FFN2(4, 2); break;
    default: HM_Q4_FFN2(4, 1); break;
  }
#undef HM_Q4_FFN2
  HM_LAUNCH_CHECK();
}

}  // namespace
}  // namespace hm

extern "C" {

int hm_expert_ffn(const uint16_t *, int, int, int, const hm_group *, int, const uint16_t *, int, uint16_t *, float *,
                  int, void *);

int hm_q4_image_bytes(int H, int I, size_t *bytes) {
  HM_API_BEGIN
  HM_REQUIRE(H > 0 && I > 0 && H % 128 == 0 && I % 128 == 0, HM_EVALUE, "4-bit experts need H, I multiples of 128");
  *bytes = hm::q4_layout(H, I).bytes;
  HM_API_END
}

int hm_q4_quantize(const uint16_t *bf16_image, int H, int I, uint8_t *q4_image, void *stream) {
  HM_API_BEGIN
  HM_REQUIRE(H % 128 == 0 && I % 128 == 0, HM_EVALUE, "4-bit experts need H, I multiples of 128");
  const long n = static_cast<long>(3) * H * I / hm::kQG;
  hm::q4_quantize_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      bf16_image, H, I, q4_image);
  HM_LAUNCH_CHECK();
  HM_API_END
}

int hm_q4_dequantize(const uint8_t *q4_image, int H, int I, uint16_t *bf16_image, void *stream) {
  HM_API_BEGIN
  HM_REQUIRE(H % 128 == 0 && I % 128 == 0, HM_EVALUE, "4-bit experts need H, I multiples of 128");
  const long n = static_cast<long>(3) * H * I / hm::kQG;
  hm::q4_dequantize_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      q4_image, H, I, bf16_image);
  HM_LAUNCH_CHECK();
  HM_API_END
}

int hm_expert_ffn_q4(const uint8_t *pool, size_t slot_bytes, int n_slots, int H, int I, const hm_group *groups,
                     int n_groups, const uint16_t *xp, int total_rows, uint16_t *h, float *out, uint16_t *scratch,
                     int n_scratch, int path, void *stream) {
  HM_API_BEGIN
  HM_REQUIRE(H % 128 == 0 && I % 128 == 0, HM_EVALUE, "4-bit experts need H, I multiples of 128");
  HM_REQUIRE(slot_bytes >= hm::q4_layout(H, I).bytes, HM_EVALUE, "slot smaller than a 4-bit expert image");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::vector<hm_group> small, big;
  for (int g = 0; g < n_groups; ++g) {
    const hm_group &gr = groups[g];
    HM_REQUIRE(gr.slot >= 0 && gr.slot < n_slots && gr.row_begin >= 0 && gr.row_count >= 0 &&
                   gr.row_begin + gr.row_count <= total_rows,
               HM_EVALUE, "expert group outside the pool or the row range");
    if (gr.row_count == 0) continue;
    const bool gemv = path == HM_FFN_GEMV || (path == HM_FFN_AUTO && gr.row_count <= 4);
    HM_REQUIRE(!gemv || gr.row_count <= 4, HM_EVALUE, "GEMV path takes at most 4 rows per expert");
    (gemv ? small : big).push_back(gr);
  }
  for (size_t b = 0; b < small.size(); b += hm::kQ4MaxGroups) {
    std::vector<hm_group> part(small.begin() + b, small.begin() + std::min(small.size(), b + hm::kQ4MaxGroups));
    hm::launch_q4_gemv(pool, slot_bytes, H, I, part, xp, h, out, st);
  }
  // prefill-sized groups: dequantize into bf16 scratch slots, then the tcgen05 GEMM
  const size_t elems = static_cast<size_t>(3) * H * I;
  for (size_t b = 0; b < big.size(); b += static_cast<size_t>(std::max(1, n_scratch))) {
    HM_REQUIRE(scratch && n_scratch >= 1, HM_EVALUE, "4-bit GEMM path needs bf16 scratch slots");
    std::vector<hm_group> part;
    for (size_t i = b; i < std::min(big.size(), b + static_cast<size_t>(n_scratch)); ++i) {
      const int k = static_cast<int>(i - b);
      const int rc = hm_q4_dequantize(pool + static_cast<size_t>(big[i].slot) * slot_bytes, H, I,
                                      scratch + static_cast<size_t>(k) * elems, stream);
      if (rc != HM_OK) hm::raise(rc, hm::last_error());
      part.push_back(hm_group{k, big[i].row_begin, big[i].row_count, 0});
    }
    const int rc = hm_expert_ffn(scratch, n_scratch, H, I, part.data(), static_cast<int>(part.size()), xp,
                                 total_rows, h, out, HM_FFN_GEMM, stream);
    if (rc != HM_OK) hm::raise(rc, hm::last_error());
  }
  HM_API_END
}

}  // extern "C"
