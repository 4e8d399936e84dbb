// Expert FFN kernels for the HybriMoE layer on sm_100a:
//   E(x) = W2 ( silu(Wg x) * (Wu x) )            (Eq. 1; SwiGLU experts)
//
// Weights live in an HBM slot pool: slot s is one expert image of 3*H*I bf16
//   [0, 2IH)   W13 = gate/up rows interleaved in 128-row blocks
//              (rows 256b..256b+127 = gate rows 128b.., the next 128 = up rows)
//   [2IH, 3IH) W2  = [H, I] row-major
// so one H2D copy moves an expert and one 256-row W13 tile carries matching
// gate and up columns for a fused SwiGLU epilogue.
//
// Two paths, chosen per token group by size:
//   * decode (<= 4 rows): weight-streaming warp GEMV, 16-byte L1-bypassing
//     loads, activations staged in shared memory; HBM-bound.
//   * prefill: persistent grouped GEMM, TMA (SWIZZLE_128B) -> 4-stage smem
//     ring -> tcgen05.mma (M=128, N=256, fp32 accumulators in TMEM, double
//     buffered) -> tcgen05.ld epilogue (SwiGLU for W13, fp32 store for W2).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "device.cuh"

namespace hm {
namespace {

constexpr int kMaxGroups = 96;
constexpr int kGemvMaxRows = 4;
constexpr int kIlv = 128;  // gate/up interleave block

struct GemvParams {
  const uint16_t *pool;
  size_t slot_elems;
  int H, I;
  int n_groups;
  int bpg;    // blocks per group
  int chunk;  // pairs (ffn1) or rows (ffn2) per block
  int l2_prefetch;  // ffn2: warm L2 with the block's W2 rows before waiting on ffn1
  const uint16_t *xp;
  uint16_t *h;
  float *out;
  int32_t slot[kMaxGroups];
  int32_t row_begin[kMaxGroups];
  int32_t row_count[kMaxGroups];
};

// h[r, i] = silu(gate_i . x_r) * (up_i . x_r) for the rows of one group.
// The warp's first weight batch is issued before the activations are staged:
// at decode sizes a warp owns only a few rows, so the kernel is a short chain
// of DRAM round trips and the staging round trip is taken off it.
template <int MR>
__global__ void __launch_bounds__(256) ffn1_gemv_kernel(const __grid_constant__ GemvParams p) {
  extern __shared__ __align__(16) uint16_t xs[];  // [MR][H]
  // let ffn2 (launched with programmatic stream serialization) get scheduled
  // onto SMs as this grid's blocks retire: its prologue overlaps our tail
  asm volatile("griddepcontrol.launch_dependents;");
  const int g = blockIdx.x / p.bpg, cid = blockIdx.x % p.bpg;
  const int M = p.row_count[g], rb = p.row_begin[g], H = p.H, I = p.I;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint16_t *w13 = p.pool + static_cast<size_t>(p.slot[g]) * p.slot_elems;
  const int i_end = min(I, (cid + 1) * p.chunk);
  constexpr int U = 4;
  auto rows_of = [&](int i, const uint16_t *&wg, const uint16_t *&wu) {
    const size_t grow = static_cast<size_t>((i / kIlv) * 2 * kIlv + (i % kIlv));
    wg = w13 + grow * H;
    wu = wg + static_cast<size_t>(kIlv) * H;
  };
  // first batch of this warp's first pair, in flight during the staging
  uint4 gv[U], uv[U];
  const int i0 = cid * p.chunk + wid;
  if (i0 < i_end) {
    const uint16_t *wg, *wu;
    rows_of(i0, wg, wu);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = lane * 8 + u * 256;
      if (c < H) {
        gv[u] = dev::ld_stream(wg + c);
        uv[u] = dev::ld_stream(wu + c);
      }
    }
  }
  for (int v = threadIdx.x; v < M * H / 8; v += blockDim.x)
    reinterpret_cast<uint4 *>(xs)[v] = reinterpret_cast<const uint4 *>(p.xp + static_cast<size_t>(rb) * H)[v];
  __syncthreads();
  for (int i = i0; i < i_end; i += nw) {
    const uint16_t *wg, *wu;
    rows_of(i, wg, wu);
    float ag[MR], au[MR];
#pragma unroll
    for (int m = 0; m < MR; ++m) ag[m] = au[m] = 0.f;
    for (int c0 = lane * 8; c0 < H; c0 += 256 * U) {
      if (i != i0 || c0 != lane * 8) {  // (the first batch is already in gv / uv)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int c = c0 + u * 256;
          if (c < H) {
            gv[u] = dev::ld_stream(wg + c);
            uv[u] = dev::ld_stream(wu + c);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + u * 256;
        if (c < H) {
#pragma unroll
          for (int m = 0; m < MR; ++m) {
            if (m < M) {
              const uint4 xv = *reinterpret_cast<const uint4 *>(xs + m * H + c);
              ag[m] += dev::dot8(gv[u], xv);
              au[m] += dev::dot8(uv[u], xv);
            }
          }
        }
      }
    }
#pragma unroll
    for (int m = 0; m < MR; ++m) {
      if (m < M) {
        const float gs = dev::warp_sum(ag[m]), us = dev::warp_sum(au[m]);
        if (lane == 0) p.h[static_cast<size_t>(rb + m) * I + i] = dev::f2bf(dev::silu(gs) * us);
      }
    }
  }
}

// out[r, j] = W2[j, :] . h[r, :].  The warp's first weight batch is loaded
// BEFORE waiting for ffn1 (programmatic dependent launch): W2 does not depend
// on h, so at decode sizes most of a warp's bytes are in flight while ffn1
// finishes, and the wait + h staging overlap them.
template <int MR>
__global__ void __launch_bounds__(256) ffn2_gemv_kernel(const __grid_constant__ GemvParams p) {
  extern __shared__ __align__(16) uint16_t hs[];  // [MR][I]
  const int g = blockIdx.x / p.bpg, cid = blockIdx.x % p.bpg;
  const int M = p.row_count[g], rb = p.row_begin[g], H = p.H, I = p.I;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint16_t *w2 = p.pool + static_cast<size_t>(p.slot[g]) * p.slot_elems + static_cast<size_t>(2) * I * H;
  const int j_end = min(H, (cid + 1) * p.chunk);
  // two rows per warp at a time (rows j and j + nw): twice the loads in flight
  // per warp -- small-I experts (DeepSeek: 2.8 KB rows) were latency-bound
  constexpr int RW = 2, U = 4;
  const int jf = cid * p.chunk + wid;
  uint4 wv[RW][U];
  if (jf < j_end) {
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      const bool live = jf + r * nw < j_end;
      const uint16_t *wr = w2 + static_cast<size_t>(live ? jf + r * nw : jf) * I;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = lane * 8 + u * 256;
        if (c < I && live) wv[r][u] = dev::ld_stream(wr + c);
      }
    }
  }
  if (p.l2_prefetch) {  // the rest of this block's W2 rows into L2 (independent of ffn1)
    const int j0 = cid * p.chunk, j1 = min(H, (cid + 1) * p.chunk);
    const char *base = reinterpret_cast<const char *>(w2 + static_cast<size_t>(j0) * I);
    const size_t bytes = j1 > j0 ? static_cast<size_t>(j1 - j0) * I * 2 : 0;
    for (size_t o = static_cast<size_t>(threadIdx.x) * 128; o < bytes; o += static_cast<size_t>(blockDim.x) * 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(base + o));
  }
  // h comes from ffn1: wait for the primary grid (no-op without PDL)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int v = threadIdx.x; v < M * I / 8; v += blockDim.x)
    reinterpret_cast<uint4 *>(hs)[v] = reinterpret_cast<const uint4 *>(p.h + static_cast<size_t>(rb) * I)[v];
  __syncthreads();
  for (int j0 = jf; j0 < j_end; j0 += nw * RW) {
    const uint16_t *wr[RW];
    bool live[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      live[r] = j0 + r * nw < j_end;
      wr[r] = w2 + static_cast<size_t>(live[r] ? j0 + r * nw : j0) * I;
    }
    float acc[MR][RW];
#pragma unroll
    for (int m = 0; m < MR; ++m)
#pragma unroll
      for (int r = 0; r < RW; ++r) acc[m][r] = 0.f;
    for (int c0 = lane * 8; c0 < I; c0 += 256 * U) {
      if (j0 != jf || c0 != lane * 8) {  // (the first batch is already in wv)
#pragma unroll
        for (int r = 0; r < RW; ++r)
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int c = c0 + u * 256;
            if (c < I && live[r]) wv[r][u] = dev::ld_stream(wr[r] + c);
          }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + u * 256;
        if (c < I) {
#pragma unroll
          for (int m = 0; m < MR; ++m)
            if (m < M) {
              const uint4 hv = *reinterpret_cast<const uint4 *>(hs + m * I + c);
#pragma unroll
              for (int r = 0; r < RW; ++r)
                if (live[r]) acc[m][r] += dev::dot8(wv[r][u], hv);
            }
        }
      }
    }
#pragma unroll
    for (int m = 0; m < MR; ++m) {
      if (m < M) {
#pragma unroll
        for (int r = 0; r < RW; ++r) {
          if (!live[r]) continue;
          const float s = dev::warp_sum(acc[m][r]);
          if (lane == 0) p.out[static_cast<size_t>(rb + m) * H + j0 + r * nw] = s;
        }
      }
    }
  }
}

// ------------------------------------------------------------ fused decode GEMV
// ONE persistent launch per layer for ffn1 -> ffn2 (instead of two short
// launches that each pay a ramp and a tail; DeepSeek's 4-6 small experts ran
// at 3.7 TB/s that way).  Work items, statically strided over the warps of a
// cooperative (co-resident) grid -- warp w takes items w, w + W, w + 2W, ...:
//   phase 1 item (g, i):   gate row i and up row i of group g's W13 (2 rows of
//                          H), h[r, i] = bf16(silu(gate.x_r) * (up.x_r)); a
//                          warp publishes its count of finished items of g
//                          with one release-add on sub-counter done[g][w % 32]
//   phase 2 item (g, j..): NR2 rows of W2 (I columns), out[r, j] = W2[j].h_r;
//                          the item's first weight loads are issued BEFORE the
//                          warp waits (lane k acquires sub-counter k, the warp
//                          sums them) for group g's I phase-1 items, so the
//                          phase boundary overlaps with DRAM streaming.
// All phase-1 items precede all phase-2 items in the item order, and the grid
// is co-resident (cooperative launch), so every wait is on a running warp.
// The 32 sub-counters per group sit on separate 128-byte lines (a single
// counter serialised the adds of thousands of warps); they are never reset:
// they only grow, and the host passes each group's running total at launch
// (bases, tracked per stream) so the target is base + I.  Per
// lane, columns are accumulated in the same order as ffn1/ffn2_gemv_kernel
// (c = lane*8 + 256k, k increasing): outputs bit-identical to the pair.
constexpr int kDoneStride = 32;  // ints: one 128-byte line per counter

struct FusedGemvParams {
  const uint16_t *pool;
  size_t slot_elems;
  int H, I, n_groups;
  int n1, n2, items2_per_group, total_warps;
  const uint16_t *xp;
  uint16_t *h;
  float *out;
  uint32_t *done;  // [kMaxGroups][32 counters][kDoneStride]
  uint32_t base[kMaxGroups];
  int32_t slot[kMaxGroups];
  int32_t row_begin[kMaxGroups];
  int32_t row_count[kMaxGroups];
};

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu(uint32_t *p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int MR, int U>
__device__ __forceinline__ void fused_phase1(const FusedGemvParams &p, int it, int lane) {
  const int H = p.H, I = p.I;
  const int g = it / I, i = it - g * I;
  const int M = p.row_count[g], rb = p.row_begin[g];
  const uint16_t *w13 = p.pool + static_cast<size_t>(p.slot[g]) * p.slot_elems;
  const size_t grow = static_cast<size_t>((i / kIlv) * 2 * kIlv + (i % kIlv));
  const uint16_t *wg = w13 + grow * H;
  const uint16_t *wu = wg + static_cast<size_t>(kIlv) * H;
  const uint16_t *x = p.xp + static_cast<size_t>(rb) * H;
  float ag[MR], au[MR];
#pragma unroll
  for (int m = 0; m < MR; ++m) ag[m] = au[m] = 0.f;
  for (int c0 = lane * 8; c0 < H; c0 += 256 * U) {
    uint4 gv[U], uv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u * 256;
      if (c < H) {
        gv[u] = dev::ld_stream(wg + c);
        uv[u] = dev::ld_stream(wu + c);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u * 256;
      if (c < H) {
#pragma unroll
        for (int m = 0; m < MR; ++m) {
          if (m < M) {
            const uint4 xv = __ldg(reinterpret_cast<const uint4 *>(x + static_cast<size_t>(m) * H + c));
            ag[m] += dev::dot8(gv[u], xv);
            au[m] += dev::dot8(uv[u], xv);
          }
        }
      }
    }
  }
#pragma unroll
  for (int m = 0; m < MR; ++m) {
    if (m < M) {
      const float gs = dev::warp_sum(ag[m]), us = dev::warp_sum(au[m]);
      if (lane == 0) p.h[static_cast<size_t>(rb + m) * I + i] = dev::f2bf(dev::silu(gs) * us);
    }
  }
}

template <int MR, int NR2, int U2>
__device__ __forceinline__ void fused_phase2(const FusedGemvParams &p, int it2, int lane) {
  const int H = p.H, I = p.I;
  const int g = it2 / p.items2_per_group, j0 = (it2 - g * p.items2_per_group) * NR2;
  const int M = p.row_count[g], rb = p.row_begin[g];
  const uint16_t *w2 = p.pool + static_cast<size_t>(p.slot[g]) * p.slot_elems + static_cast<size_t>(2) * I * H;
  bool live[NR2];
  const uint16_t *wr[NR2];
#pragma unroll
  for (int r = 0; r < NR2; ++r) {
    live[r] = j0 + r < H;
    wr[r] = w2 + static_cast<size_t>(live[r] ? j0 + r : j0) * I;
  }
  float acc[MR][NR2];
#pragma unroll
  for (int m = 0; m < MR; ++m)
#pragma unroll
    for (int r = 0; r < NR2; ++r) acc[m][r] = 0.f;
  const uint16_t *hrow = p.h + static_cast<size_t>(rb) * I;
  bool ready = false;
  for (int c0 = lane * 8; c0 < I; c0 += 256 * U2) {
    uint4 wv[NR2][U2];
#pragma unroll
    for (int r = 0; r < NR2; ++r)
#pragma unroll
      for (int u = 0; u < U2; ++u) {
        const int c = c0 + u * 256;
        if (c < I && live[r]) wv[r][u] = dev::ld_stream(wr[r] + c);
      }
    if (!ready) {  // h of group g complete?  (the loads above are already in flight)
      const uint32_t *d = p.done + (static_cast<size_t>(g) * 32 + lane) * kDoneStride;
      const uint32_t target = p.base[g] + static_cast<uint32_t>(I);
      for (;;) {  // every lane acquires its own sub-counter; the warp sums them
        uint32_t v = ld_acquire_gpu(d);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (static_cast<int32_t>(v - target) >= 0) break;
        __nanosleep(32);
      }
      __syncwarp();
      ready = true;
    }
#pragma unroll
    for (int u = 0; u < U2; ++u) {
      const int c = c0 + u * 256;
      if (c < I) {
#pragma unroll
        for (int m = 0; m < MR; ++m)
          if (m < M) {
            const uint4 hv = __ldcg(reinterpret_cast<const uint4 *>(hrow + static_cast<size_t>(m) * I + c));
#pragma unroll
            for (int r = 0; r < NR2; ++r)
              if (live[r]) acc[m][r] += dev::dot8(wv[r][u], hv);
          }
      }
    }
  }
#pragma unroll
  for (int m = 0; m < MR; ++m) {
    if (m < M) {
#pragma unroll
      for (int r = 0; r < NR2; ++r) {
        if (!live[r]) continue;
        const float s = dev::warp_sum(acc[m][r]);
        if (lane == 0) p.out[static_cast<size_t>(rb + m) * H + j0 + r] = s;
      }
    }
  }
}

// MINB resident CTAs per SM.  Phase-1 items go to the first total_warps warps
// in warp-major order (spread over the SMs), a count chosen so that each does
// the same number of items (a plain stride left a last round running a few
// percent of the warps while all phase-2 warps waited); phase-2 items are
// strided over all warps of the grid.
template <int MR, int NR2, int MINB>
__global__ void __launch_bounds__(256, MINB) ffn_decode_fused_kernel(const __grid_constant__ FusedGemvParams p) {
  constexpr int U1 = 4;
  constexpr int U2 = (MINB >= 4 ? 4 : 8) / NR2;
  const int lane = threadIdx.x & 31;
  const int w0 = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  const int all = gridDim.x * (blockDim.x >> 5);
  // phase 1; completions are published once per group this warp worked on
  // (one release-add on the warp's own sub-counter), not per item: a release
  // per item stalled the warp's next loads
  int cur_g = -1;
  uint32_t n_done = 0;
  for (int it = w0; w0 < p.total_warps && it < p.n1; it += p.total_warps) {
    const int g = it / p.I;
    if (g != cur_g) {
      if (cur_g >= 0 && lane == 0)
        red_release_gpu(p.done + (static_cast<size_t>(cur_g) * 32 + (w0 & 31)) * kDoneStride, n_done);
      cur_g = g;
      n_done = 0;
    }
    fused_phase1<MR, U1>(p, it, lane);
    ++n_done;
  }
  if (cur_g >= 0 && lane == 0)
    red_release_gpu(p.done + (static_cast<size_t>(cur_g) * 32 + (w0 & 31)) * kDoneStride, n_done);
  for (int it2 = w0; it2 < p.n2; it2 += all) fused_phase2<MR, NR2, U2>(p, it2, lane);
}

// ------------------------------------------------------------ tcgen05 GEMM
constexpr int BM = 128, BK = 64, STAGES = 4;

struct GemmParams {
  int n_groups, n_tiles, K, n_blocks, ldo;
  uint16_t *h;
  float *out;
  int32_t tile_start[kMaxGroups + 1];
  int32_t row_begin[kMaxGroups];
  int32_t row_count[kMaxGroups];
  int32_t b_row_base[kMaxGroups];
};

template <int BN>
constexpr int gemm_smem_bytes() {
  return STAGES * (BM + BN) * BK * 2 + 1024 /*align*/ + 256 /*barriers*/;
}

// MODE 0: A = xp [rows, H], B = W13 view, epilogue SwiGLU -> h (bf16, ldo = I)
// MODE 1: A = h  [rows, I], B = W2 view,  epilogue fp32 -> out (ldo = H)
template <int BN, int MODE>
__global__ void __launch_bounds__(256, 1)
    expert_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const __grid_constant__ GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = dev::smem_u32(smem_raw);
  uint8_t *smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t *sA = smem;                                    // STAGES x BM x BK bf16
  uint8_t *sB = smem + STAGES * BM * BK * 2;             // STAGES x BN x BK bf16
  uint64_t *bars = reinterpret_cast<uint64_t *>(sB + STAGES * BN * BK * 2);
  uint64_t *full = bars, *empty = bars + STAGES, *tfull = bars + 2 * STAGES, *tempty = bars + 2 * STAGES + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * STAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&tmA);
    dev::tma_prefetch_desc(&tmB);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      dev::mbar_init(&tfull[a], 1);
      dev::mbar_init(&tempty[a], 4);
    }
    dev::fence_barrier_init();
  }
  if (warp == 2) dev::tmem_alloc<512>(tmem_slot);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto decode = [&](int t, int &g, int &mb, int &nb) {
    g = 0;
    while (g + 1 < p.n_groups && p.tile_start[g + 1] <= t) ++g;
    const int local = t - p.tile_start[g];
    const int mblocks = (p.row_count[g] + BM - 1) / BM;
    nb = local / mblocks;
    mb = local % mblocks;
  };
  const int nkb = p.K / BK;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
        int g, mb, nb;
        decode(t, g, mb, nb);
        const int a_row = p.row_begin[g] + mb * BM;
        const int b_row = p.b_row_base[g] + nb * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          dev::mbar_wait(&empty[stage], phase ^ 1u);
          dev::mbar_arrive_expect_tx(&full[stage], (BM + BN) * BK * 2);
          dev::tma_load_2d(sA + stage * BM * BK * 2, &tmA, &full[stage], kb * BK, a_row);
          dev::tma_load_2d(sB + stage * BN * BK * 2, &tmB, &full[stage], kb * BK, b_row);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer (single thread)
      constexpr uint32_t idesc = dev::umma_idesc_bf16(BM, BN);
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
        dev::mbar_wait(&tempty[acc], aphase ^ 1u);
        dev::tc_fence_after();
        const uint32_t d = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = 0; kb < nkb; ++kb) {
          dev::mbar_wait(&full[stage], phase);
          dev::tc_fence_after();
          const uint32_t a0 = dev::smem_u32(sA + stage * BM * BK * 2);
          const uint32_t b0 = dev::smem_u32(sB + stage * BN * BK * 2);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            dev::umma_bf16(d, dev::umma_desc_sw128(a0 + k * 32), dev::umma_desc_sw128(b0 + k * 32), idesc,
                           (kb | k) != 0 ? 1u : 0u);
          dev::umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        dev::umma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) aphase ^= 1u;
      }
    }
    __syncwarp();
  } else if (warp >= 4) {  // ---------------- epilogue: TMEM -> registers -> global
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    int acc = 0;
    uint32_t aphase = 0;
    for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
      int g, mb, nb;
      decode(t, g, mb, nb);
      dev::mbar_wait(&tfull[acc], aphase);
      dev::tc_fence_after();
      const int lrow = mb * BM + q * 32 + lane;
      const bool live = lrow < p.row_count[g];
      const size_t row = static_cast<size_t>(p.row_begin[g] + lrow);
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * BN);
      if constexpr (MODE == 0) {
#pragma unroll 1
        for (int c = 0; c < BN / 2; c += 32) {
          uint32_t gr[32], ur[32];
          dev::tmem_ld_32x32b_x32(tbase + c, gr);
          dev::tmem_ld_32x32b_x32(tbase + BN / 2 + c, ur);
          dev::tmem_ld_wait();
          if (live) {
            uint4 *dst = reinterpret_cast<uint4 *>(p.h + row * p.ldo + nb * (BN / 2) + c);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              uint32_t w[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int j = v * 8 + e * 2;
                const float h0 = dev::silu(__uint_as_float(gr[j])) * __uint_as_float(ur[j]);
                const float h1 = dev::silu(__uint_as_float(gr[j + 1])) * __uint_as_float(ur[j + 1]);
                w[e] = dev::pack_bf2(h0, h1);
              }
              dst[v] = make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t r[32];
          dev::tmem_ld_32x32b_x32(tbase + c, r);
          dev::tmem_ld_wait();
          if (live) {
            float4 *dst = reinterpret_cast<float4 *>(p.out + row * p.ldo + nb * BN + c);
#pragma unroll
            for (int v = 0; v < 8; ++v)
              dst[v] = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                   __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
          }
        }
      }
      dev::tc_fence_before();
      __syncwarp();
      if (lane == 0) dev::mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) aphase ^= 1u;
    }
  }
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  if (warp == 2) dev::tmem_dealloc<512>(tmem_base);
}

// ------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void *f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  if (!fn) raise(HM_ECUDA, "cuTensorMapEncodeTiled is unavailable");
  return fn;
}

// 2D bf16 tensor [outer, inner] with a (64 x box_rows) box and 128-byte swizzle.
// Encoded maps are cached by (base, inner, outer, box): the pool and the
// activation buffers are fixed, so steady state does no host-side encoding.
CUtensorMap make_map_uncached(const void *base, uint64_t inner, uint64_t outer, uint32_t box_rows);
CUtensorMap make_map(const void *base, uint64_t inner, uint64_t outer, uint32_t box_rows) {
  struct Key {
    const void *b;
    uint64_t i, o;
    uint32_t r;
  };
  static std::mutex mu;
  static std::vector<std::pair<Key, CUtensorMap>> cache;
  std::lock_guard<std::mutex> g(mu);
  for (auto &kv : cache)
    if (kv.first.b == base && kv.first.i == inner && kv.first.o == outer && kv.first.r == box_rows) return kv.second;
  CUtensorMap m = make_map_uncached(base, inner, outer, box_rows);
  if (cache.size() >= 64) cache.erase(cache.begin());
  cache.push_back({Key{base, inner, outer, box_rows}, m});
  return m;
}

CUtensorMap make_map_uncached(const void *base, uint64_t inner, uint64_t outer, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) raise(HM_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  return m;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Raise a kernel's dynamic shared-memory limit only when a launch needs more
// than it was last set to (the attribute call is not free on the host).
template <typename K>
void set_smem(K kernel, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void *, int>> done;
  std::lock_guard<std::mutex> g(mu);
  const void *key = reinterpret_cast<const void *>(kernel);
  for (auto &kv : done)
    if (kv.first == key && kv.second >= bytes) return;
  HM_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  for (auto &kv : done)
    if (kv.first == key) {
      kv.second = bytes;
      return;
    }
  done.emplace_back(key, bytes);
}

// Programmatic dependent launch (HM_PDL=0 disables): the kernel may start
// while the previous kernel on the stream finishes; it calls
// griddepcontrol.wait before touching that kernel's output.
bool pdl_enabled() {
  static const bool on = [] {
    const char *e = std::getenv("HM_PDL");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

template <typename K>
void launch_pdl(K kernel, int grid, int smem, cudaStream_t st, const GemvParams &p) {
  set_smem(kernel, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  HM_CUDA(cudaLaunchKernelEx(&cfg, kernel, p));
  HM_LAUNCH_CHECK();
}

// HM_GEMV_FUSED=1 selects the persistent one-launch kernel; the default is
// the two-launch ffn1/ffn2 pair, which measured faster at every decode shape
// (tools/gemv_lib_bench.py).
bool gemv_fused_enabled() {
  static const bool on = [] {
    const char *e = std::getenv("HM_GEMV_FUSED");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

// Completion counters of the fused GEMV, one set per stream, with the host's
// running count of the increments every counter received (the kernel never
// resets them; each launch waits for base + I/32 per counter of its groups).
struct FusedCounters {
  cudaStream_t st;
  uint32_t *dev;
  uint32_t base[kMaxGroups];
};
FusedCounters &fused_counters(cudaStream_t st) {
  static std::mutex mu;
  static std::vector<FusedCounters *> sets;
  std::lock_guard<std::mutex> g(mu);
  for (auto *c : sets)
    if (c->st == st) return *c;
  auto *c = new FusedCounters{st, nullptr, {}};
  const size_t bytes = static_cast<size_t>(kMaxGroups) * 32 * kDoneStride * sizeof(uint32_t);
  HM_CUDA(cudaMalloc(&c->dev, bytes));
  HM_CUDA(cudaMemset(c->dev, 0, bytes));
  HM_CUDA(cudaDeviceSynchronize());
  sets.push_back(c);
  return *c;
}

template <int MR, int NR2, int MINB>
void launch_fused_one(FusedGemvParams &p, cudaStream_t st) {
  static int per_sm = 0;
  if (!per_sm) {
    HM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ffn_decode_fused_kernel<MR, NR2, MINB>, 256, 0));
    per_sm = std::max(1, std::min(per_sm, 4));
  }
  // the whole co-resident grid; phase 1 in whole rounds over total_warps of it
  const int grid = num_sms() * per_sm;
  const long wmax = static_cast<long>(grid) * 8;
  const long rounds = (static_cast<long>(p.n1) + wmax - 1) / wmax;
  p.total_warps = static_cast<int>((p.n1 + rounds - 1) / rounds);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // co-residency: phase-2 warps wait on phase-1 warps
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  HM_CUDA(cudaLaunchKernelEx(&cfg, ffn_decode_fused_kernel<MR, NR2, MINB>, p));
  HM_LAUNCH_CHECK();
}

void launch_gemv_fused(const uint16_t *pool, size_t slot_elems, int H, int I, const std::vector<hm_group> &gs,
                       const uint16_t *xp, uint16_t *h, float *out, cudaStream_t st) {
  FusedGemvParams p{};
  p.pool = pool;
  p.slot_elems = slot_elems;
  p.H = H;
  p.I = I;
  p.n_groups = static_cast<int>(gs.size());
  p.xp = xp;
  p.h = h;
  p.out = out;
  FusedCounters &fc = fused_counters(st);
  p.done = fc.dev;
  int mr = 1;
  for (size_t g = 0; g < gs.size(); ++g) {
    p.slot[g] = gs[g].slot;
    p.row_begin[g] = gs[g].row_begin;
    p.row_count[g] = gs[g].row_count;
    p.base[g] = fc.base[g];
    fc.base[g] += static_cast<uint32_t>(I);  // what this launch adds to group g's 32 sub-counters together
    mr = std::max(mr, gs[g].row_count);
  }
  // long W2 rows (Mixtral, I = 14336): one row per item, 8 loads in flight per
  // lane; short rows (DeepSeek 1408, Qwen2 2560): two rows per item
  const bool one = I >= 4096;
  const int nr2 = one ? 1 : 2;
  p.n1 = p.n_groups * I;
  p.items2_per_group = (H + nr2 - 1) / nr2;
  p.n2 = p.n_groups * p.items2_per_group;
  static const int minb = [] {  // HM_GEMV_MINB=3|4 (A/B); default 4
    const char *e = std::getenv("HM_GEMV_MINB");
    return e && std::atoi(e) == 3 ? 3 : 4;
  }();
  switch (mr * 2 + (one ? 1 : 0)) {
    case 2: minb == 4 ? launch_fused_one<1, 2, 4>(p, st) : launch_fused_one<1, 2, 3>(p, st); break;
    case 3: minb == 4 ? launch_fused_one<1, 1, 4>(p, st) : launch_fused_one<1, 1, 3>(p, st); break;
    case 4: launch_fused_one<2, 2, 2>(p, st); break;
    case 5: launch_fused_one<2, 1, 2>(p, st); break;
    default:
      if (one)
        launch_fused_one<4, 1, 2>(p, st);
      else
        launch_fused_one<4, 2, 2>(p, st);
  }
}

// path HM_FFN_GEMV: HM_GEMV_FUSED decides; HM_FFN_GEMV_SPLIT / _FUSED force one
void launch_gemv(const uint16_t *pool, size_t slot_elems, int H, int I, const std::vector<hm_group> &gs,
                 const uint16_t *xp, uint16_t *h, float *out, cudaStream_t st, int path) {
  if (gs.empty()) return;
  if (path == HM_FFN_GEMV_FUSED || (path != HM_FFN_GEMV_SPLIT && gemv_fused_enabled())) {
    HM_REQUIRE(static_cast<int>(gs.size()) <= kMaxGroups, HM_EVALUE, "too many expert groups in one launch");
    HM_REQUIRE(H % 8 == 0 && I % 8 == 0 && I % kIlv == 0, HM_EVALUE, "GEMV needs H % 8 == 0 and I % 128 == 0");
    launch_gemv_fused(pool, slot_elems, H, I, gs, xp, h, out, st);
    return;
  }
  HM_REQUIRE(static_cast<int>(gs.size()) <= kMaxGroups, HM_EVALUE, "too many expert groups in one launch");
  HM_REQUIRE(H % 8 == 0 && I % 8 == 0 && I % kIlv == 0, HM_EVALUE, "GEMV needs H % 8 == 0 and I % 128 == 0");
  GemvParams p{};
  p.pool = pool;
  p.slot_elems = slot_elems;
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
  const int target = num_sms() * 4;
  const int G = p.n_groups;
  // ffn1: pairs of (gate, up) rows
  int chunk = static_cast<int>((static_cast<long>(G) * I + target - 1) / target);
  chunk = std::max(8, (chunk + 7) / 8 * 8);
  p.chunk = chunk;
  p.bpg = (I + chunk - 1) / chunk;
  int smem = mr * H * 2;
  HM_REQUIRE(smem <= 200 * 1024, HM_EVALUE, "decode rows do not fit shared memory");
  switch (mr) {
    case 1: set_smem(ffn1_gemv_kernel<1>, smem); ffn1_gemv_kernel<1><<<G * p.bpg, 256, smem, st>>>(p); break;
    case 2: set_smem(ffn1_gemv_kernel<2>, smem); ffn1_gemv_kernel<2><<<G * p.bpg, 256, smem, st>>>(p); break;
    default: set_smem(ffn1_gemv_kernel<4>, smem); ffn1_gemv_kernel<4><<<G * p.bpg, 256, smem, st>>>(p); break;
  }
  HM_LAUNCH_CHECK();
  chunk = static_cast<int>((static_cast<long>(G) * H + target - 1) / target);
  chunk = std::max(8, (chunk + 7) / 8 * 8);
  p.chunk = chunk;
  p.bpg = (H + chunk - 1) / chunk;
  smem = mr * I * 2;
  HM_REQUIRE(smem <= 200 * 1024, HM_EVALUE, "decode rows do not fit shared memory");
  // warm L2 only while the layer's W2 bytes fit comfortably in the 126 MB L2
  p.l2_prefetch = static_cast<long>(G) * H * I * 2 <= (64L << 20) ? 1 : 0;
  switch (mr) {
    case 1: launch_pdl(ffn2_gemv_kernel<1>, G * p.bpg, smem, st, p); break;
    case 2: launch_pdl(ffn2_gemv_kernel<2>, G * p.bpg, smem, st, p); break;
    default: launch_pdl(ffn2_gemv_kernel<4>, G * p.bpg, smem, st, p); break;
  }
}

template <int BN, int MODE>
void launch_gemm_one(const CUtensorMap &ta, const CUtensorMap &tb, GemmParams &p, cudaStream_t st) {
  if (p.n_tiles == 0) return;
  constexpr int smem = gemm_smem_bytes<BN>();
  set_smem(expert_gemm_kernel<BN, MODE>, smem);
  const int grid = std::min(p.n_tiles, num_sms());
  expert_gemm_kernel<BN, MODE><<<grid, 256, smem, st>>>(ta, tb, p);
  HM_LAUNCH_CHECK();
}

void launch_gemm(const uint16_t *pool, int n_slots, int H, int I, const std::vector<hm_group> &gs,
                 const uint16_t *xp, int total_rows, uint16_t *h, float *out, cudaStream_t st) {
  if (gs.empty()) return;
  HM_REQUIRE(static_cast<int>(gs.size()) <= kMaxGroups, HM_EVALUE, "too many expert groups in one launch");
  HM_REQUIRE(H % 128 == 0 && I % 128 == 0, HM_EVALUE, "GEMM path needs H % 128 == 0 and I % 128 == 0");
  const uint64_t rows = static_cast<uint64_t>(std::max(total_rows, 1));
  // ffn1: [rows, H] x W13^T -> h[rows, I]   (B view: pool as [n_slots*3I, H])
  {
    CUtensorMap ta = make_map(xp, H, rows, BM);
    CUtensorMap tb = make_map(pool, H, static_cast<uint64_t>(n_slots) * 3 * I, 256);
    GemmParams p{};
    p.n_groups = static_cast<int>(gs.size());
    p.K = H;
    p.n_blocks = 2 * I / 256;
    p.ldo = I;
    p.h = h;
    int t = 0;
    for (size_t g = 0; g < gs.size(); ++g) {
      p.tile_start[g] = t;
      p.row_begin[g] = gs[g].row_begin;
      p.row_count[g] = gs[g].row_count;
      p.b_row_base[g] = gs[g].slot * 3 * I;
      t += ((gs[g].row_count + BM - 1) / BM) * p.n_blocks;
    }
    p.tile_start[gs.size()] = t;
    p.n_tiles = t;
    launch_gemm_one<256, 0>(ta, tb, p, st);
  }
  // ffn2: h[rows, I] x W2^T -> out[rows, H]   (B view: pool as [n_slots*3H, I])
  {
    CUtensorMap ta = make_map(h, I, rows, BM);
    const bool wide = H % 256 == 0;
    CUtensorMap tb = make_map(pool, I, static_cast<uint64_t>(n_slots) * 3 * H, wide ? 256 : 128);
    GemmParams p{};
    p.n_groups = static_cast<int>(gs.size());
    p.K = I;
    p.n_blocks = H / (wide ? 256 : 128);
    p.ldo = H;
    p.out = out;
    int t = 0;
    for (size_t g = 0; g < gs.size(); ++g) {
      p.tile_start[g] = t;
      p.row_begin[g] = gs[g].row_begin;
      p.row_count[g] = gs[g].row_count;
      p.b_row_base[g] = gs[g].slot * 3 * H + 2 * H;
      t += ((gs[g].row_count + BM - 1) / BM) * p.n_blocks;
    }
    p.tile_start[gs.size()] = t;
    p.n_tiles = t;
    if (wide)
      launch_gemm_one<256, 1>(ta, tb, p, st);
    else
      launch_gemm_one<128, 1>(ta, tb, p, st);
  }
}

}  // namespace
}  // namespace hm

extern "C" {

// Back-to-back launches from the host library (no Python between launches):
// `reps` calls of hm_expert_ffn, group r of call i on slot (i*n + r) % n_slots,
// timed with events on `stream`.  Kernel micro-benchmark for the roofline.
int hm_bench_expert_ffn(const uint16_t *pool, int n_slots, int H, int I, int n_groups, int rows_per_group,
                        const uint16_t *xp, uint16_t *h, float *out, int path, int reps, void *stream, float *ms) {
  HM_API_BEGIN
  HM_REQUIRE(n_groups >= 1 && n_groups <= n_slots && rows_per_group >= 1 && reps >= 1, HM_EVALUE, "bad bench");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::vector<hm_group> g(n_groups);
  auto one = [&](int i) {
    for (int r = 0; r < n_groups; ++r)
      g[r] = hm_group{static_cast<int32_t>((static_cast<long>(i) * n_groups + r) % n_slots), r * rows_per_group,
                      rows_per_group, 0};
    const int rc = hm_expert_ffn(pool, n_slots, H, I, g.data(), n_groups, xp, n_groups * rows_per_group, h, out,
                                 path, stream);
    if (rc != HM_OK) hm::raise(rc, hm::last_error());
  };
  for (int i = 0; i < 3; ++i) one(i);
  cudaEvent_t a, b;
  HM_CUDA(cudaEventCreate(&a));
  HM_CUDA(cudaEventCreate(&b));
  HM_CUDA(cudaEventRecord(a, st));
  for (int i = 0; i < reps; ++i) one(3 + i);
  HM_CUDA(cudaEventRecord(b, st));
  HM_CUDA(cudaEventSynchronize(b));
  HM_CUDA(cudaEventElapsedTime(ms, a, b));
  *ms /= static_cast<float>(reps);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  HM_API_END
}

int hm_expert_ffn(const uint16_t *pool, int n_slots, int H, int I, const hm_group *groups, int n_groups,
                  const uint16_t *xp, int total_rows, uint16_t *h, float *out, int path, void *stream) {
  HM_API_BEGIN
  HM_REQUIRE(n_groups >= 0 && (n_groups == 0 || groups), HM_EVALUE, "bad group table");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::vector<hm_group> small, big;
  for (int g = 0; g < n_groups; ++g) {
    const hm_group &gr = groups[g];
    HM_REQUIRE(gr.slot >= 0 && gr.slot < n_slots && gr.row_begin >= 0 && gr.row_count >= 0 &&
                   gr.row_begin + gr.row_count <= total_rows,
               HM_EVALUE, "expert group outside the pool or the row range");
    if (gr.row_count == 0) continue;
    const bool gemv = path == HM_FFN_GEMV || path == HM_FFN_GEMV_SPLIT || path == HM_FFN_GEMV_FUSED ||
                      (path == HM_FFN_AUTO && gr.row_count <= hm::kGemvMaxRows);
    if (gemv) {
      HM_REQUIRE(gr.row_count <= hm::kGemvMaxRows, HM_EVALUE, "GEMV path takes at most 4 rows per expert");
      small.push_back(gr);
    } else {
      big.push_back(gr);
    }
  }
  const size_t slot_elems = static_cast<size_t>(3) * H * I;
  for (size_t b = 0; b < small.size(); b += hm::kMaxGroups) {
    std::vector<hm_group> part(small.begin() + b, small.begin() + std::min(small.size(), b + hm::kMaxGroups));
    hm::launch_gemv(pool, slot_elems, H, I, part, xp, h, out, st, path);
  }
  for (size_t b = 0; b < big.size(); b += hm::kMaxGroups) {
    std::vector<hm_group> part(big.begin() + b, big.begin() + std::min(big.size(), b + hm::kMaxGroups));
    hm::launch_gemm(pool, n_slots, H, I, part, xp, total_rows, h, out, st);
  }
  HM_API_END
}

}  // extern "C"
