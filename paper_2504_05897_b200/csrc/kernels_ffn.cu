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
template <int MR, int U = 4>
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
template <int MR, int RW = 2, int U = 4>
__global__ void __launch_bounds__(256) ffn2_gemv_kernel(const __grid_constant__ GemvParams p) {
  extern __shared__ __align__(16) uint16_t hs[];  // [MR][I]
  const int g = blockIdx.x / p.bpg, cid = blockIdx.x % p.bpg;
  const int M = p.row_count[g], rb = p.row_begin[g], H = p.H, I = p.I;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint16_t *w2 = p.pool + static_cast<size_t>(p.slot[g]) * p.slot_elems + static_cast<size_t>(2) * I * H;
  const int j_end = min(H, (cid + 1) * p.chunk);
  // RW rows per warp at a time (rows j, j + nw, ..): RW x U loads in flight
  // per lane -- small-I experts (DeepSeek: 2.8 KB rows) were latency-bound
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

// ------------------------------------------------------------ stream-read floor
// The achievable floor of a weight-streaming launch of a given size: every
// thread streams 16-byte L1-bypassing loads (U in flight) over a contiguous
// byte range and folds them into one word per block.  hm_bench_stream_read
// times it back to back (and as a dependent pair, like ffn1 -> ffn2) so the
// GEMV's per-size efficiency can be read against what a pure read achieves.
__global__ void __launch_bounds__(256) stream_read_kernel(const uint4 *src, size_t n16, uint32_t *sink) {
  constexpr int U = 8;
  uint32_t acc = 0;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = dev::ld_stream(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n16; i += stride) {
    const uint4 v = dev::ld_stream(src + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  acc = __reduce_xor_sync(0xffffffffu, acc);
  if ((threadIdx.x & 31) == 0 && acc == 0x9e3779b9u) sink[blockIdx.x] = acc;  // keep the loads live
}

// ------------------------------------------------------------ bulk-copy decode GEMV
// The same ffn1 -> ffn2 pair with the weights moved by the bulk-copy engine
// (cp.async.bulk, mbarrier complete_tx) instead of per-lane loads.  Every
// warp runs its own ring of kBulkMaxStages stage buffers in shared memory and
// streams a contiguous range of work units through it: lane 0 keeps up to S
// stages in flight (2 copies per ffn1 stage: gate and up rows; 1..NR rows per
// ffn2 stage), all lanes wait on the stage's mbarrier, take their dot products
// from shared memory and hand the stage back.  So each warp has S x 4-8 KB in
// flight at every instant with no register cost, where the register kernels
// above hold one 4 KB batch and pay one DRAM round trip per batch: small
// experts (DeepSeek's 2048 x 1408) were a short chain of such round trips per
// warp.  Per lane the columns are accumulated in the register kernels' order
// (c = lane*8 + 256k, k increasing, chunk after chunk): outputs are
// bit-identical to ffn1/ffn2_gemv_kernel.
constexpr int kBulkMaxStages = 4;
constexpr int kBulkWarps = 8;

struct BulkParams {
  const uint16_t *pool;
  size_t slot_elems;
  int H, I;
  int n_units;      // ffn1: G*I (gate, up) pairs; ffn2: G*ceil(H/nr) row blocks
  int units_per_group;
  int ck, nck;      // columns per stage chunk, chunks per unit
  int nr;           // ffn2: W2 rows per stage (nck == 1 when nr > 1)
  int stages;       // ring depth per warp (<= kBulkMaxStages)
  int stage_bytes;  // bytes per stage buffer (multiple of 128)
  const uint16_t *xp;
  uint16_t *h;
  float *out;
  int32_t slot[kMaxGroups];
  int32_t row_begin[kMaxGroups];
  int32_t row_count[kMaxGroups];
};

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dev::smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(dev::smem_u32(bar))
      : "memory");
}

// the warp's contiguous unit range, balanced over all warps of the grid
__device__ __forceinline__ void bulk_range(int n_units, int &u0, int &u1) {
  const long W = static_cast<long>(gridDim.x) * kBulkWarps;
  const long w = static_cast<long>(blockIdx.x) * kBulkWarps + (threadIdx.x >> 5);
  u0 = static_cast<int>(n_units * w / W);
  u1 = static_cast<int>(n_units * (w + 1) / W);
}

// ffn1 step t of unit range [u0, ..): unit u0 + t / nck, column chunk t % nck
__device__ __forceinline__ void bulk_issue1(const BulkParams &p, int u0, int t, uint16_t *stage, uint64_t *bar) {
  const int u = u0 + t / p.nck, c = t - (t / p.nck) * p.nck;
  const int g = u / p.I, i = u - g * p.I;
  const uint16_t *w13 = p.pool + static_cast<size_t>(p.slot[g]) * p.slot_elems;
  const size_t grow = static_cast<size_t>((i / kIlv) * 2 * kIlv + (i % kIlv));
  const int c0 = c * p.ck, cols = min(p.ck, p.H - c0);
  const uint16_t *wg = w13 + grow * p.H + c0;
  const uint32_t bytes = static_cast<uint32_t>(cols) * 2;
  dev::mbar_arrive_expect_tx(bar, 2 * bytes);
  bulk_g2s(stage, wg, bytes, bar);
  bulk_g2s(stage + p.ck, wg + static_cast<size_t>(kIlv) * p.H, bytes, bar);
}

// Activations are read through L1 (__ldg): a warp's unit range can span
// groups, each with its own rows, and the few KB per group stay L1-resident.
template <int MR>
__global__ void __launch_bounds__(kBulkWarps * 32, 1) ffn1_bulk_kernel(const __grid_constant__ BulkParams p) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ uint64_t bars[kBulkWarps][kBulkMaxStages];
  asm volatile("griddepcontrol.launch_dependents;");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int H = p.H, I = p.I, S = p.stages;
  uint8_t *ring = smem_raw + static_cast<size_t>(wid) * S * p.stage_bytes;
  auto stage = [&](int s) { return reinterpret_cast<uint16_t *>(ring + static_cast<size_t>(s) * p.stage_bytes); };
  int u0, u1;
  bulk_range(p.n_units, u0, u1);
  const int steps = (u1 - u0) * p.nck;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) dev::mbar_init(&bars[wid][s], 1);
    dev::fence_barrier_init();
    for (int t = 0; t < min(S, steps); ++t) bulk_issue1(p, u0, t, stage(t), &bars[wid][t]);
  }
  __syncwarp();
  float ag[MR], au[MR];
#pragma unroll
  for (int m = 0; m < MR; ++m) ag[m] = au[m] = 0.f;
  for (int t = 0; t < steps; ++t) {
    const int u = u0 + t / p.nck, c = t - (t / p.nck) * p.nck;
    const int g = u / I, i = u - g * I;
    const int M = p.row_count[g], rb = p.row_begin[g];
    const uint16_t *x = p.xp + static_cast<size_t>(rb) * H;
    const int s = t % S;
    dev::mbar_wait(&bars[wid][s], static_cast<uint32_t>((t / S) & 1));
    const uint16_t *sg = stage(s), *su = sg + p.ck;
    const int c0 = c * p.ck, cols = min(p.ck, H - c0);
    for (int k = lane * 8; k < cols; k += 256) {
      const uint4 wg = *reinterpret_cast<const uint4 *>(sg + k);
      const uint4 wu = *reinterpret_cast<const uint4 *>(su + k);
#pragma unroll
      for (int m = 0; m < MR; ++m) {
        if (m < M) {
          const uint4 xv = __ldg(reinterpret_cast<const uint4 *>(x + static_cast<size_t>(m) * H + c0 + k));
          ag[m] += dev::dot8(wg, xv);
          au[m] += dev::dot8(wu, xv);
        }
      }
    }
    __syncwarp();
    if (lane == 0 && t + S < steps) bulk_issue1(p, u0, t + S, stage(s), &bars[wid][s]);
    if (c == p.nck - 1) {
#pragma unroll
      for (int m = 0; m < MR; ++m) {
        if (m < M) {
          const float gs = dev::warp_sum(ag[m]), us = dev::warp_sum(au[m]);
          if (lane == 0) p.h[static_cast<size_t>(rb + m) * I + i] = dev::f2bf(dev::silu(gs) * us);
        }
        ag[m] = au[m] = 0.f;
      }
    }
  }
}

// ffn2 step t: unit u0 + t / nck is a block of nr W2 rows (nck == 1) or one
// row's column chunk t % nck (nr == 1)
__device__ __forceinline__ void bulk_issue2(const BulkParams &p, int u0, int t, uint16_t *stage, uint64_t *bar) {
  const int u = u0 + t / p.nck, c = t - (t / p.nck) * p.nck;
  const int g = u / p.units_per_group, j0 = (u - g * p.units_per_group) * p.nr;
  const int rows = min(p.nr, p.H - j0);
  const uint16_t *w2 = p.pool + static_cast<size_t>(p.slot[g]) * p.slot_elems + static_cast<size_t>(2) * p.I * p.H;
  const int c0 = c * p.ck, cols = min(p.ck, p.I - c0);
  // nr > 1 only with whole rows (ck == I): the rows are contiguous
  const uint32_t bytes = static_cast<uint32_t>(rows) * cols * 2;
  dev::mbar_arrive_expect_tx(bar, bytes);
  bulk_g2s(stage, w2 + static_cast<size_t>(j0) * p.I + c0, bytes, bar);
}

// W2's first stages are issued BEFORE the programmatic wait for ffn1: they do
// not depend on h.  h is read through L1 like the activations above.
template <int MR, int NR>
__global__ void __launch_bounds__(kBulkWarps * 32, 1) ffn2_bulk_kernel(const __grid_constant__ BulkParams p) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ uint64_t bars[kBulkWarps][kBulkMaxStages];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int H = p.H, I = p.I, S = p.stages;
  uint8_t *ring = smem_raw + static_cast<size_t>(wid) * S * p.stage_bytes;
  auto stage = [&](int s) { return reinterpret_cast<uint16_t *>(ring + static_cast<size_t>(s) * p.stage_bytes); };
  int u0, u1;
  bulk_range(p.n_units, u0, u1);
  const int steps = (u1 - u0) * p.nck;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) dev::mbar_init(&bars[wid][s], 1);
    dev::fence_barrier_init();
    for (int t = 0; t < min(S, steps); ++t) bulk_issue2(p, u0, t, stage(t), &bars[wid][t]);
  }
  __syncwarp();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  float acc[MR][NR];
#pragma unroll
  for (int m = 0; m < MR; ++m)
#pragma unroll
    for (int r = 0; r < NR; ++r) acc[m][r] = 0.f;
  for (int t = 0; t < steps; ++t) {
    const int u = u0 + t / p.nck, c = t - (t / p.nck) * p.nck;
    const int g = u / p.units_per_group, j0 = (u - g * p.units_per_group) * p.nr;
    const int M = p.row_count[g], rb = p.row_begin[g];
    const int rows = min(p.nr, H - j0);
    const uint16_t *hr = p.h + static_cast<size_t>(rb) * I;
    const int s = t % S;
    dev::mbar_wait(&bars[wid][s], static_cast<uint32_t>((t / S) & 1));
    const uint16_t *sw = stage(s);
    const int c0 = c * p.ck, cols = min(p.ck, I - c0);
    for (int k = lane * 8; k < cols; k += 256) {
#pragma unroll
      for (int m = 0; m < MR; ++m) {
        if (m < M) {
          const uint4 hv = __ldcg(reinterpret_cast<const uint4 *>(hr + static_cast<size_t>(m) * I + c0 + k));
#pragma unroll
          for (int r = 0; r < NR; ++r)
            if (r < rows) acc[m][r] += dev::dot8(*reinterpret_cast<const uint4 *>(sw + r * cols + k), hv);
        }
      }
    }
    __syncwarp();
    if (lane == 0 && t + S < steps) bulk_issue2(p, u0, t + S, stage(s), &bars[wid][s]);
    if (c == p.nck - 1) {
#pragma unroll
      for (int m = 0; m < MR; ++m) {
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          if (m < M && r < rows) {
            const float v = dev::warp_sum(acc[m][r]);
            if (lane == 0) p.out[static_cast<size_t>(rb + m) * H + j0 + r] = v;
          }
          acc[m][r] = 0.f;
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

bool gemv_narrow_enabled() {
  static const bool on = [] {
    const char *e = std::getenv("HM_GEMV_NARROW");
    return e && std::atoi(e) != 0;
  }();
  return on;
}
int gemv_narrow_rows_per_warp() {
  static const int v = [] {
    const char *e = std::getenv("HM_GEMV_NARROW_RPW");
    return e ? std::max(1, std::min(8, std::atoi(e))) : 1;
  }();
  return v;
}

// HM_GEMV_BULK=1 makes the bulk-copy pair the default GEMV (A/B switch);
// HM_BULK_SMEM_KB sets the ring budget per CTA (default 192: one CTA per SM).
bool gemv_bulk_enabled() {
  static const bool on = [] {
    const char *e = std::getenv("HM_GEMV_BULK");
    return e && std::atoi(e) != 0;
  }();
  return on;
}
int bulk_smem_budget() {
  static const int kb = [] {
    const char *e = std::getenv("HM_BULK_SMEM_KB");
    const int v = e ? std::atoi(e) : 192;
    return std::max(24, std::min(v, 200));
  }();
  return kb * 1024;
}

template <typename K>
void launch_bulk(K kernel, int grid, int smem, bool pdl, cudaStream_t st, const BulkParams &p) {
  set_smem(kernel, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kBulkWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl && pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  HM_CUDA(cudaLaunchKernelEx(&cfg, kernel, p));
  HM_LAUNCH_CHECK();
}

void launch_gemv_bulk(const uint16_t *pool, size_t slot_elems, int H, int I, const std::vector<hm_group> &gs,
                      const uint16_t *xp, uint16_t *h, float *out, cudaStream_t st) {
  BulkParams p{};
  p.pool = pool;
  p.slot_elems = slot_elems;
  p.H = H;
  p.I = I;
  p.xp = xp;
  p.h = h;
  p.out = out;
  int mr = 1;
  const int G = static_cast<int>(gs.size());
  for (int g = 0; g < G; ++g) {
    p.slot[g] = gs[g].slot;
    p.row_begin[g] = gs[g].row_begin;
    p.row_count[g] = gs[g].row_count;
    mr = std::max(mr, gs[g].row_count);
  }
  const int budget = bulk_smem_budget();
  const int per_sm = budget <= 110 * 1024 ? 2 : 1;
  const int grid = num_sms() * per_sm;
  auto ring = [&](int stage_bytes) {
    p.stage_bytes = (stage_bytes + 127) / 128 * 128;
    p.stages = std::max(1, std::min(kBulkMaxStages, budget / (kBulkWarps * p.stage_bytes)));
    return kBulkWarps * p.stages * p.stage_bytes;
  };
  // ffn1: (gate, up) row pairs, columns in chunks of <= 2048 (8 KB stages)
  p.nck = (H + 2047) / 2048;
  p.ck = ((H + p.nck - 1) / p.nck + 7) / 8 * 8;
  p.nr = 1;
  p.n_units = G * I;
  p.units_per_group = I;
  int smem = ring(2 * p.ck * 2);
  switch (mr) {
    case 1: launch_bulk(ffn1_bulk_kernel<1>, grid, smem, false, st, p); break;
    case 2: launch_bulk(ffn1_bulk_kernel<2>, grid, smem, false, st, p); break;
    default: launch_bulk(ffn1_bulk_kernel<4>, grid, smem, false, st, p); break;
  }
  // ffn2: blocks of whole W2 rows up to 12 KB, or one row in <= 8 KB chunks
  const int row_bytes = I * 2;
  if (row_bytes <= 6 * 1024) {
    p.nck = 1;
    p.ck = I;
    p.nr = std::max(1, std::min(4, (12 * 1024) / row_bytes));
  } else {
    p.nr = 1;
    p.nck = (I + 4095) / 4096;
    p.ck = ((I + p.nck - 1) / p.nck + 7) / 8 * 8;
  }
  p.units_per_group = (H + p.nr - 1) / p.nr;
  p.n_units = G * p.units_per_group;
  smem = ring(p.nr * p.ck * 2);
  const int nrk = p.nr == 1 ? 1 : p.nr == 2 ? 2 : 4;
  switch (mr * 8 + nrk) {
    case 9: launch_bulk(ffn2_bulk_kernel<1, 1>, grid, smem, true, st, p); break;
    case 10: launch_bulk(ffn2_bulk_kernel<1, 2>, grid, smem, true, st, p); break;
    case 12: launch_bulk(ffn2_bulk_kernel<1, 4>, grid, smem, true, st, p); break;
    case 17: launch_bulk(ffn2_bulk_kernel<2, 1>, grid, smem, true, st, p); break;
    case 18: launch_bulk(ffn2_bulk_kernel<2, 2>, grid, smem, true, st, p); break;
    case 20: launch_bulk(ffn2_bulk_kernel<2, 4>, grid, smem, true, st, p); break;
    case 33: case 25: launch_bulk(ffn2_bulk_kernel<4, 1>, grid, smem, true, st, p); break;
    case 34: case 26: launch_bulk(ffn2_bulk_kernel<4, 2>, grid, smem, true, st, p); break;
    default: launch_bulk(ffn2_bulk_kernel<4, 4>, grid, smem, true, st, p); break;
  }
}

// path HM_FFN_GEMV: HM_GEMV_FUSED decides; HM_FFN_GEMV_SPLIT / _FUSED force one
void launch_gemv(const uint16_t *pool, size_t slot_elems, int H, int I, const std::vector<hm_group> &gs,
                 const uint16_t *xp, uint16_t *h, float *out, cudaStream_t st, int path) {
  if (gs.empty()) return;
  if (path == HM_FFN_GEMV_BULK || ((path == HM_FFN_GEMV || path == HM_FFN_AUTO) && gemv_bulk_enabled())) {
    HM_REQUIRE(static_cast<int>(gs.size()) <= kMaxGroups, HM_EVALUE, "too many expert groups in one launch");
    HM_REQUIRE(H % 8 == 0 && I % 8 == 0 && I % kIlv == 0, HM_EVALUE, "GEMV needs H % 8 == 0 and I % 128 == 0");
    launch_gemv_bulk(pool, slot_elems, H, I, gs, xp, h, out, st);
    return;
  }
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
  // narrow experts (a whole W13 row pair / W2 row in one batch of U loads per
  // lane): every warp's bytes go out in ONE DRAM round trip and the grid is
  // sized to a fixed number of rows per warp (HM_GEMV_NARROW=1; measured
  // slower than the 4-load batches at every DeepSeek count, so off;
  // HM_GEMV_NARROW_RPW: rows per warp)
  const bool narrow1 = gemv_narrow_enabled() && H <= 2048;
  const bool narrow2 = gemv_narrow_enabled() && I <= 2048;
  const int rpw = gemv_narrow_rows_per_warp();
  // ffn1: pairs of (gate, up) rows
  int chunk = static_cast<int>((static_cast<long>(G) * I + target - 1) / target);
  chunk = std::max(8, (chunk + 7) / 8 * 8);
  if (narrow1) chunk = 8 * rpw;
  p.chunk = chunk;
  p.bpg = (I + chunk - 1) / chunk;
  int smem = mr * H * 2;
  HM_REQUIRE(smem <= 200 * 1024, HM_EVALUE, "decode rows do not fit shared memory");
  auto l1 = [&](auto kern) {
    set_smem(kern, smem);
    kern<<<G * p.bpg, 256, smem, st>>>(p);
  };
  if (narrow1) {
    switch (mr) {
      case 1: l1(ffn1_gemv_kernel<1, 8>); break;
      case 2: l1(ffn1_gemv_kernel<2, 8>); break;
      default: l1(ffn1_gemv_kernel<4, 8>); break;
    }
  } else {
    switch (mr) {
      case 1: l1(ffn1_gemv_kernel<1>); break;
      case 2: l1(ffn1_gemv_kernel<2>); break;
      default: l1(ffn1_gemv_kernel<4>); break;
    }
  }
  HM_LAUNCH_CHECK();
  chunk = static_cast<int>((static_cast<long>(G) * H + target - 1) / target);
  chunk = std::max(8, (chunk + 7) / 8 * 8);
  if (narrow2) chunk = 8 * rpw;
  p.chunk = chunk;
  p.bpg = (H + chunk - 1) / chunk;
  smem = mr * I * 2;
  HM_REQUIRE(smem <= 200 * 1024, HM_EVALUE, "decode rows do not fit shared memory");
  // warm L2 only while the layer's W2 bytes fit comfortably in the 126 MB L2
  p.l2_prefetch = !narrow2 && static_cast<long>(G) * H * I * 2 <= (64L << 20) ? 1 : 0;
  if (narrow2) {
    switch (mr) {
      case 1: launch_pdl(ffn2_gemv_kernel<1, 1, 8>, G * p.bpg, smem, st, p); break;
      case 2: launch_pdl(ffn2_gemv_kernel<2, 1, 8>, G * p.bpg, smem, st, p); break;
      default: launch_pdl(ffn2_gemv_kernel<4, 1, 8>, G * p.bpg, smem, st, p); break;
    }
  } else {
    switch (mr) {
      case 1: launch_pdl(ffn2_gemv_kernel<1>, G * p.bpg, smem, st, p); break;
      case 2: launch_pdl(ffn2_gemv_kernel<2>, G * p.bpg, smem, st, p); break;
      default: launch_pdl(ffn2_gemv_kernel<4>, G * p.bpg, smem, st, p); break;
    }
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

// Pure-read floor for a launch of `bytes` (and, pair != 0, two dependent
// launches of bytes*2/3 and bytes/3 -- the ffn1 / ffn2 split of an expert),
// over `n_buf` rotating buffers of `bytes` each at `base`.
int hm_bench_stream_read(const void *base, size_t bytes, int n_buf, int pair, int blocks_per_sm, int reps,
                         void *stream, float *ms) {
  HM_API_BEGIN
  HM_REQUIRE(base && bytes >= 16 && n_buf >= 1 && reps >= 1 && blocks_per_sm >= 1, HM_EVALUE, "bad bench");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint32_t *sink = nullptr;
  const int grid = hm::num_sms() * blocks_per_sm;
  HM_CUDA(cudaMallocAsync(&sink, static_cast<size_t>(grid) * 4, st));
  auto one = [&](int i) {
    const char *b = static_cast<const char *>(base) + static_cast<size_t>(i % n_buf) * bytes;
    if (!pair) {
      hm::stream_read_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4 *>(b), bytes / 16, sink);
    } else {
      const size_t a = bytes * 2 / 3 / 16 * 16;
      hm::stream_read_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4 *>(b), a / 16, sink);
      hm::stream_read_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4 *>(b + a), (bytes - a) / 16, sink);
    }
    HM_LAUNCH_CHECK();
  };
  for (int i = 0; i < 3; ++i) one(i);
  cudaEvent_t e0, e1;
  HM_CUDA(cudaEventCreate(&e0));
  HM_CUDA(cudaEventCreate(&e1));
  HM_CUDA(cudaEventRecord(e0, st));
  for (int i = 0; i < reps; ++i) one(3 + i);
  HM_CUDA(cudaEventRecord(e1, st));
  HM_CUDA(cudaEventSynchronize(e1));
  HM_CUDA(cudaEventElapsedTime(ms, e0, e1));
  *ms /= static_cast<float>(reps);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  HM_CUDA(cudaFreeAsync(sink, st));
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
                      path == HM_FFN_GEMV_BULK ||
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
