// Expert-parallel exchange over peer memory: the
// combine of Eq. 1 fused with the cross-rank reduction in ONE
// kernel, instead of combine -> NCCL all-reduce -> residual add.
//
// Every rank holds the replicated hidden state and routes it identically; it
// computes only its home experts (e % G == rank), so its weighted combine is a
// partial sum.  Each block of hm_ep_combine_allreduce owns one tile (token t,
// 512 columns):
//   1. partial = sum_k w[t,k] * out[pos[t,k], cols]   (non-home w are 0; rows
//      of host-worker experts read zero-copy from mapped host memory)
//   2. st.global the partial into inbox[parity][rank][t, cols] of EVERY rank
//      (NVLink P2P stores through CUDA IPC mappings), fence.sys, then raise
//      flag[parity][rank][tile] = seq on every rank
//   3. wait until flag[parity][r][tile] == seq for all r (own inbox), then
//      y[t, cols] = residual + sum_{r = 0..G-1} inbox[parity][r][t, cols]
//      in rank order -- every rank computes bit-identical y.
// The grid is persistent (tiles strided over co-resident blocks, each block
// signals a tile before waiting on it), which keeps the cross-GPU waits
// deadlock-free.  Inbox and flags are double-buffered by the parity of the
// call sequence number: a rank can run at most one exchange ahead of a peer.
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "device.cuh"

namespace hm {
namespace {

constexpr int kEpThreads = 128;  // x 4 columns = 512 columns per tile
constexpr int kEpMaxWorld = 8;
constexpr int kEpMaxKp = 64;

struct EpParams {
  const float *out, *host_out;
  const int32_t *pos;
  const float *w;
  int T, Kp, H, cs, n_tiles;
  const uint16_t *residual;
  uint16_t *y;
  float *y32;  // optional fp32 copy of the reduced MoE sum (without residual)
  unsigned long long host_mask[4];
  int rank, world;
  uint32_t seq;
  size_t inbox_stride;  // floats per (parity, rank) block = max_rows * H
  int max_tiles;
  float *inbox[kEpMaxWorld];     // peer r's inbox base (parity 0, src 0)
  uint32_t *flags[kEpMaxWorld];  // peer r's flag base (parity 0, src 0)
};

__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(kEpThreads) ep_combine_allreduce_kernel(const __grid_constant__ EpParams p) {
  __shared__ float s_w[kEpMaxKp];
  __shared__ int32_t s_pos[kEpMaxKp];
  const int par = static_cast<int>(p.seq & 1u);
  for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
    const int t = tile / p.cs, col = ((tile % p.cs) * kEpThreads + threadIdx.x) * 4;
    __syncthreads();  // s_w / s_pos reuse across tiles
    for (int k = threadIdx.x; k < p.Kp; k += blockDim.x) {
      s_w[k] = p.w[static_cast<size_t>(t) * p.Kp + k];
      s_pos[k] = p.pos[static_cast<size_t>(t) * p.Kp + k];
    }
    __syncthreads();
    const bool active = col < p.H;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    if (active) {
      constexpr int U = 8;
      for (int k0 = 0; k0 < p.Kp; k0 += U) {
        float4 o[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int k = k0 + u;
          o[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (k < p.Kp && s_w[k] != 0.0f) {
            const int pp = s_pos[k];
            const bool host = pp < 256 && ((p.host_mask[pp >> 6] >> (pp & 63)) & 1ull);
            o[u] = *reinterpret_cast<const float4 *>((host ? p.host_out : p.out) + static_cast<size_t>(pp) * p.H + col);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int k = k0 + u;
          if (k < p.Kp && s_w[k] != 0.0f) {
            const float wk = s_w[k];
            a.x = fmaf(wk, o[u].x, a.x);
            a.y = fmaf(wk, o[u].y, a.y);
            a.z = fmaf(wk, o[u].z, a.z);
            a.w = fmaf(wk, o[u].w, a.w);
          }
        }
      }
      // push the partial into every rank's inbox slot [par][rank]
      const size_t off = (static_cast<size_t>(par) * p.world + p.rank) * p.inbox_stride +
                         static_cast<size_t>(t) * p.H + col;
      for (int r = 0; r < p.world; ++r) *reinterpret_cast<float4 *>(p.inbox[r] + off) = a;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x < p.world) {  // raise this tile's flag on every rank
      const size_t fo = (static_cast<size_t>(par) * p.world + p.rank) * p.max_tiles + tile;
      st_release_sys(p.flags[threadIdx.x] + fo, p.seq);
    }
    if (threadIdx.x < p.world) {  // wait for every rank's partial of this tile
      const uint32_t *f = p.flags[p.rank] + (static_cast<size_t>(par) * p.world + threadIdx.x) * p.max_tiles + tile;
      while (ld_acquire_sys(f) != p.seq) {
      }
    }
    __syncthreads();
    if (!active) continue;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    const float *mine = p.inbox[p.rank] + static_cast<size_t>(par) * p.world * p.inbox_stride +
                        static_cast<size_t>(t) * p.H + col;
    for (int r = 0; r < p.world; ++r) {  // rank order: identical on every rank
      const float4 v = __ldcv(reinterpret_cast<const float4 *>(mine + static_cast<size_t>(r) * p.inbox_stride));
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
    if (p.y32) *reinterpret_cast<float4 *>(p.y32 + static_cast<size_t>(t) * p.H + col) = s;
    if (p.y) {
      if (p.residual) {
        const uint2 rv = *reinterpret_cast<const uint2 *>(p.residual + static_cast<size_t>(t) * p.H + col);
        s.x += dev::bf_lo(rv.x);
        s.y += dev::bf_hi(rv.x);
        s.z += dev::bf_lo(rv.y);
        s.w += dev::bf_hi(rv.y);
      }
      uint2 o2;
      o2.x = dev::pack_bf2(s.x, s.y);
      o2.y = dev::pack_bf2(s.z, s.w);
      *reinterpret_cast<uint2 *>(p.y + static_cast<size_t>(t) * p.H + col) = o2;
    }
  }
}

}  // namespace

struct EpExchange {
  int rank, world, max_rows, H, cs, max_tiles;
  size_t inbox_stride;
  float *inbox = nullptr;     // local: [2][world][max_rows * H] fp32
  uint32_t *flags = nullptr;  // local: [2][world][max_tiles]
  float *peer_inbox[kEpMaxWorld] = {};
  uint32_t *peer_flags[kEpMaxWorld] = {};
  bool opened[kEpMaxWorld] = {};
  uint32_t seq = 0;
  int grid = 0;

  EpExchange(int r, int w, int rows, int h) : rank(r), world(w), max_rows(rows), H(h) {
    HM_REQUIRE(w >= 1 && w <= kEpMaxWorld && r >= 0 && r < w, HM_EVALUE, "expert-parallel world must be 1..8");
    HM_REQUIRE(rows >= 1 && h % 4 == 0, HM_EVALUE, "bad exchange shape");
    cs = (H + 4 * kEpThreads - 1) / (4 * kEpThreads);
    max_tiles = max_rows * cs;
    inbox_stride = static_cast<size_t>(max_rows) * H;
    HM_CUDA(cudaMalloc(&inbox, 2ull * world * inbox_stride * sizeof(float)));
    HM_CUDA(cudaMalloc(&flags, 2ull * world * max_tiles * sizeof(uint32_t)));
    HM_CUDA(cudaMemset(flags, 0, 2ull * world * max_tiles * sizeof(uint32_t)));
    peer_inbox[rank] = inbox;
    peer_flags[rank] = flags;
    opened[rank] = true;
    int dev = 0, sms = 0, per_sm = 0;
    HM_CUDA(cudaGetDevice(&dev));
    HM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    HM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ep_combine_allreduce_kernel, kEpThreads, 0));
    grid = sms * (per_sm > 4 ? 4 : per_sm);  // co-resident persistent grid
    HM_CUDA(cudaDeviceSynchronize());
  }
  ~EpExchange() {
    for (int r = 0; r < world; ++r)
      if (r != rank && opened[r]) {
        cudaIpcCloseMemHandle(peer_inbox[r]);
        cudaIpcCloseMemHandle(peer_flags[r]);
      }
    if (inbox) cudaFree(inbox);
    if (flags) cudaFree(flags);
  }
};

}  // namespace hm

extern "C" {

int hm_ep_create(int rank, int world, int max_rows, int H, hm_ep **out) {
  HM_API_BEGIN
  HM_REQUIRE(out, HM_EVALUE, "null argument");
  *out = reinterpret_cast<hm_ep *>(new hm::EpExchange(rank, world, max_rows, H));
  HM_API_END
}

void hm_ep_destroy(hm_ep *ep) { delete reinterpret_cast<hm::EpExchange *>(ep); }

int hm_ep_ipc_handles(hm_ep *ep, void *inbox_handle, void *flags_handle) {
  HM_API_BEGIN
  auto *e = reinterpret_cast<hm::EpExchange *>(ep);
  HM_REQUIRE(inbox_handle && flags_handle, HM_EVALUE, "null handle buffer");
  HM_CUDA(cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t *>(inbox_handle), e->inbox));
  HM_CUDA(cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t *>(flags_handle), e->flags));
  HM_API_END
}

int hm_ep_open_peer(hm_ep *ep, int peer, const void *inbox_handle, const void *flags_handle) {
  HM_API_BEGIN
  auto *e = reinterpret_cast<hm::EpExchange *>(ep);
  HM_REQUIRE(peer >= 0 && peer < e->world, HM_EVALUE, "peer rank out of range");
  if (peer == e->rank || e->opened[peer]) return HM_OK;
  cudaIpcMemHandle_t hi, hf;
  memcpy(&hi, inbox_handle, sizeof hi);
  memcpy(&hf, flags_handle, sizeof hf);
  void *pi = nullptr, *pf = nullptr;
  HM_CUDA(cudaIpcOpenMemHandle(&pi, hi, cudaIpcMemLazyEnablePeerAccess));
  HM_CUDA(cudaIpcOpenMemHandle(&pf, hf, cudaIpcMemLazyEnablePeerAccess));
  e->peer_inbox[peer] = static_cast<float *>(pi);
  e->peer_flags[peer] = static_cast<uint32_t *>(pf);
  e->opened[peer] = true;
  HM_API_END
}

int hm_ep_combine_allreduce(hm_ep *ep, const float *out, const float *host_out, const uint64_t *host_mask4,
                            const int32_t *pos, const float *w, int T, int Kp, int H, const uint16_t *residual,
                            uint16_t *y, float *y32, void *stream) {
  HM_API_BEGIN
  auto *e = reinterpret_cast<hm::EpExchange *>(ep);
  HM_REQUIRE(H == e->H && T >= 0 && T <= e->max_rows, HM_EVALUE, "exchange shape exceeds the buffers");
  HM_REQUIRE(Kp >= 1 && Kp <= hm::kEpMaxKp, HM_EVALUE, "too many selections per token");
  for (int r = 0; r < e->world; ++r) HM_REQUIRE(e->opened[r], HM_EVALUE, "exchange peers not opened");
  HM_REQUIRE(!host_mask4 || host_out, HM_EVALUE, "host rows need the host output buffer");
  if (T == 0) return HM_OK;
  hm::EpParams p{};
  p.out = out;
  p.host_out = host_out;
  p.pos = pos;
  p.w = w;
  p.T = T;
  p.Kp = Kp;
  p.H = H;
  p.cs = e->cs;
  p.n_tiles = T * e->cs;
  p.residual = residual;
  p.y = y;
  p.y32 = y32;
  for (int i = 0; i < 4; ++i) p.host_mask[i] = host_mask4 ? host_mask4[i] : 0ull;
  p.rank = e->rank;
  p.world = e->world;
  p.seq = ++e->seq;
  p.inbox_stride = e->inbox_stride;
  p.max_tiles = e->max_tiles;
  for (int r = 0; r < e->world; ++r) {
    p.inbox[r] = e->peer_inbox[r];
    p.flags[r] = e->peer_flags[r];
  }
  const int grid = p.n_tiles < e->grid ? p.n_tiles : e->grid;
  hm::ep_combine_allreduce_kernel<<<grid, hm::kEpThreads, 0, static_cast<cudaStream_t>(stream)>>>(p);
  HM_LAUNCH_CHECK();
  HM_API_END
}

}  // extern "C"
