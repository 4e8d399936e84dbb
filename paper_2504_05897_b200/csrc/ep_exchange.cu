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
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
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
      while (static_cast<int32_t>(ld_acquire_sys(f) - p.seq) < 0) {  // reached (wrap-safe)
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

// ---------------------------------------------------------------- dispatch mode
// Token-sharded expert parallelism (SURVEY.md §8e "dispatch: all-to-all(v) of
// token rows to home ranks ... combine: all-to-all(v) back plus weighted
// sum"): each rank routes only ITS tokens; three kernels per layer move data
// over peer memory:
//   ep_meta_kernel      all-gather of every rank's per-expert counts and fp64
//                       score sums -> global LayerRequest (rank-order sums,
//                       identical on every rank), the home-rank row layout and
//                       the host mirror + flag the decision core waits on
//   ep_dispatch_kernel  all-to-all: each local permuted row -> its expert's
//                       home rank, at (home base of e) + (rows of e from lower
//                       ranks) + (rank within e)
//   ep_return_kernel    all-to-all back: each expert output row -> its source
//                       rank, at the source's own permuted position
// after which the source combines locally (hm_combine).  Home layout: experts
// in index order, inside an expert rows by source rank then source order.
constexpr int kDispMaxE = 320;

struct DispParams {
  // region layout (byte offsets, identical on every rank)
  size_t off_meta, off_mflags, off_dflags, off_rflags, off_xrecv, off_ret, meta_slot;
  char *region[kEpMaxWorld];  // every rank's region (own included)
  int rank, world, E, N, H, Kp;
  uint32_t seq;
  // local tables (device)
  int32_t *counts_all;  // [world][E]
  int32_t *recv_base;   // [E]   row base of expert e inside its home rank's layout
  int32_t *src_base;    // [world + 1][E] rows of e from ranks < s
  int32_t *local_off;   // [world][E + 1] rank s's own permuted offsets
  int32_t *gcount;      // [E]
  int32_t *ret_map;     // [max received rows] (source rank << 24) | source position
  int32_t *done;        // [2] block-completion counters (dispatch, return)
};

__device__ __forceinline__ int home_of(int e, int N, int world) { return (e < N ? e : e - N) % world; }

// Last-block protocol: every block fences its peer stores; the last block to
// finish raises this rank's flag on every rank, then waits for every rank's
// flag on its own region (so the kernel completes only when all incoming
// rows have landed), and resets the counter.
__device__ void all_to_all_handshake(const DispParams &p, size_t off_flags, int *done) {
  __threadfence_system();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(done, 1) == static_cast<int>(gridDim.x) - 1;
  __syncthreads();
  if (!last) return;
  if (threadIdx.x < p.world)
    st_release_sys(reinterpret_cast<uint32_t *>(p.region[threadIdx.x] + off_flags) + p.rank, p.seq);
  if (threadIdx.x < p.world) {
    const uint32_t *f = reinterpret_cast<const uint32_t *>(p.region[p.rank] + off_flags) + threadIdx.x;
    while (static_cast<int32_t>(ld_acquire_sys(f) - p.seq) < 0) {  // reached (wrap-safe)
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *done = 0;
}

// GATHERED: the slots [par][*] of this rank's region were already filled by an
// NCCL all-gather (NCCL transport), so step 1 (peer stores + flags) is skipped
// and the [world][E] count matrix is also mirrored to the host (host_counts),
// which sizes the grouped ncclSend/ncclRecv of the row all-to-alls.
template <bool GATHERED>
__global__ void __launch_bounds__(256) ep_meta_kernel(const __grid_constant__ DispParams p,
                                                      const int32_t *__restrict__ counts,
                                                      const double *__restrict__ score_sum, int32_t *dev_meta_i,
                                                      double *dev_meta_d, int32_t *host_meta_i, double *host_meta_d,
                                                      uint32_t *host_flag, uint32_t host_seq,
                                                      int32_t *host_counts) {
  __shared__ int32_t s_cnt[kEpMaxWorld][kDispMaxE];
  __shared__ double s_sum[kEpMaxWorld][256];
  __shared__ int32_t s_gc[kDispMaxE], s_rb[kDispMaxE];
  __shared__ double s_gs[256];
  __shared__ double s_tot;
  const int par = static_cast<int>(p.seq & 1u), E = p.E, N = p.N, G = p.world;
  // 1. my counts and score sums into every rank's slot [par][me]
  if (!GATHERED) {
  for (int r = 0; r < G; ++r) {
    char *slot = p.region[r] + p.off_meta + (static_cast<size_t>(par) * G + p.rank) * p.meta_slot;
    for (int e = threadIdx.x; e < E; e += blockDim.x) reinterpret_cast<int32_t *>(slot)[e] = counts[e];
    double *d = reinterpret_cast<double *>(slot + (static_cast<size_t>(E) * 4 + 7) / 8 * 8);
    for (int e = threadIdx.x; e < N; e += blockDim.x) d[e] = score_sum[e];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < G)
    st_release_sys(reinterpret_cast<uint32_t *>(p.region[threadIdx.x] + p.off_mflags) + par * G + p.rank, p.seq);
  if (threadIdx.x < G) {
    const uint32_t *f = reinterpret_cast<const uint32_t *>(p.region[p.rank] + p.off_mflags) + par * G + threadIdx.x;
    while (static_cast<int32_t>(ld_acquire_sys(f) - p.seq) < 0) {  // reached (wrap-safe)
    }
  }
  }
  __syncthreads();
  // 2. gather every rank's slot from my own region
  for (int s = 0; s < G; ++s) {
    const char *slot = p.region[p.rank] + p.off_meta + (static_cast<size_t>(par) * G + s) * p.meta_slot;
    for (int e = threadIdx.x; e < E; e += blockDim.x) s_cnt[s][e] = __ldcv(reinterpret_cast<const int32_t *>(slot) + e);
    const double *d = reinterpret_cast<const double *>(slot + (static_cast<size_t>(E) * 4 + 7) / 8 * 8);
    for (int e = threadIdx.x; e < N; e += blockDim.x) s_sum[s][e] = __ldcv(d + e);
  }
  __syncthreads();
  // 3. global counts / score sums (rank order), tables
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int32_t c = 0, run = 0;
    for (int s = 0; s < G; ++s) {
      p.src_base[s * E + e] = run;
      run += s_cnt[s][e];
      p.counts_all[s * E + e] = s_cnt[s][e];
      if (GATHERED) host_counts[s * E + e] = s_cnt[s][e];
    }
    p.src_base[G * E + e] = run;
    c = run;
    s_gc[e] = c;
    p.gcount[e] = c;
  }
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    double acc = 0.0;
    for (int s = 0; s < G; ++s) acc += s_sum[s][e];
    s_gs[e] = acc;
  }
  if (threadIdx.x < G) {  // rank s's own permuted offsets (its local layout)
    const int s = threadIdx.x;
    int32_t run = 0;
    for (int e = 0; e < E; ++e) {
      p.local_off[s * (E + 1) + e] = run;
      run += s_cnt[s][e];
    }
    p.local_off[s * (E + 1) + E] = run;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // home layouts (per home rank, experts in index order) and the tot of scores
    int32_t run[kEpMaxWorld];
    for (int r = 0; r < G; ++r) run[r] = 0;
    for (int e = 0; e < E; ++e) {
      const int h = home_of(e, N, G);
      s_rb[e] = run[h];
      run[h] += s_gc[e];
    }
    double tot = 0.0;
    for (int e = 0; e < N; ++e) tot += s_gs[e];
    s_tot = tot;
    dev_meta_i[2 * E] = run[p.rank];   // total rows this rank receives
    host_meta_i[2 * E] = run[p.rank];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    p.recv_base[e] = s_rb[e];
    dev_meta_i[e] = s_gc[e];
    dev_meta_i[E + e] = s_rb[e];
    host_meta_i[e] = s_gc[e];
    host_meta_i[E + e] = s_rb[e];
  }
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    const double tot = s_tot;
    const double sc = tot > 0.0 ? s_gs[e] / tot : 0.0;
    dev_meta_d[e] = s_gs[e];
    dev_meta_d[N + e] = sc;
    host_meta_d[e] = s_gs[e];
    host_meta_d[N + e] = sc;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) *reinterpret_cast<volatile uint32_t *>(host_flag) = host_seq;
  // off the host's critical path: where each received row goes back to
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    if (home_of(e, N, G) != p.rank) continue;
    for (int s = 0; s < G; ++s) {
      const int base = s_rb[e] + p.src_base[s * E + e], n = s_cnt[s][e], lo = p.local_off[s * (E + 1) + e];
      for (int i = 0; i < n; ++i) p.ret_map[base + i] = (s << 24) | (lo + i);
    }
  }
}

// NCCL transport: this rank's counts and score sums into its own slot [par][rank]
// (the in-place send buffer of the all-gather)
__global__ void ep_pack_meta_kernel(const __grid_constant__ DispParams p, const int32_t *__restrict__ counts,
                                    const double *__restrict__ score_sum) {
  const int par = static_cast<int>(p.seq & 1u);
  char *slot = p.region[p.rank] + p.off_meta + (static_cast<size_t>(par) * p.world + p.rank) * p.meta_slot;
  for (int e = threadIdx.x; e < p.E; e += blockDim.x) reinterpret_cast<int32_t *>(slot)[e] = counts[e];
  double *d = reinterpret_cast<double *>(slot + (static_cast<size_t>(p.E) * 4 + 7) / 8 * 8);
  for (int e = threadIdx.x; e < p.N; e += blockDim.x) d[e] = score_sum[e];
}

// one block per 256 (row, 16-byte column) items of the local permuted rows
__global__ void __launch_bounds__(256) ep_dispatch_kernel(const __grid_constant__ DispParams p,
                                                          const uint16_t *__restrict__ xp,
                                                          const int32_t *__restrict__ sel,
                                                          const int32_t *__restrict__ row_src, int rows) {
  const int H8 = p.H / 8;
  const long v = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v < static_cast<long>(rows) * H8) {
    const int q = static_cast<int>(v / H8), c = static_cast<int>(v - static_cast<long>(q) * H8);
    const int e = sel[row_src[q]];
    const int h = home_of(e, p.N, p.world);
    const int dst = p.recv_base[e] + p.src_base[p.rank * p.E + e] + (q - p.local_off[p.rank * (p.E + 1) + e]);
    uint4 *d = reinterpret_cast<uint4 *>(p.region[h] + p.off_xrecv) + static_cast<size_t>(dst) * H8 + c;
    *d = reinterpret_cast<const uint4 *>(xp)[static_cast<size_t>(q) * H8 + c];
  }
  all_to_all_handshake(p, p.off_dflags, p.done);
}

// one block per received row: expert output row -> its source rank's position
__global__ void __launch_bounds__(256) ep_return_kernel(const __grid_constant__ DispParams p,
                                                        const float *__restrict__ out, int rows) {
  const int q = blockIdx.x;
  if (q < rows) {
    const int m = p.ret_map[q], src = m >> 24, dst = m & 0xffffff;
    float4 *d = reinterpret_cast<float4 *>(p.region[src] + p.off_ret) + static_cast<size_t>(dst) * (p.H / 4);
    const float4 *row = reinterpret_cast<const float4 *>(out) + static_cast<size_t>(q) * (p.H / 4);
    for (int c = threadIdx.x; c < p.H / 4; c += blockDim.x) d[c] = row[c];
  }
  all_to_all_handshake(p, p.off_rflags, p.done + 1);
}

}  // namespace

// ---------------------------------------------------------------- NCCL transport
// The token-sharded all-to-alls over NCCL (grouped ncclSend /
// ncclRecv), the baseline and the fallback of the peer-memory kernels when
// CUDA IPC between the ranks is unavailable.  libnccl is loaded at run time
// (the copy torch already mapped into the process when there is one), so the
// library has no link-time NCCL dependency.
struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char *(*error_string)(ncclResult_t) = nullptr;
};

const Nccl &nccl() {
  static Nccl n;
  static std::string err;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char *name) {
      void *f = dlsym(h, name);
      if (!f && err.empty()) err = std::string("libnccl lacks ") + name;
      return f;
    };
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym("ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(sym("ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(sym("ncclCommDestroy"));
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(sym("ncclAllGather"));
    n.send = reinterpret_cast<decltype(n.send)>(sym("ncclSend"));
    n.recv = reinterpret_cast<decltype(n.recv)>(sym("ncclRecv"));
    n.group_start = reinterpret_cast<decltype(n.group_start)>(sym("ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(n.group_end)>(sym("ncclGroupEnd"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
  });
  if (!err.empty()) raise(HM_ECUDA, err);
  return n;
}

#define HM_NCCL(call)                                                                                  \
  do {                                                                                                 \
    const ncclResult_t r_ = (call);                                                                    \
    if (r_ != ncclSuccess) hm::raise(HM_ECUDA, std::string("NCCL: ") + hm::nccl().error_string(r_) + \
                                                   " (" #call ")");                                  \
  } while (0)

// The all-to-all(v) schedule of one layer from the all-gathered [world][E]
// count matrix -- the same layout the peer-memory kernels write (home layout:
// experts in index order, inside an expert rows by source rank then source
// order; a source's own rows stay in its expert-contiguous permuted order).
// Between any two ranks the sends and the receives are both issued in expert
// index order, so NCCL's in-order pairing of p2p operations matches them.
void a2a_plan(const int32_t *cnt, int world, int E, int N, int rank, int direction, std::vector<hm_a2a_op> &ops) {
  ops.clear();
  const size_t SE = static_cast<size_t>(E);
  std::vector<int64_t> loff(world * SE), sbase(world * SE), rbase(E);
  std::vector<int64_t> run_home(world, 0);
  auto home = [&](int e) { return (e < N ? e : e - N) % world; };
  auto c = [&](int s, int e) { return static_cast<int64_t>(cnt[s * SE + e]); };
  for (int s = 0; s < world; ++s) {
    int64_t run = 0;
    for (int e = 0; e < E; ++e) {
      loff[s * SE + e] = run;
      run += c(s, e);
    }
  }
  for (int e = 0; e < E; ++e) {
    int64_t run = 0;
    for (int s = 0; s < world; ++s) {
      sbase[s * SE + e] = run;
      run += c(s, e);
    }
    rbase[e] = run_home[home(e)];
    run_home[home(e)] += run;
  }
  if (direction == 0) {  // dispatch: local permuted rows -> home layouts
    for (int e = 0; e < E; ++e) {
      const int64_t n = c(rank, e), h = home(e);
      if (n) ops.push_back(hm_a2a_op{h == rank ? HM_A2A_COPY : HM_A2A_SEND, static_cast<int32_t>(h),
                                     loff[rank * SE + e], rbase[e] + sbase[rank * SE + e], n});
    }
    for (int e = 0; e < E; ++e)
      if (home(e) == rank)
        for (int s = 0; s < world; ++s)
          if (s != rank && c(s, e))
            ops.push_back(hm_a2a_op{HM_A2A_RECV, s, loff[s * SE + e], rbase[e] + sbase[s * SE + e], c(s, e)});
  } else {  // return: home-layout output rows -> their sources' permuted positions
    for (int e = 0; e < E; ++e)
      if (home(e) == rank)
        for (int s = 0; s < world; ++s)
          if (c(s, e))
            ops.push_back(hm_a2a_op{s == rank ? HM_A2A_COPY : HM_A2A_SEND, s, rbase[e] + sbase[s * SE + e],
                                    loff[s * SE + e], c(s, e)});
    for (int e = 0; e < E; ++e) {
      const int h = home(e);
      if (h != rank && c(rank, e))
        ops.push_back(hm_a2a_op{HM_A2A_RECV, h, rbase[e] + sbase[rank * SE + e], loff[rank * SE + e], c(rank, e)});
    }
  }
}

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
  // dispatch mode (hm_ep_enable_dispatch)
  bool disp = false;
  int E = 0, N = 0, Kp = 0;
  char *region = nullptr;  // local IPC region
  char *peer_region[kEpMaxWorld] = {};
  bool region_opened[kEpMaxWorld] = {};
  size_t off_meta = 0, off_mflags = 0, off_dflags = 0, off_rflags = 0, off_xrecv = 0, off_ret = 0, meta_slot = 0,
         region_bytes = 0;
  int32_t *tables = nullptr;  // counts_all | recv_base | src_base | local_off | gcount | ret_map | done
  uint32_t dseq = 0;
  // NCCL transport (hm_ep_create_nccl): no IPC, the region is private
  bool use_nccl = false;
  ncclComm_t comm = nullptr;
  int32_t *h_counts = nullptr;   // mapped pinned [world][E]: the all-gathered count matrix
  int32_t *dv_counts = nullptr;  // its device alias
  std::vector<hm_a2a_op> plan;

  // The rows of `plan` through grouped ncclSend/ncclRecv (local rows by a D2D
  // copy); src/dst are the row bases, row_bytes the bytes of one row.
  void run_plan(const char *src, char *dst, size_t row_bytes, cudaStream_t st) {
    const Nccl &n = nccl();
    for (const hm_a2a_op &o : plan)
      if (o.kind == HM_A2A_COPY)
        HM_CUDA(cudaMemcpyAsync(dst + o.dst_row * row_bytes, src + o.src_row * row_bytes, o.rows * row_bytes,
                                cudaMemcpyDeviceToDevice, st));
    HM_NCCL(n.group_start());
    for (const hm_a2a_op &o : plan) {
      if (o.kind == HM_A2A_SEND)
        HM_NCCL(n.send(src + o.src_row * row_bytes, o.rows * row_bytes, ncclUint8, o.peer, comm, st));
      else if (o.kind == HM_A2A_RECV)
        HM_NCCL(n.recv(dst + o.dst_row * row_bytes, o.rows * row_bytes, ncclUint8, o.peer, comm, st));
    }
    HM_NCCL(n.group_end());
  }

  static size_t align256(size_t v) { return (v + 255) / 256 * 256; }

  void enable_dispatch(int e_total, int n_routed, int kp) {
    HM_REQUIRE(!disp, HM_EVALUE, "dispatch mode already enabled");
    HM_REQUIRE(e_total >= 1 && e_total <= kDispMaxE && n_routed >= 1 && n_routed <= 256 && n_routed <= e_total &&
                   kp >= 1 && H % 8 == 0,
               HM_EVALUE, "dispatch mode shape out of range");
    E = e_total;
    N = n_routed;
    Kp = kp;
    meta_slot = align256((static_cast<size_t>(E) * 4 + 7) / 8 * 8 + static_cast<size_t>(N) * 8);
    size_t o = 0;
    off_meta = o;
    o += align256(2ull * world * meta_slot);
    off_mflags = o;
    o += align256(2ull * world * 4);
    off_dflags = o;
    o += align256(world * 4ull);
    off_rflags = o;
    o += align256(world * 4ull);
    off_xrecv = o;
    o += align256(static_cast<size_t>(max_rows) * Kp * H * 2);
    off_ret = o;
    o += align256(static_cast<size_t>(max_rows) * Kp * H * 4);
    region_bytes = o;
    HM_CUDA(cudaMalloc(&region, region_bytes));
    HM_CUDA(cudaMemset(region, 0, off_xrecv));  // metadata and flags
    peer_region[rank] = region;
    region_opened[rank] = true;
    if (use_nccl)
      for (int q = 0; q < world; ++q) region_opened[q] = true;  // no peer mappings: NCCL moves the rows
    const size_t nt = static_cast<size_t>(world) * E + E + (world + 1ull) * E + world * (E + 1ull) + E +
                      static_cast<size_t>(max_rows) * Kp + 2;
    HM_CUDA(cudaMalloc(&tables, nt * 4));
    HM_CUDA(cudaMemset(tables, 0, nt * 4));
    HM_CUDA(cudaDeviceSynchronize());
    disp = true;
  }

  DispParams params() const {
    DispParams p{};
    p.off_meta = off_meta;
    p.off_mflags = off_mflags;
    p.off_dflags = off_dflags;
    p.off_rflags = off_rflags;
    p.off_xrecv = off_xrecv;
    p.off_ret = off_ret;
    p.meta_slot = meta_slot;
    for (int r = 0; r < world; ++r) p.region[r] = peer_region[r];
    p.rank = rank;
    p.world = world;
    p.E = E;
    p.N = N;
    p.H = H;
    p.Kp = Kp;
    p.seq = dseq;
    int32_t *t = tables;
    p.counts_all = t;
    t += static_cast<size_t>(world) * E;
    p.recv_base = t;
    t += E;
    p.src_base = t;
    t += (world + 1ull) * E;
    p.local_off = t;
    t += world * (E + 1ull);
    p.gcount = t;
    t += E;
    p.ret_map = t;
    t += static_cast<size_t>(max_rows) * Kp;
    p.done = t;
    return p;
  }

  EpExchange(int r, int w, int rows, int h, const ncclUniqueId *nccl_id = nullptr)
      : rank(r), world(w), max_rows(rows), H(h) {
    HM_REQUIRE(w >= 1 && w <= kEpMaxWorld && r >= 0 && r < w, HM_EVALUE, "expert-parallel world must be 1..8");
    HM_REQUIRE(rows >= 1 && h % 4 == 0, HM_EVALUE, "bad exchange shape");
    if (nccl_id) {  // NCCL transport: a communicator instead of IPC inboxes
      use_nccl = true;
      HM_NCCL(nccl().comm_init_rank(&comm, world, *nccl_id, rank));
      HM_CUDA(cudaHostAlloc(&h_counts, static_cast<size_t>(world) * kDispMaxE * 4, cudaHostAllocMapped));
      HM_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void **>(&dv_counts), h_counts, 0));
      for (int q = 0; q < world; ++q) opened[q] = true;
      return;
    }
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
    for (int r = 0; r < world; ++r)
      if (r != rank && region_opened[r]) cudaIpcCloseMemHandle(peer_region[r]);
    if (inbox) cudaFree(inbox);
    if (flags) cudaFree(flags);
    if (region) cudaFree(region);
    if (tables) cudaFree(tables);
    if (h_counts) cudaFreeHost(h_counts);
    if (comm) nccl().comm_destroy(comm);
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

int hm_ep_enable_dispatch(hm_ep *ep, int n_experts_total, int n_routed, int Kp, void *region_handle) {
  HM_API_BEGIN
  auto *e = reinterpret_cast<hm::EpExchange *>(ep);
  HM_REQUIRE(region_handle, HM_EVALUE, "null handle buffer");
  HM_REQUIRE(!e->use_nccl, HM_EVALUE, "the NCCL transport enables dispatch at creation (hm_ep_create_nccl)");
  e->enable_dispatch(n_experts_total, n_routed, Kp);
  HM_CUDA(cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t *>(region_handle), e->region));
  HM_API_END
}

int hm_ep_open_peer_dispatch(hm_ep *ep, int peer, const void *region_handle) {
  HM_API_BEGIN
  auto *e = reinterpret_cast<hm::EpExchange *>(ep);
  HM_REQUIRE(e->disp && peer >= 0 && peer < e->world, HM_EVALUE, "dispatch mode not enabled or bad peer");
  if (peer == e->rank || e->region_opened[peer]) return HM_OK;
  cudaIpcMemHandle_t h;
  memcpy(&h, region_handle, sizeof h);
  void *ptr = nullptr;
  HM_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
  e->peer_region[peer] = static_cast<char *>(ptr);
  e->region_opened[peer] = true;
  HM_API_END
}

int hm_ep_dispatch_meta(hm_ep *ep, const int32_t *counts, const double *score_sum, int32_t *dev_meta_i,
                        double *dev_meta_d, int32_t *host_meta_i, double *host_meta_d, uint32_t *host_flag,
                        uint32_t host_seq, void *stream) {
  HM_API_BEGIN
  auto *e = reinterpret_cast<hm::EpExchange *>(ep);
  HM_REQUIRE(e->disp, HM_EVALUE, "dispatch mode not enabled");
  for (int r = 0; r < e->world; ++r) HM_REQUIRE(e->region_opened[r], HM_EVALUE, "dispatch peers not opened");
  ++e->dseq;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const hm::DispParams p = e->params();
  if (e->use_nccl) {  // pack my slot, in-place ncclAllGather of the slots, then the tables
    hm::ep_pack_meta_kernel<<<1, 256, 0, st>>>(p, counts, score_sum);
    HM_LAUNCH_CHECK();
    char *slots = e->region + e->off_meta + static_cast<size_t>(e->dseq & 1u) * e->world * e->meta_slot;
    HM_NCCL(hm::nccl().all_gather(slots + static_cast<size_t>(e->rank) * e->meta_slot, slots, e->meta_slot,
                                  ncclUint8, e->comm, st));
    hm::ep_meta_kernel<true><<<1, 256, 0, st>>>(p, counts, score_sum, dev_meta_i, dev_meta_d, host_meta_i,
                                                host_meta_d, host_flag, host_seq, e->dv_counts);
  } else {
    hm::ep_meta_kernel<false><<<1, 256, 0, st>>>(p, counts, score_sum, dev_meta_i, dev_meta_d, host_meta_i,
                                                 host_meta_d, host_flag, host_seq, nullptr);
  }
  HM_LAUNCH_CHECK();
  HM_API_END
}

int hm_ep_dispatch_rows(hm_ep *ep, const uint16_t *xp, const int32_t *sel, const int32_t *row_src, int rows,
                        void *stream) {
  HM_API_BEGIN
  auto *e = reinterpret_cast<hm::EpExchange *>(ep);
  HM_REQUIRE(e->disp && rows >= 0 && rows <= e->max_rows * e->Kp, HM_EVALUE, "bad dispatch");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (e->use_nccl) {  // the host holds the count matrix (after the meta flag): grouped send/recv
    hm::a2a_plan(e->h_counts, e->world, e->E, e->N, e->rank, 0, e->plan);
    int64_t recv = 0;
    for (const hm_a2a_op &o : e->plan)
      if (o.kind != HM_A2A_SEND) recv = std::max(recv, o.dst_row + o.rows);
    HM_REQUIRE(recv <= static_cast<int64_t>(e->max_rows) * e->Kp, HM_EVALUE, "received rows exceed the buffer");
    e->run_plan(reinterpret_cast<const char *>(xp), e->region + e->off_xrecv, static_cast<size_t>(e->H) * 2, st);
    return HM_OK;
  }
  const long items = static_cast<long>(rows) * (e->H / 8);
  const int grid = static_cast<int>(std::max<long>(1, (items + 255) / 256));
  hm::ep_dispatch_kernel<<<grid, 256, 0, st>>>(e->params(), xp, sel, row_src, rows);
  HM_LAUNCH_CHECK();
  HM_API_END
}

int hm_ep_return_rows(hm_ep *ep, const float *out, int rows, void *stream) {
  HM_API_BEGIN
  auto *e = reinterpret_cast<hm::EpExchange *>(ep);
  HM_REQUIRE(e->disp && rows >= 0 && rows <= e->max_rows * e->Kp, HM_EVALUE, "bad return");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (e->use_nccl) {
    hm::a2a_plan(e->h_counts, e->world, e->E, e->N, e->rank, 1, e->plan);
    e->run_plan(reinterpret_cast<const char *>(out), e->region + e->off_ret, static_cast<size_t>(e->H) * 4, st);
    return HM_OK;
  }
  hm::ep_return_kernel<<<std::max(1, rows), 256, 0, st>>>(e->params(), out, rows);
  HM_LAUNCH_CHECK();
  HM_API_END
}

int hm_ep_nccl_unique_id(void *id) {
  HM_API_BEGIN
  HM_REQUIRE(id, HM_EVALUE, "null id buffer");
  HM_NCCL(hm::nccl().get_unique_id(static_cast<ncclUniqueId *>(id)));
  HM_API_END
}

int hm_ep_create_nccl(int rank, int world, int max_rows, int H, const void *id, int n_experts_total, int n_routed,
                      int Kp, hm_ep **out) {
  HM_API_BEGIN
  HM_REQUIRE(out && id, HM_EVALUE, "null argument");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  auto *e = new hm::EpExchange(rank, world, max_rows, H, &uid);
  try {
    e->enable_dispatch(n_experts_total, n_routed, Kp);
  } catch (...) {
    delete e;
    throw;
  }
  *out = reinterpret_cast<hm_ep *>(e);
  HM_API_END
}

int hm_ep_uses_nccl(const hm_ep *ep) { return reinterpret_cast<const hm::EpExchange *>(ep)->use_nccl ? 1 : 0; }

int hm_ep_world(const hm_ep *ep) { return reinterpret_cast<const hm::EpExchange *>(ep)->world; }

int hm_ep_a2a_plan(const int32_t *counts_all, int world, int n_experts_total, int n_routed, int rank, int direction,
                   hm_a2a_op *ops, int max_ops, int *n_ops) {
  HM_API_BEGIN
  HM_REQUIRE(counts_all && n_ops && world >= 1 && rank >= 0 && rank < world && n_routed >= 1 &&
                 n_routed <= n_experts_total && (direction == 0 || direction == 1),
             HM_EVALUE, "bad all-to-all plan arguments");
  for (int i = 0; i < world * n_experts_total; ++i) HM_REQUIRE(counts_all[i] >= 0, HM_EVALUE, "negative count");
  std::vector<hm_a2a_op> v;
  hm::a2a_plan(counts_all, world, n_experts_total, n_routed, rank, direction, v);
  *n_ops = static_cast<int>(v.size());
  HM_REQUIRE(!ops || static_cast<int>(v.size()) <= max_ops, HM_EVALUE, "plan exceeds max_ops");
  if (ops) std::copy(v.begin(), v.end(), ops);
  HM_API_END
}

int hm_ep_dispatch_buffers(hm_ep *ep, uint16_t **xrecv, float **ret) {
  HM_API_BEGIN
  auto *e = reinterpret_cast<hm::EpExchange *>(ep);
  HM_REQUIRE(e->disp, HM_EVALUE, "dispatch mode not enabled");
  if (xrecv) *xrecv = reinterpret_cast<uint16_t *>(e->region + e->off_xrecv);
  if (ret) *ret = reinterpret_cast<float *>(e->region + e->off_ret);
  HM_API_END
}

}  // extern "C"
