// Router, token permutation, combine and the GPU MRS update (sm_100a).
//
// Router semantics (Eq. 1; transformers mixtral / deepseek_v2 /
// qwen2_moe routers): softmax over the N routed logits in fp32, top-K by
// (logit desc, expert index asc) -- the reference's documented tie rule
// (core.py:94-97, tracegen.py:139-141) -- combine weight = softmax probability,
// optionally renormalised over the selected K (Mixtral).  Shared experts are
// appended as always-selected columns N..N+S-1 with weight 1 or, for the
// Qwen2 shared expert, sigmoid of a gate logit.  Per-expert loads are the
// bincount of the selection (tracegen.py:148); score sums are the fp64
// token-sum of the routed softmax (tracegen.py:149) reduced in a fixed order.
#include <cfloat>

#include "device.cuh"

namespace hm {
namespace {

constexpr int kMaxPerLane = 8;  // N <= 256 routed experts

__global__ void router_topk_kernel(const float *__restrict__ logits, int T, int N, int ld, int K, int renorm,
                                   int n_shared, int shared_gate_col, int32_t *__restrict__ sel,
                                   float *__restrict__ w, float *__restrict__ probs, int32_t *__restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (blockIdx.x == 0 && threadIdx.x < n_shared) counts[N + threadIdx.x] = T;
  if (t >= T) return;
  const float *row = logits + static_cast<size_t>(t) * ld;
  float v[kMaxPerLane];
  float m = -FLT_MAX;
#pragma unroll
  for (int j = 0; j < kMaxPerLane; ++j) {
    int e = lane + 32 * j;
    v[j] = e < N ? row[e] : -FLT_MAX;
    m = fmaxf(m, v[j]);
  }
  m = dev::warp_max(m);
  float ex[kMaxPerLane];
  float s = 0.0f;
#pragma unroll
  for (int j = 0; j < kMaxPerLane; ++j) {
    int e = lane + 32 * j;
    ex[j] = e < N ? expf(v[j] - m) : 0.0f;
    s += ex[j];
  }
  s = dev::warp_sum(s);
  const float inv = 1.0f / s;
#pragma unroll
  for (int j = 0; j < kMaxPerLane; ++j) {
    int e = lane + 32 * j;
    if (e < N) probs[static_cast<size_t>(t) * N + e] = ex[j] * inv;
  }
  // top-K: repeated warp arg-max with (value desc, index asc)
  const int Kp = K + n_shared;
  uint32_t taken = 0;
  float psel[8];
  float psum = 0.0f;
  for (int k = 0; k < K; ++k) {
    float bv = -FLT_MAX;
    int bi = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < kMaxPerLane; ++j) {
      int e = lane + 32 * j;
      if (e < N && !((taken >> j) & 1u) && (v[j] > bv || (v[j] == bv && e < bi))) {
        bv = v[j];
        bi = e;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (bi >= N) {  // non-finite logits (NaN compares false): take the lowest free index, never write out of range
      bi = 0;
      while (bi < N && __shfl_sync(0xffffffffu, ((taken >> (bi >> 5)) & 1u), bi & 31)) ++bi;
      bv = m;
    }
    if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
    float p = expf(bv - m) * inv;
    psel[k] = p;
    psum += p;
    if (lane == 0) {
      sel[static_cast<size_t>(t) * Kp + k] = bi;
      atomicAdd(&counts[bi], 1);
    }
  }
  if (lane == 0) {
    for (int k = 0; k < K; ++k) w[static_cast<size_t>(t) * Kp + k] = renorm ? psel[k] / psum : psel[k];
    float g = 1.0f;
    if (shared_gate_col >= 0) g = 1.0f / (1.0f + expf(-row[shared_gate_col]));
    for (int s2 = 0; s2 < n_shared; ++s2) {
      sel[static_cast<size_t>(t) * Kp + K + s2] = N + s2;
      w[static_cast<size_t>(t) * Kp + K + s2] = g;
    }
  }
}

// Decode-sized layers (T*(K+S) <= 1024, N <= 256, E <= 320) in ONE block:
// router (same math as router_topk_kernel), counts, fp64 score sums and the
// normalised LayerRequest scores (sequential sums, bit-identical to the host
// core's arithmetic), expert offsets, the permutation and the row gather.
// meta = [counts E | offsets E+1] int32 followed (8-byte aligned) by
// [score_sum N | scores N] fp64, so one D2H copy carries the LayerRequest.
// Optional mirror of the fused router's results in mapped pinned host memory
// (device pointers of cudaHostAlloc'd buffers): the LayerRequest block, the
// routed rows of xp for the host worker, and a completion flag the host spins
// on -- no D2H copy and no event round trip on the per-layer critical path.
struct HostMirror {
  int32_t *meta_i;
  double *meta_d;
  uint16_t *xp;
  uint32_t *flag;
  uint32_t seq;
  // optional MRS update of this layer's row (caching.py:65-76) on the GPU:
  // S = the decision core's [L, N] table (mapped host memory, read only), the
  // new row goes to mrs_row (mapped) for the decision core's step (5)
  double *S = nullptr;
  double *mrs_row = nullptr;
  int layer = 0, p = 0;
  double alpha = 0.0;
};

constexpr int kFusedMaxRows = 1024;
constexpr int kFusedMaxE = 320;

// PL = experts per lane, ceil(N / 32) rounded up to a power of two: the top-K
// scans touch only the lanes' live values (same selection as PL = 8)
template <int PL>
__global__ void __launch_bounds__(256) router_fused_small_kernel(
    const float *__restrict__ logits, int T, int N, int ld, int K, int renorm, int n_shared, int shared_gate_col,
    const uint16_t *__restrict__ x, int H, int32_t *__restrict__ sel, float *__restrict__ w, int32_t *__restrict__ pos,
    int32_t *__restrict__ row_src, uint16_t *__restrict__ xp, int32_t *__restrict__ meta_i, double *__restrict__ meta_d,
    HostMirror hm_) {
  __shared__ int32_t s_sel[kFusedMaxRows];
  __shared__ int32_t s_counts[kFusedMaxE];
  __shared__ int32_t s_off[kFusedMaxE + 1];
  __shared__ int32_t s_rowtok[kFusedMaxRows];
  __shared__ float s_probs[32 * 256];  // T <= 32 tokens x N <= 256
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int E = N + n_shared, Kp = K + n_shared, R = T * Kp;
  // the old MRS row is read from the decision core's mapped table now; the
  // PCIe round trip overlaps with the routing below
  double mrs_old = 0.0;
  if (hm_.S && threadIdx.x < N) mrs_old = __ldcv(hm_.S + static_cast<size_t>(hm_.layer) * N + threadIdx.x);
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_counts[e] = 0;
  __syncthreads();
  for (int t = wid; t < T; t += nw) {
    const float *row = logits + static_cast<size_t>(t) * ld;
    float v[PL];
    float m = -FLT_MAX;
#pragma unroll
    for (int j = 0; j < PL; ++j) {
      const int e = lane + 32 * j;
      v[j] = e < N ? row[e] : -FLT_MAX;
      m = fmaxf(m, v[j]);
    }
    m = dev::warp_max(m);
    float s = 0.0f, ex[PL];
#pragma unroll
    for (int j = 0; j < PL; ++j) {
      const int e = lane + 32 * j;
      ex[j] = e < N ? expf(v[j] - m) : 0.0f;
      s += ex[j];
    }
    s = dev::warp_sum(s);
    const float inv = 1.0f / s;
#pragma unroll
    for (int j = 0; j < PL; ++j) {
      const int e = lane + 32 * j;
      if (e < N) s_probs[t * N + e] = ex[j] * inv;
    }
    uint32_t taken = 0;
    float psel[8], psum = 0.0f;
    for (int k = 0; k < K; ++k) {
      float bv = -FLT_MAX;
      int bi = 0x7fffffff;
#pragma unroll
      for (int j = 0; j < PL; ++j) {
        const int e = lane + 32 * j;
        if (e < N && !((taken >> j) & 1u) && (v[j] > bv || (v[j] == bv && e < bi))) {
          bv = v[j];
          bi = e;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (bi >= N) {  // non-finite logits: lowest free index (as router_topk_kernel)
        bi = 0;
        while (bi < N && __shfl_sync(0xffffffffu, ((taken >> (bi >> 5)) & 1u), bi & 31)) ++bi;
        bv = m;
      }
      if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
      const float p = expf(bv - m) * inv;
      psel[k] = p;
      psum += p;
      if (lane == 0) {
        s_sel[t * Kp + k] = bi;
        atomicAdd(&s_counts[bi], 1);
      }
    }
    if (lane == 0) {
      for (int k = 0; k < K; ++k) w[static_cast<size_t>(t) * Kp + k] = renorm ? psel[k] / psum : psel[k];
      const float g = shared_gate_col >= 0 ? 1.0f / (1.0f + expf(-row[shared_gate_col])) : 1.0f;
      for (int c = 0; c < n_shared; ++c) {
        s_sel[t * Kp + K + c] = N + c;
        w[static_cast<size_t>(t) * Kp + K + c] = g;
        atomicAdd(&s_counts[N + c], 1);
      }
    }
  }
  __syncthreads();
  // offsets: warp 0 scans the counts (each lane a contiguous run of experts);
  // fp64 score sums: thread e sums its column over tokens in token order;
  // everything stays in shared memory (a global store followed by a load of
  // the same word costs an L2 round trip per element when done serially).
  __shared__ double s_sum[256];
  __shared__ double s_tot;
  if (wid == 0) {
    const int per = (E + 31) / 32, e0 = min(E, lane * per), e1 = min(E, e0 + per);
    int32_t local = 0;
    for (int e = e0; e < e1; ++e) local += s_counts[e];
    int32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int32_t run = incl - local;
    for (int e = e0; e < e1; ++e) {
      s_off[e] = run;
      run += s_counts[e];
    }
    if (lane == 31) s_off[E] = incl;
  }
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    double acc = 0.0;
    for (int t = 0; t < T; ++t) acc += static_cast<double>(s_probs[t * N + e]);
    s_sum[e] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // the host core's order: tot = sum_e score_sum[e], e ascending
    double tot = 0.0;
    for (int e = 0; e < N; ++e) tot += s_sum[e];
    s_tot = tot;
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    meta_i[e] = s_counts[e];
    meta_i[E + e] = s_off[e];
  }
  if (threadIdx.x == 0) meta_i[2 * E] = s_off[E];
  __syncthreads();
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    const double tot = s_tot;
    meta_d[e] = s_sum[e];
    meta_d[N + e] = tot > 0.0 ? s_sum[e] / tot : 0.0;
  }
  __syncthreads();
  // The LayerRequest (and this layer's MRS row) go to mapped host memory and
  // the request flag is raised BEFORE the permutation and the row gather: the
  // host's decision core runs while the rows are gathered and mirrored; the
  // host worker waits for the rows flag (flag[2]) before it reads them.
  if (hm_.flag) {
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      hm_.meta_i[e] = s_counts[e];
      hm_.meta_i[E + e] = s_off[e];
    }
    if (threadIdx.x == 0) hm_.meta_i[2 * E] = s_off[E];
    __shared__ double s_nrm[256];  // normalised scores, each divided once
    for (int e = threadIdx.x; e < N; e += blockDim.x) {
      const double tot = s_tot;
      const double v = tot > 0.0 ? s_sum[e] / tot : 0.0;
      s_nrm[e] = v;
      hm_.meta_d[e] = s_sum[e];
      hm_.meta_d[N + e] = v;
    }
    __syncthreads();
    if (hm_.S && threadIdx.x < N) {  // this layer's new MRS row, a * TopP(s) + (1 - a) * S (caching.py:65-76)
      const int i = threadIdx.x;
      const double si = s_nrm[i];
      int rank = 0;
      for (int j = 0; j < N; ++j) {
        const double sj = s_nrm[j];
        rank += (sj > si || (sj == si && j < i)) ? 1 : 0;
      }
      const double t = rank < hm_.p ? si : 0.0;
      hm_.mrs_row[i] = __dadd_rn(__dmul_rn(hm_.alpha, t), __dmul_rn(__dsub_rn(1.0, hm_.alpha), mrs_old));
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) *reinterpret_cast<volatile uint32_t *>(hm_.flag) = hm_.seq;
  }

  for (int j = threadIdx.x; j < R; j += blockDim.x) {  // stable rank inside the expert
    const int e = s_sel[j];
    int r = 0;
    for (int q = 0; q < j; ++q) r += s_sel[q] == e;
    const int p = s_off[e] + r;
    sel[j] = e;
    pos[j] = p;
    row_src[p] = j;
    s_rowtok[p] = j / Kp;  // token of the row at position p (shared: no global round trip)
  }
  __syncthreads();
  const int H8 = H / 8;
  // routed rows also go to the host worker's input; one token (decode): every
  // routed row is that token, so one copy crosses PCIe (the host reads row 0)
  const int n_host = hm_.xp ? (T == 1 ? min(1, s_off[N]) : s_off[N]) : 0;
#pragma unroll 4
  for (int v = threadIdx.x; v < R * H8; v += blockDim.x) {  // gather rows in permuted order
    const int p = v / H8, c = v - p * H8;
    const uint4 v4 = __ldg(reinterpret_cast<const uint4 *>(x + static_cast<size_t>(s_rowtok[p]) * H) + c);
    reinterpret_cast<uint4 *>(xp + static_cast<size_t>(p) * H)[c] = v4;
    if (p < n_host) reinterpret_cast<uint4 *>(hm_.xp + static_cast<size_t>(p) * H)[c] = v4;
  }
  if (hm_.flag && hm_.xp) {  // the host worker's rows have landed
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) reinterpret_cast<volatile uint32_t *>(hm_.flag)[2] = hm_.seq;
  }
}

void launch_router_fused(const float *logits, int T, int N, int ld, int K, int renorm, int n_shared,
                         int shared_gate_col, const uint16_t *x, int H, int32_t *sel, float *w, int32_t *pos,
                         int32_t *row_src, uint16_t *xp, int32_t *meta_i, double *meta_d, HostMirror m,
                         cudaStream_t st) {
#define HM_ROUTER_FUSED(PLV)                                                                                     \
  router_fused_small_kernel<PLV><<<1, 256, 0, st>>>(logits, T, N, ld, K, renorm, n_shared, shared_gate_col, x, H, \
                                                    sel, w, pos, row_src, xp, meta_i, meta_d, m)
  if (N <= 32)
    HM_ROUTER_FUSED(1);
  else if (N <= 64)
    HM_ROUTER_FUSED(2);
  else if (N <= 128)
    HM_ROUTER_FUSED(4);
  else
    HM_ROUTER_FUSED(8);
#undef HM_ROUTER_FUSED
}

// score_sum[e] = sum_t probs[t, e] in fp64, fixed reduction order.
__global__ void score_sum_kernel(const float *__restrict__ probs, int T, int N, double *__restrict__ out) {
  __shared__ double red[256];
  const int e = blockIdx.x;
  double acc = 0.0;
  for (int t = threadIdx.x; t < T; t += blockDim.x) acc += static_cast<double>(probs[static_cast<size_t>(t) * N + e]);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[e] = red[0];
}

// logits[t, n] = x[t, :] . wg[n, :]  (bf16 in, fp32 accumulate); one warp per (t, n).
__global__ void router_logits_kernel(const uint16_t *__restrict__ x, const uint16_t *__restrict__ wg, int T, int H,
                                     int N, float *__restrict__ logits) {
  const int lane = threadIdx.x & 31;
  const long item = static_cast<long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (item >= static_cast<long>(T) * N) return;
  const int t = static_cast<int>(item / N), n = static_cast<int>(item % N);
  const uint16_t *xr = x + static_cast<size_t>(t) * H;
  const uint16_t *wr = wg + static_cast<size_t>(n) * H;
  float acc = 0.0f;
  for (int c = lane * 8; c < H; c += 256) acc += dev::dot8(dev::ld_stream(wr + c), *reinterpret_cast<const uint4 *>(xr + c));
  acc = dev::warp_sum(acc);
  if (lane == 0) logits[item] = acc;
}

__global__ void offsets_kernel(const int32_t *__restrict__ counts, int E, int32_t *__restrict__ offsets) {
  if (threadIdx.x == 0) {
    int32_t run = 0;
    for (int e = 0; e < E; ++e) {
      offsets[e] = run;
      run += counts[e];
    }
    offsets[E] = run;
  }
}

// One block per expert: rows of expert e in (token, slot) order.
__global__ void permute_kernel(const int32_t *__restrict__ sel, int TK, const int32_t *__restrict__ offsets,
                               int32_t *__restrict__ pos, int32_t *__restrict__ row_src) {
  __shared__ int32_t warp_tot[32];
  __shared__ int32_t base;
  const int e = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) base = offsets[e];
  __syncthreads();
  for (int j0 = 0; j0 < TK; j0 += blockDim.x) {
    const int j = j0 + threadIdx.x;
    const bool hit = j < TK && sel[j] == e;
    const uint32_t ballot = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) warp_tot[wid] = __popc(ballot);
    __syncthreads();
    int before = 0;
    for (int w2 = 0; w2 < wid; ++w2) before += warp_tot[w2];
    if (hit) {
      const int p = base + before + __popc(ballot & ((1u << lane) - 1u));
      pos[j] = p;
      row_src[p] = j;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w2 = 0; w2 < nw; ++w2) tot += warp_tot[w2];
      base += tot;
    }
    __syncthreads();
  }
}

// xp[r, :] = x[row_src[r] / Kp, :]
__global__ void gather_kernel(const uint16_t *__restrict__ x, const int32_t *__restrict__ row_src, int rows, int Kp,
                              int H, uint16_t *__restrict__ xp) {
  const int r = blockIdx.x;
  if (r >= rows) return;
  const int t = row_src[r] / Kp;
  const uint4 *src = reinterpret_cast<const uint4 *>(x + static_cast<size_t>(t) * H);
  uint4 *dst = reinterpret_cast<uint4 *>(xp + static_cast<size_t>(r) * H);
  for (int c = threadIdx.x; c < H / 8; c += blockDim.x) dst[c] = src[c];
}

// Expert parallelism: drop selections whose expert lives on another rank.
__global__ void mask_nonhome_kernel(const int32_t *__restrict__ sel, float *__restrict__ w, int TKp, int N, int rank,
                                    int world) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= TKp) return;
  const int e = sel[j];
  const int owner = (e < N ? e : e - N) % world;
  if (owner != rank) w[j] = 0.0f;
}

// y32[t, :] = sum_k w[t, k] * out[pos[t, k], :]  (this rank's partial; zero weights skipped)
__global__ void combine_f32_kernel(const float *__restrict__ out, const int32_t *__restrict__ pos,
                                   const float *__restrict__ w, int Kp, int H, float *__restrict__ y32) {
  const int t = blockIdx.x;
  for (int c = threadIdx.x * 4; c < H; c += blockDim.x * 4) {
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < Kp; ++k) {
      const float wk = w[static_cast<size_t>(t) * Kp + k];
      if (wk == 0.0f) continue;
      const float4 o = *reinterpret_cast<const float4 *>(out + static_cast<size_t>(pos[static_cast<size_t>(t) * Kp + k]) * H + c);
      a.x = fmaf(wk, o.x, a.x);
      a.y = fmaf(wk, o.y, a.y);
      a.z = fmaf(wk, o.z, a.z);
      a.w = fmaf(wk, o.w, a.w);
    }
    *reinterpret_cast<float4 *>(y32 + static_cast<size_t>(t) * H + c) = a;
  }
}

// y = bf16(residual + y32)
__global__ void residual_add_kernel(const float *__restrict__ y32, const uint16_t *__restrict__ residual, int H,
                                    uint16_t *__restrict__ y) {
  const int t = blockIdx.x;
  for (int c = threadIdx.x * 4; c < H; c += blockDim.x * 4) {
    const float4 a = *reinterpret_cast<const float4 *>(y32 + static_cast<size_t>(t) * H + c);
    const uint2 rv = *reinterpret_cast<const uint2 *>(residual + static_cast<size_t>(t) * H + c);
    uint2 o2;
    o2.x = dev::pack_bf2(a.x + dev::bf_lo(rv.x), a.y + dev::bf_hi(rv.x));
    o2.y = dev::pack_bf2(a.z + dev::bf_lo(rv.y), a.w + dev::bf_hi(rv.y));
    *reinterpret_cast<uint2 *>(y + static_cast<size_t>(t) * H + c) = o2;
  }
}

// y[t, :] = residual[t, :] + sum_k w[t, k] * out[pos[t, k], :]   (k in order)
__global__ void combine_kernel(const float *__restrict__ out, const int32_t *__restrict__ pos,
                               const float *__restrict__ w, int Kp, int H, const uint16_t *__restrict__ residual,
                               uint16_t *__restrict__ y) {
  const int t = blockIdx.x;
  for (int c = threadIdx.x * 4; c < H; c += blockDim.x * 4) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    for (int k = 0; k < Kp; ++k) {
      const float wk = w[static_cast<size_t>(t) * Kp + k];
      if (wk == 0.0f) continue;  // masked (other rank's expert) or underflowed
      const float4 o = *reinterpret_cast<const float4 *>(out + static_cast<size_t>(pos[static_cast<size_t>(t) * Kp + k]) * H + c);
      a0 = fmaf(wk, o.x, a0);
      a1 = fmaf(wk, o.y, a1);
      a2 = fmaf(wk, o.z, a2);
      a3 = fmaf(wk, o.w, a3);
    }
    if (residual) {
      const uint2 rv = *reinterpret_cast<const uint2 *>(residual + static_cast<size_t>(t) * H + c);
      a0 += dev::bf_lo(rv.x);
      a1 += dev::bf_hi(rv.x);
      a2 += dev::bf_lo(rv.y);
      a3 += dev::bf_hi(rv.y);
    }
    uint2 o2;
    o2.x = dev::pack_bf2(a0, a1);
    o2.y = dev::pack_bf2(a2, a3);
    *reinterpret_cast<uint2 *>(y + static_cast<size_t>(t) * H + c) = o2;
  }
}

// Decode tail in one launch: blocks [0, T) combine (Eq. 1) + residual, rows
// whose bit is set in host_mask read straight from the host worker's mapped
// output buffer (zero-copy, no H2D); block T (if S) folds the layer's scores
// into the MRS table like mrs_update_kernel.
struct CombineTail {
  const float *out, *host_out;
  const int32_t *pos;
  const float *w;
  int Kp, H;
  const uint16_t *residual;
  uint16_t *y;
  unsigned long long host_mask[4];  // positions < 256
  double *S;
  const double *scores;
  int layer, N, p;
  double a;
  // pre-launched tail: wait until the host worker has published its rows
  // (*gate reaches gate_seq, mapped host memory) before reading them
  const uint32_t *gate;
  uint32_t gate_seq;
};

__device__ void mrs_row_update(double *__restrict__ S, const double *__restrict__ s, int layer, int N, int p,
                               double a);

// grid: T * cs column blocks (128 threads x 4 columns each) + 1 MRS block.
constexpr int kTailThreads = 128;
constexpr int kTailMaxKp = 64;

__global__ void __launch_bounds__(kTailThreads) combine_tail_kernel(const __grid_constant__ CombineTail c) {
  __shared__ float s_w[kTailMaxKp];
  __shared__ int32_t s_pos[kTailMaxKp];
  __shared__ double s_sc[256];
  const int cs = (c.H + 4 * kTailThreads - 1) / (4 * kTailThreads);
  const int b = blockIdx.x;
  if (c.S && b == static_cast<int>(gridDim.x) - 1) {  // MRS row (scores staged in smem)
    for (int i = threadIdx.x; i < c.N; i += blockDim.x) s_sc[i] = c.scores[i];
    __syncthreads();
    for (int i = threadIdx.x; i < c.N; i += blockDim.x) {
      const double si = s_sc[i];
      int rank = 0;
      for (int j = 0; j < c.N; ++j) {
        const double sj = s_sc[j];
        rank += (sj > si || (sj == si && j < i)) ? 1 : 0;
      }
      const double t = rank < c.p ? si : 0.0;
      double *row = c.S + static_cast<size_t>(c.layer) * c.N;
      row[i] = __dadd_rn(__dmul_rn(c.a, t), __dmul_rn(__dsub_rn(1.0, c.a), row[i]));
    }
    return;
  }
  const int t = b / cs, col = ((b % cs) * kTailThreads + threadIdx.x) * 4;
  for (int k = threadIdx.x; k < c.Kp; k += blockDim.x) {
    s_w[k] = c.w[static_cast<size_t>(t) * c.Kp + k];
    s_pos[k] = c.pos[static_cast<size_t>(t) * c.Kp + k];
  }
  if (c.gate && threadIdx.x == 0) {  // launched before the host worker ran: wait for its rows
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(c.gate) : "memory");
      if (static_cast<int32_t>(v - c.gate_seq) >= 0) break;
      __nanosleep(128);
    }
  }
  __syncthreads();
  if (col >= c.H) return;
  uint2 rv = make_uint2(0u, 0u);
  if (c.residual) rv = *reinterpret_cast<const uint2 *>(c.residual + static_cast<size_t>(t) * c.H + col);
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  constexpr int U = 8;  // issue U independent row loads before accumulating (k order kept)
  for (int k0 = 0; k0 < c.Kp; k0 += U) {
    float4 o[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u;
      o[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (k < c.Kp && s_w[k] != 0.0f) {
        const int pp = s_pos[k];
        const bool host = pp < 256 && ((c.host_mask[pp >> 6] >> (pp & 63)) & 1ull);
        o[u] = *reinterpret_cast<const float4 *>((host ? c.host_out : c.out) + static_cast<size_t>(pp) * c.H + col);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u;
      if (k < c.Kp && s_w[k] != 0.0f) {
        const float wk = s_w[k];
        a0 = fmaf(wk, o[u].x, a0);
        a1 = fmaf(wk, o[u].y, a1);
        a2 = fmaf(wk, o[u].z, a2);
        a3 = fmaf(wk, o[u].w, a3);
      }
    }
  }
  if (c.residual) {
    a0 += dev::bf_lo(rv.x);
    a1 += dev::bf_hi(rv.x);
    a2 += dev::bf_lo(rv.y);
    a3 += dev::bf_hi(rv.y);
  }
  uint2 o2;
  o2.x = dev::pack_bf2(a0, a1);
  o2.y = dev::pack_bf2(a2, a3);
  *reinterpret_cast<uint2 *>(c.y + static_cast<size_t>(t) * c.H + col) = o2;
}

// Live look-ahead prediction (N9): the gates of layers l+1..l+hz
// applied to the CURRENT hidden state x [T, H]; per future layer the top-K of
// each token's logits (value desc, index asc, like router_topk_kernel) are
// counted into counts[f][N] (the predicted loads).  One block per (future
// layer, token); warps split the N dot products, summed in router_logits_kernel's
// order, so the logits -- and the selection -- are bit-identical to
// router_logits + router_topk on the same gate.
__global__ void __launch_bounds__(256) lookahead_kernel(const uint16_t *__restrict__ x,
                                                        const uint16_t *__restrict__ gate_w, int first_layer,
                                                        int hz, int T, int N, int ld, int K, int H,
                                                        int32_t *__restrict__ counts) {
  __shared__ float s_lg[256];
  const int f = blockIdx.x / max(T, 1), t = blockIdx.x % max(T, 1);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint16_t *xr = x + static_cast<size_t>(t) * H;
  const uint16_t *wl = gate_w + static_cast<size_t>(first_layer + f) * ld * H;
  for (int e = wid; e < N; e += nw) {
    const uint16_t *wr = wl + static_cast<size_t>(e) * H;
    float acc = 0.f;
    for (int c = lane * 8; c < H; c += 256)
      acc += dev::dot8(*reinterpret_cast<const uint4 *>(wr + c), *reinterpret_cast<const uint4 *>(xr + c));
    acc = dev::warp_sum(acc);
    if (lane == 0) s_lg[e] = acc;
  }
  __syncthreads();
  if (wid == 0) {
    float v[kMaxPerLane];
#pragma unroll
    for (int j = 0; j < kMaxPerLane; ++j) {
      const int e = lane + 32 * j;
      v[j] = e < N ? s_lg[e] : -FLT_MAX;
    }
    uint32_t taken = 0;
    for (int k = 0; k < K; ++k) {
      float bv = -FLT_MAX;
      int bi = 0x7fffffff;
#pragma unroll
      for (int j = 0; j < kMaxPerLane; ++j) {
        const int e = lane + 32 * j;
        if (e < N && !((taken >> j) & 1u) && (v[j] > bv || (v[j] == bv && e < bi))) {
          bv = v[j];
          bi = e;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (bi >= N) {  // non-finite logits: lowest free index
        bi = 0;
        while (bi < N && __shfl_sync(0xffffffffu, ((taken >> (bi >> 5)) & 1u), bi & 31)) ++bi;
      }
      if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
      if (lane == 0) atomicAdd(&counts[f * N + bi], 1);
    }
  }
}

__global__ void lookahead_publish_kernel(const int32_t *__restrict__ counts, int n, int64_t *host_counts) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) host_counts[i] = counts[i];
  __threadfence_system();
}

// One thread spins until the host writes `seq` into a mapped flag: holds the
// stream while the host enqueues the kernels to be timed, so the CUDA events
// around them measure GPU time, not host launch latency (bench roofline).
// The host releases gates in order and may run several gates ahead of the GPU
// (e.g. launches queued behind H2D copies), so a gate opens once the flag has
// reached ITS sequence number, not only while it equals it (wrap-safe compare).
__global__ void gate_kernel(const uint32_t *flag, uint32_t seq) {
  while (static_cast<int32_t>(*reinterpret_cast<const volatile uint32_t *>(flag) - seq) < 0) {
  }
}

// S[layer, i] <- a * TopP(s)[i] + (1 - a) * S[layer, i]   (caching.py:58-76)
// Round-to-nearest intrinsics keep every operation a separate IEEE rounding,
// exactly like the host core (no FMA contraction).
__global__ void mrs_update_kernel(double *__restrict__ S, const double *__restrict__ s, int layer, int N, int p,
                                  double a) {
  mrs_row_update(S, s, layer, N, p, a);
}

__device__ void mrs_row_update(double *__restrict__ S, const double *__restrict__ s, int layer, int N, int p,
                               double a) {
  const int i = threadIdx.x;
  if (i >= N) return;
  const double si = s[i];
  int rank = 0;
  for (int j = 0; j < N; ++j) {
    const double sj = s[j];
    rank += (sj > si || (sj == si && j < i)) ? 1 : 0;
  }
  const double t = rank < p ? si : 0.0;
  const double keep = __dsub_rn(1.0, a);
  double *row = S + static_cast<size_t>(layer) * N;
  row[i] = __dadd_rn(__dmul_rn(a, t), __dmul_rn(keep, row[i]));
}

}  // namespace
}  // namespace hm

using hm::raise;

#include <atomic>
namespace hm {
static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace hm

extern "C" {

long long hm_launch_count(void) { return hm::g_launches.load(); }

int hm_router_topk(const float *logits, int T, int N, int ld, int K, int renormalize, int n_shared,
                   int shared_gate_col, int32_t *sel, float *w, float *probs, int32_t *counts, void *stream) {
  HM_API_BEGIN
  HM_REQUIRE(N >= 1 && N <= 256 && K >= 1 && K <= 8 && K <= N && ld >= N, HM_EVALUE, "router shape out of range");
  HM_REQUIRE(n_shared >= 0 && n_shared <= 32, HM_EVALUE, "too many shared expert columns");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  HM_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * (N + n_shared), st));
  if (T > 0) {
    const int warps = 8;
    hm::router_topk_kernel<<<(T + warps - 1) / warps, 32 * warps, 0, st>>>(logits, T, N, ld, K, renormalize, n_shared,
                                                                          shared_gate_col, sel, w, probs, counts);
    HM_LAUNCH_CHECK();
  } else if (n_shared > 0) {
    HM_CUDA(cudaMemsetAsync(counts + N, 0, sizeof(int32_t) * n_shared, st));
  }
  HM_API_END
}

int hm_router_fused_small(const float *logits, int T, int N, int ld, int K, int renormalize, int n_shared,
                          int shared_gate_col, const uint16_t *x, int H, int32_t *sel, float *w, int32_t *pos,
                          int32_t *row_src, uint16_t *xp, int32_t *meta_i, double *meta_d, void *stream) {
  HM_API_BEGIN
  HM_REQUIRE(T >= 1 && T <= 32 && N >= 1 && N <= 256 && K >= 1 && K <= 8 && K <= N && ld >= N &&
                 T * (K + n_shared) <= hm::kFusedMaxRows && N + n_shared <= hm::kFusedMaxE && H % 8 == 0,
             HM_EVALUE, "shape outside the fused small-T router");
  hm::launch_router_fused(logits, T, N, ld, K, renormalize, n_shared, shared_gate_col, x, H, sel, w, pos, row_src,
                          xp, meta_i, meta_d, hm::HostMirror{}, static_cast<cudaStream_t>(stream));
  HM_LAUNCH_CHECK();
  HM_API_END
}

int hm_router_fused_mirror(const float *logits, int T, int N, int ld, int K, int renormalize, int n_shared,
                           int shared_gate_col, const uint16_t *x, int H, int32_t *sel, float *w, int32_t *pos,
                           int32_t *row_src, uint16_t *xp, int32_t *meta_i, double *meta_d, int32_t *host_meta_i,
                           double *host_meta_d, uint16_t *host_xp, uint32_t *host_flag, uint32_t seq, void *stream) {
  HM_API_BEGIN
  HM_REQUIRE(T >= 1 && T <= 32 && N >= 1 && N <= 256 && K >= 1 && K <= 8 && K <= N && ld >= N &&
                 T * (K + n_shared) <= hm::kFusedMaxRows && N + n_shared <= hm::kFusedMaxE && H % 8 == 0,
             HM_EVALUE, "shape outside the fused small-T router");
  HM_REQUIRE(host_meta_i && host_meta_d && host_flag, HM_EVALUE, "host mirror needs meta and flag pointers");
  hm::launch_router_fused(logits, T, N, ld, K, renormalize, n_shared, shared_gate_col, x, H, sel, w, pos, row_src,
                          xp, meta_i, meta_d, hm::HostMirror{host_meta_i, host_meta_d, host_xp, host_flag, seq},
                          static_cast<cudaStream_t>(stream));
  HM_LAUNCH_CHECK();
  HM_API_END
}

int hm_router_fused_mirror_mrs(const float *logits, int T, int N, int ld, int K, int renormalize, int n_shared,
                               int shared_gate_col, const uint16_t *x, int H, int32_t *sel, float *w, int32_t *pos,
                               int32_t *row_src, uint16_t *xp, int32_t *meta_i, double *meta_d, int32_t *host_meta_i,
                               double *host_meta_d, uint16_t *host_xp, uint32_t *host_flag, uint32_t seq, double *S,
                               int layer, int mrs_p, double mrs_alpha, double *host_mrs_row, void *stream) {
  HM_API_BEGIN
  HM_REQUIRE(T >= 1 && T <= 32 && N >= 1 && N <= 256 && K >= 1 && K <= 8 && K <= N && ld >= N &&
                 T * (K + n_shared) <= hm::kFusedMaxRows && N + n_shared <= hm::kFusedMaxE && H % 8 == 0,
             HM_EVALUE, "shape outside the fused small-T router");
  HM_REQUIRE(host_meta_i && host_meta_d && host_flag && S && host_mrs_row && layer >= 0, HM_EVALUE,
             "host mirror needs meta, flag, MRS table and row pointers");
  hm::HostMirror m{host_meta_i, host_meta_d, host_xp, host_flag, seq};
  m.S = S;
  m.mrs_row = host_mrs_row;
  m.layer = layer;
  m.p = mrs_p;
  m.alpha = mrs_alpha;
  hm::launch_router_fused(logits, T, N, ld, K, renormalize, n_shared, shared_gate_col, x, H, sel, w, pos, row_src,
                          xp, meta_i, meta_d, m, static_cast<cudaStream_t>(stream));
  HM_LAUNCH_CHECK();
  HM_API_END
}

int hm_score_sums(const float *probs, int T, int N, double *score_sum, void *stream) {
  HM_API_BEGIN
  hm::score_sum_kernel<<<N, 256, 0, static_cast<cudaStream_t>(stream)>>>(probs, T, N, score_sum);
  HM_LAUNCH_CHECK();
  HM_API_END
}

int hm_router_logits(const uint16_t *x, const uint16_t *wg, int T, int H, int N, float *logits, void *stream) {
  HM_API_BEGIN
  HM_REQUIRE(H % 8 == 0, HM_EVALUE, "hidden size must be a multiple of 8");
  const long items = static_cast<long>(T) * N;
  if (items > 0) {
    hm::router_logits_kernel<<<static_cast<unsigned>((items + 7) / 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        x, wg, T, H, N, logits);
    HM_LAUNCH_CHECK();
  }
  HM_API_END
}

int hm_offsets(const int32_t *counts, int E, int32_t *offsets, void *stream) {
  HM_API_BEGIN
  hm::offsets_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(counts, E, offsets);
  HM_LAUNCH_CHECK();
  HM_API_END
}

int hm_permute(const int32_t *sel, int T, int Kp, int E, const int32_t *offsets, int32_t *pos, int32_t *row_src,
               void *stream) {
  HM_API_BEGIN
  if (T > 0) {
    hm::permute_kernel<<<E, 256, 0, static_cast<cudaStream_t>(stream)>>>(sel, T * Kp, offsets, pos, row_src);
    HM_LAUNCH_CHECK();
  }
  HM_API_END
}

int hm_gather_rows(const uint16_t *x, const int32_t *row_src, int rows, int Kp, int H, uint16_t *xp, void *stream) {
  HM_API_BEGIN
  HM_REQUIRE(H % 8 == 0, HM_EVALUE, "hidden size must be a multiple of 8");
  if (rows > 0) {
    hm::gather_kernel<<<rows, 128, 0, static_cast<cudaStream_t>(stream)>>>(x, row_src, rows, Kp, H, xp);
    HM_LAUNCH_CHECK();
  }
  HM_API_END
}

int hm_combine(const float *out, const int32_t *pos, const float *w, int T, int Kp, int H, const uint16_t *residual,
               uint16_t *y, void *stream) {
  HM_API_BEGIN
  HM_REQUIRE(H % 4 == 0, HM_EVALUE, "hidden size must be a multiple of 4");
  if (T > 0) {
    hm::combine_kernel<<<T, 256, 0, static_cast<cudaStream_t>(stream)>>>(out, pos, w, Kp, H, residual, y);
    HM_LAUNCH_CHECK();
  }
  HM_API_END
}

int hm_mask_nonhome(const int32_t *sel, float *w, int TKp, int N, int rank, int world, void *stream) {
  HM_API_BEGIN
  HM_REQUIRE(world >= 1 && rank >= 0 && rank < world, HM_EVALUE, "bad expert-parallel rank");
  if (TKp > 0 && world > 1) {
    hm::mask_nonhome_kernel<<<(TKp + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(sel, w, TKp, N, rank,
                                                                                             world);
    HM_LAUNCH_CHECK();
  }
  HM_API_END
}

int hm_combine_f32(const float *out, const int32_t *pos, const float *w, int T, int Kp, int H, float *y32,
                   void *stream) {
  HM_API_BEGIN
  HM_REQUIRE(H % 4 == 0, HM_EVALUE, "hidden size must be a multiple of 4");
  if (T > 0) {
    hm::combine_f32_kernel<<<T, 256, 0, static_cast<cudaStream_t>(stream)>>>(out, pos, w, Kp, H, y32);
    HM_LAUNCH_CHECK();
  }
  HM_API_END
}

int hm_residual_add(const float *y32, const uint16_t *residual, int T, int H, uint16_t *y, void *stream) {
  HM_API_BEGIN
  HM_REQUIRE(H % 4 == 0, HM_EVALUE, "hidden size must be a multiple of 4");
  if (T > 0) {
    hm::residual_add_kernel<<<T, 256, 0, static_cast<cudaStream_t>(stream)>>>(y32, residual, H, y);
    HM_LAUNCH_CHECK();
  }
  HM_API_END
}

int hm_combine_tail_gated(const float *out, const float *host_out, const uint64_t *host_mask4, const int32_t *pos,
                          const float *w, int T, int Kp, int H, const uint16_t *residual, uint16_t *y, double *S,
                          const double *scores, int layer, int N, int p, double alpha, const uint32_t *gate,
                          uint32_t gate_seq, void *stream);

int hm_combine_tail(const float *out, const float *host_out, const uint64_t *host_mask4, const int32_t *pos,
                    const float *w, int T, int Kp, int H, const uint16_t *residual, uint16_t *y, double *S,
                    const double *scores, int layer, int N, int p, double alpha, void *stream) {
  return hm_combine_tail_gated(out, host_out, host_mask4, pos, w, T, Kp, H, residual, y, S, scores, layer, N, p,
                               alpha, nullptr, 0u, stream);
}

int hm_combine_tail_gated(const float *out, const float *host_out, const uint64_t *host_mask4, const int32_t *pos,
                          const float *w, int T, int Kp, int H, const uint16_t *residual, uint16_t *y, double *S,
                          const double *scores, int layer, int N, int p, double alpha, const uint32_t *gate,
                          uint32_t gate_seq, void *stream) {
  HM_API_BEGIN
  HM_REQUIRE(H % 4 == 0, HM_EVALUE, "hidden size must be a multiple of 4");
  HM_REQUIRE(!S || (N >= 1 && N <= 256), HM_EVALUE, "MRS row too wide for the fused tail");
  hm::CombineTail c{};
  c.out = out;
  c.host_out = host_out;
  c.pos = pos;
  c.w = w;
  c.Kp = Kp;
  c.H = H;
  c.residual = residual;
  c.y = y;
  for (int i = 0; i < 4; ++i) c.host_mask[i] = host_mask4 ? host_mask4[i] : 0ull;
  HM_REQUIRE(!host_mask4 || host_out, HM_EVALUE, "host rows need the host output buffer");
  c.S = S;
  c.scores = scores;
  c.layer = layer;
  c.N = N;
  c.p = p;
  c.a = alpha;
  c.gate = gate;
  c.gate_seq = gate_seq;
  HM_REQUIRE(Kp <= hm::kTailMaxKp, HM_EVALUE, "too many selections per token for the fused tail");
  const int cs = (H + 4 * hm::kTailThreads - 1) / (4 * hm::kTailThreads);
  const long blocks = static_cast<long>(T) * cs + (S ? 1 : 0);
  if (blocks > 0) {
    hm::combine_tail_kernel<<<static_cast<unsigned>(blocks), hm::kTailThreads, 0, static_cast<cudaStream_t>(stream)>>>(c);
    HM_LAUNCH_CHECK();
  }
  HM_API_END
}

int hm_lookahead(const uint16_t *x, const uint16_t *gate_w, int first_layer, int hz, int T, int N, int ld, int K,
                 int H, int32_t *counts, int64_t *host_counts, void *stream) {
  HM_API_BEGIN
  HM_REQUIRE(N >= 1 && N <= 256 && K >= 1 && K <= N && ld >= N && H % 8 == 0 && hz >= 0 && T >= 0, HM_EVALUE,
             "look-ahead shape out of range");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (hz == 0) return HM_OK;
  HM_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * hz * N, st));
  if (T > 0) {
    hm::lookahead_kernel<<<hz * T, 256, 0, st>>>(x, gate_w, first_layer, hz, T, N, ld, K, H, counts);
    HM_LAUNCH_CHECK();
  }
  if (host_counts) {
    hm::lookahead_publish_kernel<<<1, 256, 0, st>>>(counts, hz * N, host_counts);
    HM_LAUNCH_CHECK();
  }
  HM_API_END
}

int hm_gate_wait(const uint32_t *flag, uint32_t seq, void *stream) {
  HM_API_BEGIN
  hm::gate_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(flag, seq);
  HM_LAUNCH_CHECK();
  HM_API_END
}

int hm_mrs_update_dev(double *S, const double *scores, int layer, int N, int p, double alpha, void *stream) {
  HM_API_BEGIN
  HM_REQUIRE(N >= 1 && N <= 1024, HM_EVALUE, "MRS row too wide");
  hm::mrs_update_kernel<<<1, ((N + 31) / 32) * 32, 0, static_cast<cudaStream_t>(stream)>>>(S, scores, layer, N, p,
                                                                                          alpha);
  HM_LAUNCH_CHECK();
  HM_API_END
}

}  // extern "C"
