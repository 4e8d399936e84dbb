// The HybriMoE layer executor on one B200: turns the decision core's per-layer
// record into real work (engine.py:288-389 step order).
//
//   compute stream : router -> score sums -> offsets -> permute/gather
//                    -> [host decides] -> GPU experts (cached batch, then each
//                    transferred expert after its copy) -> combine (+ residual)
//   copy stream    : demand H2D copies in plan transfer order, then prefetches,
//                    each from the pinned master store into its HBM slot
//   host worker    : CPU-assigned experts in plan CPU order, from the pinned
//                    master store, results H2D'd into the permuted output rows
//
// Slot reuse is event-guarded: a copy into a slot waits for the last kernel
// that read it (a demand insert may evict an expert inserted earlier in the
// same layer, engine.py:318-330), and a kernel waits for its slot's copy.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "decision.hpp"
#include "host_worker.hpp"

extern "C" {
int hm_router_topk(const float *, int, int, int, int, int, int, int, int32_t *, float *, float *, int32_t *, void *);
int hm_score_sums(const float *, int, int, double *, void *);
int hm_offsets(const int32_t *, int, int32_t *, void *);
int hm_permute(const int32_t *, int, int, int, const int32_t *, int32_t *, int32_t *, void *);
int hm_gather_rows(const uint16_t *, const int32_t *, int, int, int, uint16_t *, void *);
int hm_expert_ffn(const uint16_t *, int, int, int, const hm_group *, int, const uint16_t *, int, uint16_t *, float *,
                  int, void *);
int hm_combine(const float *, const int32_t *, const float *, int, int, int, const uint16_t *, uint16_t *, void *);
int hm_mrs_update_dev(double *, const double *, int, int, int, double, void *);
int hm_mask_nonhome(const int32_t *, float *, int, int, int, int, void *);
int hm_predict_layers(const int64_t *, int, int, int64_t, int, int64_t, int, double, int32_t *, int64_t *, int *);
int hm_router_fused_small(const float *, int, int, int, int, int, int, int, const uint16_t *, int, int32_t *,
                          float *, int32_t *, int32_t *, uint16_t *, int32_t *, double *, void *);
int hm_combine_f32(const float *, const int32_t *, const float *, int, int, int, float *, void *);
int hm_lookahead(const uint16_t *, const uint16_t *, int, int, int, int, int, int, int, int32_t *, int64_t *, void *);
int hm_router_fused_mirror(const float *, int, int, int, int, int, int, int, const uint16_t *, int, int32_t *, float *,
                           int32_t *, int32_t *, uint16_t *, int32_t *, double *, int32_t *, double *, uint16_t *,
                           uint32_t *, uint32_t, void *);
int hm_ep_combine_allreduce(hm_ep *, const float *, const float *, const uint64_t *, const int32_t *, const float *,
                            int, int, int, const uint16_t *, uint16_t *, float *, void *);
int hm_gate_wait(const uint32_t *, uint32_t, void *);
int hm_q4_image_bytes(int, int, size_t *);
int hm_expert_ffn_q4(const uint8_t *, size_t, int, int, int, const hm_group *, int, const uint16_t *, int, uint16_t *,
                     float *, uint16_t *, int, int, void *);
int hm_ep_dispatch_meta(hm_ep *, const int32_t *, const double *, int32_t *, double *, int32_t *, double *, uint32_t *,
                        uint32_t, void *);
int hm_ep_dispatch_rows(hm_ep *, const uint16_t *, const int32_t *, const int32_t *, int, void *);
int hm_ep_return_rows(hm_ep *, const float *, int, void *);
int hm_ep_dispatch_buffers(hm_ep *, uint16_t **, float **);
int hm_ep_uses_nccl(const hm_ep *);
int hm_ep_world(const hm_ep *);
int hm_combine_tail_gated(const float *, const float *, const uint64_t *, const int32_t *, const float *, int, int, int,
                          const uint16_t *, uint16_t *, double *, const double *, int, int, int, double,
                          const uint32_t *, uint32_t, void *);
int hm_router_fused_mirror_mrs(const float *, int, int, int, int, int, int, int, const uint16_t *, int, int32_t *,
                               float *, int32_t *, int32_t *, uint16_t *, int32_t *, double *, int32_t *, double *,
                               uint16_t *, uint32_t *, uint32_t, double *, int, int, double, double *, void *);
int hm_combine_tail(const float *, const float *, const uint64_t *, const int32_t *, const float *, int, int, int,
                    const uint16_t *, uint16_t *, double *, const double *, int, int, int, double, void *);
}

namespace hm {
namespace {

#define RT_CUDA(call)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) hm::raise(HM_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

inline void ok(int status) {
  if (status != HM_OK) raise(status, last_error());
}

double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

struct Runtime {
  hm_runtime_config cfg;
  Engine *engine;
  int N, K, S, E, Kp, H, I, L;
  int R = 0, W = 1;          // expert-parallel rank / world
  float *y32 = nullptr;      // EP partial output (caller-owned)
  hm_ep *ep = nullptr;       // EP peer-memory exchange (caller-owned)
  // token-sharded EP (hm_runtime_set_ep_dispatch): local routing, all-to-all
  // of rows to home ranks and back; xcur = the rows the expert kernels read
  bool disp = false;
  uint16_t *xrecv = nullptr, *xcur = nullptr;
  float *retbuf = nullptr;
  int32_t *lcounts = nullptr, *loffsets = nullptr;
  double *lsums = nullptr;
  size_t slot_elems, slot_bytes;
  bool q4 = false;                 // 4-bit expert images (weight_bits == 4)
  uint16_t *q4_scratch = nullptr;  // bf16 images for the prefill GEMM on 4-bit experts
  static constexpr int kQ4Scratch = 8;
  int64_t n_slots;
  uint16_t *pool = nullptr;        // device: [n_slots][slot_elems]
  uint16_t *store = nullptr;       // pinned host: [host_images][slot_elems]
  cudaStream_t copy = nullptr;
  std::vector<cudaEvent_t> ready, last_use;
  // Event bookkeeping that skips redundant stream waits/records (each is a
  // driver call on the per-layer critical path):
  //  * copy_pending[s]: a copy into slot s was issued and the compute stream
  //    has not waited on it yet (once it has, stream order covers later work);
  //  * one "use" event per expert-FFN launch (a ring), slot_use_seq[s] = the
  //    launch that last read slot s; the copy stream waits only if it has not
  //    already waited on that launch or a later one.
  std::vector<uint8_t> copy_pending;
  std::vector<int64_t> slot_use_seq;
  static constexpr int kUseRing = 256;
  std::vector<cudaEvent_t> use_ev;
  int64_t use_seq = 0, copy_waited_seq = 0;
  cudaStream_t last_compute = nullptr;
  cudaEvent_t ev_req = nullptr, ev_rows = nullptr, ev_switch = nullptr;
  // device scratch
  int32_t *sel = nullptr, *counts = nullptr, *offsets = nullptr, *pos = nullptr, *row_src = nullptr;
  float *w = nullptr, *probs = nullptr, *out = nullptr;
  double *score_sum = nullptr, *scores_dev = nullptr;
  double *S_dev = nullptr;                   // device alias of the engine's (mapped) MRS table
  double *h_mrs_row = nullptr, *dv_mrs_row = nullptr;  // the GPU-computed new row (mapped)
  void *mrs_registered = nullptr;
  void *dmeta = nullptr, *hmeta = nullptr;  // LayerRequest block (device / pinned host)
  size_t meta_ioff = 0, meta_bytes = 0;
  uint16_t *xp = nullptr, *h = nullptr;
  // pinned host staging
  int32_t *h_counts = nullptr, *h_offsets = nullptr;
  double *h_score_sum = nullptr, *h_scores = nullptr;
  uint16_t *h_x = nullptr;
  float *h_out = nullptr;
  // zero-copy decode path (HM_ZERO_COPY, default on): device views of the
  // mapped pinned buffers above, and the router's completion flag
  bool zero_copy = true;
  bool timing_gate = true;  // HM_TIMING_GATE: gate kernel-timing launches (see ffn())
  void *dv_hmeta = nullptr;
  uint16_t *dv_h_x = nullptr;
  float *dv_h_out = nullptr;
  uint32_t *h_flag = nullptr, *dv_flag = nullptr;
  uint32_t seq = 0, gate_seq = 0;  // h_flag[0]: router flag; h_flag[8]: kernel-timing gate
  uint32_t tail_seq = 0;           // h_flag[4]: host worker done (pre-launched combine tail)
  // live look-ahead prediction (hm_runtime_set_lookahead): gates [L][la_ld][H]
  // of the model, applied to each layer's input for layers l+1..l+la_hz; the
  // predicted loads land in pinned memory (mapped: written by the kernel)
  const uint16_t *la_gate = nullptr;
  int la_ld = 0, la_hz = 0;
  int32_t *la_counts = nullptr;
  int64_t *la_host = nullptr, *la_dv = nullptr;
  std::vector<int32_t> la_layers;
  std::unique_ptr<ThreadPool> workers;
  std::vector<uint16_t> hbuf;
  std::vector<int64_t> loads;
  // optional CUDA-event timing of every expert-FFN launch (the bench's roofline)
  bool time_kernels = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> kev;
  std::vector<int64_t> kbytes;
  size_t kused = 0;

  void ffn(const hm_group *g, int n, int rows, cudaStream_t st) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (time_kernels) {
      if (kused == kev.size()) {
        cudaEvent_t e0, e1;
        RT_CUDA(cudaEventCreate(&e0));
        RT_CUDA(cudaEventCreate(&e1));
        kev.emplace_back(e0, e1);
        kbytes.push_back(0);
      }
      a = kev[kused].first;
      b = kev[kused].second;
      // gate the stream until the launches below are enqueued (released right after)
      if (timing_gate) ok(hm_gate_wait(dv_flag + 8, ++gate_seq, static_cast<void *>(st)));
      RT_CUDA(cudaEventRecord(a, st));
    }
    struct Release {  // never leave the gate closed, even on an exception
      Runtime *r;
      bool on;
      ~Release() {
        if (on) {
          std::atomic_thread_fence(std::memory_order_release);
          reinterpret_cast<volatile uint32_t *>(r->h_flag)[8] = r->gate_seq;
        }
      }
    } release{this, time_kernels && timing_gate};
    if (q4) {
      bool big = false;
      for (int i = 0; i < n; ++i) big = big || g[i].row_count > 4;
      if (big && !q4_scratch)
        RT_CUDA(cudaMalloc(&q4_scratch, static_cast<size_t>(kQ4Scratch) * 3 * H * I * 2));
      ok(hm_expert_ffn_q4(reinterpret_cast<const uint8_t *>(pool), slot_bytes, static_cast<int>(n_slots), H, I, g, n,
                          xcur, rows, h, out, q4_scratch, kQ4Scratch, HM_FFN_AUTO, static_cast<void *>(st)));
    } else {
      ok(hm_expert_ffn(pool, static_cast<int>(n_slots), H, I, g, n, xcur, rows, h, out, HM_FFN_AUTO,
                       static_cast<void *>(st)));
    }
    if (time_kernels) {
      RT_CUDA(cudaEventRecord(b, st));
      int64_t by = 0;
      for (int i = 0; i < n; ++i)  // weights streamed + activations in/out
        by += static_cast<int64_t>(slot_bytes) + static_cast<int64_t>(g[i].row_count) * (2LL * H + 2LL * I * 2 + 4LL * H);
      kbytes[kused++] = by;
    }
  }
  std::vector<double> scores;

  Runtime(const hm_runtime_config &c, Engine *eng) : cfg(c), engine(eng) {
    L = c.num_layers;
    N = c.num_routed;
    K = c.num_activated;
    S = c.n_shared;
    E = N + S;
    Kp = K + S;
    H = c.hidden;
    I = c.inter;
    W = c.ep_world > 1 ? c.ep_world : 1;
    R = W > 1 ? c.ep_rank : 0;
    HM_REQUIRE(R >= 0 && R < W, HM_EVALUE, "bad expert-parallel rank");
    HM_REQUIRE(L >= 1 && N >= 1 && K >= 1 && K <= N && S >= 0 && H > 0 && I > 0, HM_EVALUE, "bad runtime shape");
    HM_REQUIRE(engine->cfg.num_layers == L && engine->cfg.num_routed == N && engine->cache.capacity == c.capacity,
               HM_EVALUE, "engine and runtime disagree on the model shape or cache capacity");
    HM_REQUIRE(c.host_images >= 1 && c.max_tokens >= 1, HM_EVALUE, "bad runtime sizes");
    HM_REQUIRE(c.weight_bits == 0 || c.weight_bits == 16 || c.weight_bits == 4, HM_EVALUE,
               "weight_bits must be 16 (bf16) or 4");
    q4 = c.weight_bits == 4;
    if (q4) {
      size_t b = 0;
      ok(hm_q4_image_bytes(H, I, &b));
      slot_bytes = (b + 255) / 256 * 256;  // keep every image 256-byte aligned
    } else {
      slot_bytes = static_cast<size_t>(3) * H * I * 2;
    }
    slot_elems = slot_bytes / 2;
    // [0, capacity) cache slots, then the shared chunks, then one staging slot
    // for transfers that enter no cache slot (capacity 0, e.g. a small budget
    // or an expert-parallel rank whose share rounds to 0: the plan still
    // copies and computes them on the GPU, they are just not kept)
    n_slots = c.capacity + static_cast<int64_t>(L) * S + 1;
    if (n_slots > 0) RT_CUDA(cudaMalloc(&pool, static_cast<size_t>(n_slots) * slot_bytes));
    RT_CUDA(cudaHostAlloc(&store, static_cast<size_t>(c.host_images) * slot_bytes, cudaHostAllocPortable));
    RT_CUDA(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
    ready.resize(static_cast<size_t>(n_slots));
    last_use.resize(static_cast<size_t>(n_slots));
    copy_pending.assign(static_cast<size_t>(n_slots), 0);
    slot_use_seq.assign(static_cast<size_t>(n_slots), 0);
    use_ev.resize(kUseRing);
    for (auto &e : use_ev) RT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (int64_t s = 0; s < n_slots; ++s) {
      RT_CUDA(cudaEventCreateWithFlags(&ready[s], cudaEventDisableTiming));
      RT_CUDA(cudaEventCreateWithFlags(&last_use[s], cudaEventDisableTiming));
    }
    RT_CUDA(cudaEventCreateWithFlags(&ev_req, cudaEventDisableTiming));
    RT_CUDA(cudaEventCreateWithFlags(&ev_rows, cudaEventDisableTiming));
    RT_CUDA(cudaEventCreateWithFlags(&ev_switch, cudaEventDisableTiming));
    const size_t T = static_cast<size_t>(c.max_tokens);
    const size_t rows = T * Kp;
    RT_CUDA(cudaMalloc(&sel, rows * 4));
    RT_CUDA(cudaMalloc(&w, rows * 4));
    RT_CUDA(cudaMalloc(&probs, T * N * 4));
    // LayerRequest block: [counts E | offsets E+1] int32, 8-byte aligned, then
    // [score_sum N | scores N] fp64 -- one buffer on each side, one D2H copy
    meta_ioff = ((2 * static_cast<size_t>(E) + 1) * 4 + 7) / 8 * 8;
    meta_bytes = meta_ioff + 2 * static_cast<size_t>(N) * 8;
    RT_CUDA(cudaMalloc(&dmeta, meta_bytes));
    RT_CUDA(cudaHostAlloc(&hmeta, meta_bytes, cudaHostAllocMapped));
    counts = reinterpret_cast<int32_t *>(dmeta);
    offsets = counts + E;
    score_sum = reinterpret_cast<double *>(static_cast<char *>(dmeta) + meta_ioff);
    scores_dev = score_sum + N;
    h_counts = reinterpret_cast<int32_t *>(hmeta);
    h_offsets = h_counts + E;
    h_score_sum = reinterpret_cast<double *>(static_cast<char *>(hmeta) + meta_ioff);
    RT_CUDA(cudaMalloc(&pos, rows * 4));
    RT_CUDA(cudaMalloc(&row_src, rows * 4));
    RT_CUDA(cudaMalloc(&xp, rows * H * 2));
    RT_CUDA(cudaMalloc(&h, rows * I * 2));
    RT_CUDA(cudaMalloc(&out, rows * H * 4));
    // the decision core's own MRS table, mapped: the zero-copy decode router
    // reads a layer's old row from it and computes the new row on the GPU
    // (the decision core consumes that row at step (5)); one table, no copy
    if (engine->mrs_ && !engine->mrs_->S.empty()) {
      const size_t bytes = (engine->mrs_->S.size() * 8 + 4095) / 4096 * 4096;
      const cudaError_t e = cudaHostRegister(engine->mrs_->S.data(), bytes, cudaHostRegisterMapped);
      if (e == cudaSuccess) {
        mrs_registered = engine->mrs_->S.data();
      } else if (e == cudaErrorHostMemoryAlreadyRegistered) {
        (void)cudaGetLastError();
      } else {
        RT_CUDA(e);
      }
      RT_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void **>(&S_dev), engine->mrs_->S.data(), 0));
      RT_CUDA(cudaHostAlloc(&h_mrs_row, static_cast<size_t>(N) * 8, cudaHostAllocMapped));
      RT_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void **>(&dv_mrs_row), h_mrs_row, 0));
    }
    RT_CUDA(cudaHostAlloc(&h_scores, N * 8, 0));
    RT_CUDA(cudaHostAlloc(&h_x, rows * H * 2, cudaHostAllocMapped));
    RT_CUDA(cudaHostAlloc(&h_out, rows * H * 4, cudaHostAllocMapped));
    RT_CUDA(cudaHostAlloc(&h_flag, 64, cudaHostAllocMapped));
    for (int i = 0; i < 16; ++i) reinterpret_cast<volatile uint32_t *>(h_flag)[i] = 0;
    if (const char *zc = std::getenv("HM_ZERO_COPY")) zero_copy = std::atoi(zc) != 0;
    if (const char *tg = std::getenv("HM_TIMING_GATE")) timing_gate = std::atoi(tg) != 0;
    // under a kernel profiler (ncu injects itself) launches are serialised and
    // replayed: a kernel waiting for the host would never be released
    // (nor would a host-mapped flag survive the profiler's save/restore of the
    // kernel's writes): fall back to the event-synchronised copy path
    if (std::getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") || std::getenv("CUDA_INJECTION64_PATH"))
      timing_gate = zero_copy = false;

    RT_CUDA(cudaHostGetDevicePointer(&dv_hmeta, hmeta, 0));
    RT_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void **>(&dv_h_x), h_x, 0));
    RT_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void **>(&dv_h_out), h_out, 0));
    RT_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void **>(&dv_flag), h_flag, 0));
    workers.reset(new ThreadPool(c.cpu_threads > 0 ? c.cpu_threads
                                                   : static_cast<int>(std::thread::hardware_concurrency())));
    loads.assign(N, 0);
    scores.assign(N, 0.0);
  }

  ~Runtime() {
    if (copy) cudaStreamSynchronize(copy);
    for (auto e : ready) cudaEventDestroy(e);
    for (auto e : last_use) cudaEventDestroy(e);
    for (auto e : use_ev) cudaEventDestroy(e);
    for (auto &e : cev) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
    if (ev_req) cudaEventDestroy(ev_req);
    if (ev_rows) cudaEventDestroy(ev_rows);
    if (ev_switch) cudaEventDestroy(ev_switch);
    if (copy) cudaStreamDestroy(copy);
    if (lcounts) cudaFree(lcounts);
    if (q4_scratch) cudaFree(q4_scratch);
    if (lsums) cudaFree(lsums);
    if (la_counts) cudaFree(la_counts);
    if (la_host) cudaFreeHost(la_host);
    for (void *p : {static_cast<void *>(pool), static_cast<void *>(sel), static_cast<void *>(w),
                    static_cast<void *>(probs), dmeta, static_cast<void *>(pos), static_cast<void *>(row_src),
                    static_cast<void *>(xp), static_cast<void *>(h), static_cast<void *>(out)})
      if (p) cudaFree(p);
    if (mrs_registered) cudaHostUnregister(mrs_registered);
    if (h_mrs_row) cudaFreeHost(h_mrs_row);
    for (void *p : {static_cast<void *>(store), hmeta, static_cast<void *>(h_scores), static_cast<void *>(h_x),
                    static_cast<void *>(h_out), static_cast<void *>(h_flag)})
      if (p) cudaFreeHost(p);
  }

  int64_t image_of(int layer, int expert) const {
    if (W == 1) return (static_cast<int64_t>(layer) * N + expert) % cfg.host_images;
    // a rank stores only its home experts e = R + W*j, j < n_home
    const int64_t n_home = (N - R + W - 1) / W;
    return (static_cast<int64_t>(layer) * n_home + expert / W) % cfg.host_images;
  }
  int64_t shared_slot(int layer, int chunk) const { return cfg.capacity + static_cast<int64_t>(layer) * S + chunk; }
  int64_t staging_slot() const { return n_slots - 1; }
  uint16_t *slot_ptr(int64_t s) const { return pool + static_cast<size_t>(s) * slot_elems; }
  const uint16_t *image_ptr(uint32_t ref) const {
    return store + static_cast<size_t>(image_of(ref_layer(ref), ref_expert(ref))) * slot_elems;
  }

  // Spin until the router kernel raised this layer's flag; poll the stream now
  // and then so a failed launch surfaces as an error instead of a hang.
  void wait_flag(cudaStream_t st) {
    volatile uint32_t *f = h_flag;
    for (uint64_t i = 1;; ++i) {
      if (*f == seq) break;
      if ((i & 4095) == 0) {
        const cudaError_t e = cudaStreamQuery(st);
        if (e != cudaSuccess && e != cudaErrorNotReady) RT_CUDA(e);
        if (e == cudaSuccess && *f != seq) raise(HM_ECUDA, "router finished without raising the host flag");
      }
      __builtin_ia32_pause();
    }
    std::atomic_thread_fence(std::memory_order_acquire);
  }

  // The router raises its request flag before gathering the rows; the host
  // worker reads the mirrored rows only after the rows flag (h_flag[2]).
  void wait_rows_flag(cudaStream_t st) {
    volatile uint32_t *f = h_flag + 2;
    for (uint64_t i = 1;; ++i) {
      if (*f == seq) break;
      if ((i & 4095) == 0) {
        const cudaError_t e = cudaStreamQuery(st);
        if (e != cudaSuccess && e != cudaErrorNotReady) RT_CUDA(e);
        if (e == cudaSuccess && *f != seq) raise(HM_ECUDA, "router finished without raising the rows flag");
      }
      __builtin_ia32_pause();
    }
    std::atomic_thread_fence(std::memory_order_acquire);
  }

  void issue_copy(uint32_t ref, int64_t slot, cudaStream_t /*compute*/) {
    const int64_t u = slot_use_seq[slot];
    if (u > copy_waited_seq) {  // wait for the last kernel that read this slot
      RT_CUDA(cudaStreamWaitEvent(copy, use_ev[u % kUseRing], 0));
      copy_waited_seq = u;
    }
    if (time_copies) {  // H2D achieved GB/s: events on the copy stream around each copy
      if (cused == cev.size()) {
        cudaEvent_t e0, e1;
        RT_CUDA(cudaEventCreate(&e0));
        RT_CUDA(cudaEventCreate(&e1));
        cev.emplace_back(e0, e1);
      }
      RT_CUDA(cudaEventRecord(cev[cused].first, copy));
    }
    RT_CUDA(cudaMemcpyAsync(slot_ptr(slot), image_ptr(ref), slot_bytes, cudaMemcpyHostToDevice, copy));
    if (time_copies) RT_CUDA(cudaEventRecord(cev[cused++].second, copy));
    RT_CUDA(cudaEventRecord(ready[slot], copy));
    copy_pending[slot] = 1;
  }
  bool time_copies = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> cev;
  size_t cused = 0;

  // Order the compute stream after the latest copy into `slot` (if not already).
  void wait_ready(int64_t slot, cudaStream_t st) {
    if (!copy_pending[slot]) return;
    RT_CUDA(cudaStreamWaitEvent(st, ready[slot], 0));
    copy_pending[slot] = 0;
  }

  // Record that the kernels just launched on `st` read these slots.
  void mark_used(const hm_group *g, int n, cudaStream_t st) {
    ++use_seq;
    RT_CUDA(cudaEventRecord(use_ev[use_seq % kUseRing], st));
    for (int i = 0; i < n; ++i) slot_use_seq[g[i].slot] = use_seq;
  }

  // The fixed-residency baselines plan GPU experts as already cached
  // (engine.py:171-205): their experts must have been preloaded into slots.
  // Checked before the engine mutates any state, with a clear message.
  void check_fixed_residency(int layer) const {
    const int sch = engine->cfg.scheduling;
    if (sch != HM_SCHED_STATIC_SPLIT && sch != HM_SCHED_FIXED_MAP) return;
    for (int e = 0; e < N; ++e) {
      if (loads[e] <= 0) continue;
      const uint32_t r = pack_ref(layer, e);
      const bool gpu = sch == HM_SCHED_STATIC_SPLIT ? layer < engine->cfg.split_point
                                                    : engine->fixed_pinned.count(r) > 0;
      if (!gpu) continue;
      auto it = engine->cache.resident.find(r);
      HM_REQUIRE(it != engine->cache.resident.end() && it->second.slot >= 0 && it->second.slot < cfg.capacity,
                 HM_EVALUE,
                 std::string(sch == HM_SCHED_STATIC_SPLIT ? "static_layer_split" : "fixed_frequency_map") +
                     " plans expert (" + std::to_string(layer) + ", " + std::to_string(e) +
                     ") on the GPU but it is not preloaded into an HBM slot (HybridMoE.preload)");
    }
  }

  int64_t checked_slot(uint32_t ref, int64_t slot) const {
    HM_REQUIRE(slot >= 0 && slot < cfg.capacity, HM_EVALUE,
               "expert (" + std::to_string(ref_layer(ref)) + ", " + std::to_string(ref_expert(ref)) +
                   ") has no HBM slot (resident beyond the cache capacity)");
    return slot;
  }

  void forward_layer(int layer, const uint16_t *x, const float *logits, int T, int ld, uint16_t *y,
                     const int32_t *pred_layers, const int64_t *pred_loads, int n_pred, cudaStream_t st,
                     hm_layer_stats *stats) {
    HM_REQUIRE(layer >= 0 && layer < L, HM_EVALUE, "layer out of range");
    HM_REQUIRE((T >= 1 || disp) && T >= 0 && T <= cfg.max_tokens, HM_EVALUE,
               "token count exceeds the runtime's max_tokens");
    hm_layer_stats s{};
    void *vs = static_cast<void *>(st);
    const int rows = T * Kp;
    if (st != last_compute) {
      // a new compute stream: order it after ALL work of the previous one (the
      // combine / MRS launches still read out, pos, w, scores_dev and the
      // mapped h_out that this layer's router and host worker overwrite)
      if (last_compute != nullptr) {
        RT_CUDA(cudaEventRecord(ev_switch, last_compute));
        RT_CUDA(cudaStreamWaitEvent(st, ev_switch, 0));
      } else if (use_seq > 0) {
        RT_CUDA(cudaStreamWaitEvent(st, use_ev[use_seq % kUseRing], 0));
      }
      last_compute = st;
    }
    // (0) router, LayerRequest, permutation -- all on the compute stream; the
    // LayerRequest (counts, offsets, score sums, scores) lands in one pinned
    // buffer with a single D2H copy: the only per-layer host synchronisation
    const bool fused = !disp && T <= 32 && rows <= 1024 && N <= 256 && E <= 320 && H % 8 == 0;
    xcur = xp;
    // zero-copy: the router writes the LayerRequest (and, when small, the routed
    // rows) into mapped host memory and raises a flag the host spins on
    const bool mirror = fused && zero_copy;
    const bool mirror_rows = mirror && static_cast<size_t>(T) * K * H * 2 <= (512u << 10);
    // live prediction: launched ahead of the router so the predicted loads are
    // on the host when the LayerRequest is (same flag / same event)
    if (n_pred == HM_PREDICT_LIVE) {
      HM_REQUIRE(la_gate != nullptr, HM_EVALUE, "live prediction needs hm_runtime_set_lookahead");
      HM_REQUIRE(!disp, HM_EVALUE, "live prediction is not available in token-sharded dispatch mode");
      n_pred = std::max(0, std::min(layer + la_hz, L - 1) - layer);
      if (n_pred > 0) {
        // the publish kernel stores the int64 loads into mapped memory: stream
        // order puts it before the router's flag / event
        ok(hm_lookahead(x, la_gate, layer + 1, n_pred, T, N, la_ld, K, H, la_counts, la_dv, vs));
      }
      for (int d = 0; d < n_pred; ++d) la_layers[d] = layer + 1 + d;
      pred_layers = la_layers.data();
      pred_loads = la_host;
    }
    // the MRS row of this layer on the GPU, inside the router (zero-copy decode)
    const bool gpu_row = mirror && cfg.gpu_mrs && engine->cfg.cache_policy == HM_POLICY_MRS && S_dev != nullptr;
    if (mirror && gpu_row) {
      ++seq;
      ok(hm_router_fused_mirror_mrs(logits, T, N, ld, K, cfg.renormalize, S, cfg.shared_gate_col, x, H, sel, w, pos,
                                    row_src, xp, counts, score_sum, static_cast<int32_t *>(dv_hmeta),
                                    reinterpret_cast<double *>(static_cast<char *>(dv_hmeta) + meta_ioff),
                                    mirror_rows ? dv_h_x : nullptr, dv_flag, seq, S_dev, layer, engine->mrs_->p,
                                    engine->mrs_->alpha, dv_mrs_row, vs));
      if (W > 1) ok(hm_mask_nonhome(sel, w, T * Kp, N, R, W, vs));
    } else if (mirror) {
      ++seq;
      ok(hm_router_fused_mirror(logits, T, N, ld, K, cfg.renormalize, S, cfg.shared_gate_col, x, H, sel, w, pos,
                                row_src, xp, counts, score_sum, static_cast<int32_t *>(dv_hmeta),
                                reinterpret_cast<double *>(static_cast<char *>(dv_hmeta) + meta_ioff),
                                mirror_rows ? dv_h_x : nullptr, dv_flag, seq, vs));
      if (W > 1) ok(hm_mask_nonhome(sel, w, T * Kp, N, R, W, vs));
    } else if (fused) {  // decode: one launch does router .. gather
      ok(hm_router_fused_small(logits, T, N, ld, K, cfg.renormalize, S, cfg.shared_gate_col, x, H, sel, w, pos,
                               row_src, xp, counts, score_sum, vs));
      if (W > 1) ok(hm_mask_nonhome(sel, w, T * Kp, N, R, W, vs));
      RT_CUDA(cudaMemcpyAsync(hmeta, dmeta, meta_bytes, cudaMemcpyDeviceToHost, st));
      RT_CUDA(cudaEventRecord(ev_req, st));
    } else if (disp) {  // this rank's tokens: local routing, then the all-gather + all-to-all
      ok(hm_router_topk(logits, T, N, ld, K, cfg.renormalize, S, cfg.shared_gate_col, sel, w, probs, lcounts, vs));
      ok(hm_score_sums(probs, T, N, lsums, vs));
      ok(hm_offsets(lcounts, E, loffsets, vs));
      ok(hm_permute(sel, T, Kp, E, loffsets, pos, row_src, vs));
      ok(hm_gather_rows(x, row_src, rows, Kp, H, xp, vs));
      ++seq;
      ok(hm_ep_dispatch_meta(ep, lcounts, lsums, counts, score_sum, static_cast<int32_t *>(dv_hmeta),
                             reinterpret_cast<double *>(static_cast<char *>(dv_hmeta) + meta_ioff), dv_flag, seq, vs));
      // peer memory: the row all-to-all is a kernel sized on the device; NCCL
      // sizes its sends on the host, after the meta flag (below)
      if (!hm_ep_uses_nccl(ep)) ok(hm_ep_dispatch_rows(ep, xp, sel, row_src, rows, vs));
    } else {
      ok(hm_router_topk(logits, T, N, ld, K, cfg.renormalize, S, cfg.shared_gate_col, sel, w, probs, counts, vs));
      if (W > 1) ok(hm_mask_nonhome(sel, w, T * Kp, N, R, W, vs));
      ok(hm_score_sums(probs, T, N, score_sum, vs));
      ok(hm_offsets(counts, E, offsets, vs));
      RT_CUDA(cudaMemcpyAsync(hmeta, dmeta, meta_bytes, cudaMemcpyDeviceToHost, st));
      RT_CUDA(cudaEventRecord(ev_req, st));
      ok(hm_permute(sel, T, Kp, E, offsets, pos, row_src, vs));
      ok(hm_gather_rows(x, row_src, rows, Kp, H, xp, vs));
    }
    double t0 = now_us();
    if (mirror || disp) {
      wait_flag(st);
      if (disp && hm_ep_uses_nccl(ep)) ok(hm_ep_dispatch_rows(ep, xp, sel, row_src, rows, vs));
    } else {
      RT_CUDA(cudaEventSynchronize(ev_req));
    }
    double t1 = now_us();
    s.t_wait_router_us = t1 - t0;

    // (1)-(7) the decision core, engine.py:288-389
    double tot = 0.0;
    for (int e = 0; e < N; ++e) tot += h_score_sum[e];
    for (int e = 0; e < N; ++e) {
      // rank-masked LayerRequest under expert parallelism: other ranks' loads
      // are zeroed, scores stay whole so every rank's S table is identical
      loads[e] = (W == 1 || e % W == R) ? h_counts[e] : 0;
      scores[e] = tot > 0.0 ? h_score_sum[e] / tot : 0.0;  // == the fused kernel's scores, bit for bit
      h_scores[e] = scores[e];
    }
    check_fixed_residency(layer);
    if (gpu_row) engine->gpu_mrs_row = h_mrs_row;  // step (5) takes the router's row
    engine->run_layer(layer, loads.data(), scores.data(), N, pred_layers, pred_loads, n_pred);
    const LayerRecord &rec = engine->rec;
    s.makespan_planned = rec.plan.makespan;
    double t2 = now_us();
    s.t_decide_us = t2 - t1;

    // the rows the experts read: local permuted rows, or (token-sharded EP) the
    // rows every rank dispatched to this home rank, h_offsets[E] of them
    const int rows_used = disp ? h_offsets[E] : rows;
    if (disp) xcur = xrecv;
    // CPU rows to host first so the worker can start while the GPU computes
    std::vector<uint32_t> cpu_refs;
    for (const Event &ev : rec.plan.events)
      if (ev.device == HM_DEV_CPU) cpu_refs.push_back(ev.ref);
    if (!mirror_rows) {
      for (uint32_t r : cpu_refs) {
        const int e = ref_expert(r);
        const size_t rb = h_offsets[e], rc = h_counts[e];
        RT_CUDA(cudaMemcpyAsync(h_x + rb * H, xcur + rb * H, rc * H * 2, cudaMemcpyDeviceToHost, st));
      }
      if (!cpu_refs.empty()) RT_CUDA(cudaEventRecord(ev_rows, st));
    }

    auto assign_of = [&](uint32_t ref) {
      for (auto &a : rec.plan.assign)
        if (a.first == ref) return a.second;
      return -1;
    };
    // CPU experts in plan CPU order (scheduling.py:257-268)
    // CPU outputs reach the combine either zero-copy (positions < 256, the
    // combine reads the mapped host rows) or by H2D copies into `out`
    const bool do_mrs = cfg.gpu_mrs && engine->cfg.cache_policy == HM_POLICY_MRS && engine->mrs_;
    const bool tail = W == 1 && !disp && (!do_mrs || fused) && N <= 256;  // combine_tail launch
    bool zc_out = zero_copy && !disp && (tail || (W > 1 && ep));
    uint64_t host_mask[4] = {0, 0, 0, 0};
    for (uint32_t r : cpu_refs) {
      const int e = ref_expert(r);
      const int rb = h_offsets[e], rc = h_counts[e];
      if (rb + rc > 256) zc_out = false;
      for (int q = rb; q < rb + rc && q < 256; ++q) host_mask[q >> 6] |= 1ull << (q & 63);
    }
    // decode: the combine tail is launched BEFORE the host worker runs, gated on
    // a mapped flag the host raises when the worker's rows are written -- its
    // launch latency leaves the serial path (the GPU starts it within a PCIe
    // poll of the flag); the release is RAII so an exception never leaves the
    // GPU waiting
    const bool pre_tail = tail && zc_out && !cpu_refs.empty();
    struct TailGate {
      Runtime *r;
      bool on;
      void open() {
        if (!on) return;
        std::atomic_thread_fence(std::memory_order_release);
        reinterpret_cast<volatile uint32_t *>(r->h_flag)[4] = r->tail_seq;
        on = false;
      }
      ~TailGate() { open(); }
    } tail_gate{this, false};
    // Everything the GPU gets for this layer (resident experts and shared
    // chunks, transfers + their experts, prefetches, the gated combine tail).
    // In decode it is issued while the host worker's threads already run:
    // the caller joins the worker pass only after these launches (its share
    // of the rows is stolen meanwhile), so ~20 µs of launch overhead per
    // layer leaves the serial path.
    auto issue_gpu = [&]() {
      // GPU experts already resident (and the layer's shared chunks): one launch
      std::vector<hm_group> batch;
      for (const Event &ev : rec.plan.events) {
        if (ev.device != HM_DEV_GPU || assign_of(ev.ref) != HM_ASSIGN_GPU_CACHED) continue;
        const int e = ref_expert(ev.ref);
        const int64_t slot = checked_slot(ev.ref, engine->cache.resident.at(ev.ref).slot);
        wait_ready(slot, st);  // a prefetch may still be in flight
        batch.push_back(hm_group{static_cast<int32_t>(slot), h_offsets[e], h_counts[e], 0});
      }
      s.n_gpu = static_cast<int32_t>(batch.size());
      for (int c = 0; c < S; ++c)
        if (c % W == R)
          batch.push_back(hm_group{static_cast<int32_t>(shared_slot(layer, c)), h_offsets[N + c], h_counts[N + c], 0});
      s.bytes_gpu = static_cast<int64_t>(batch.size()) * static_cast<int64_t>(slot_bytes);
      if (!batch.empty()) {
        ffn(batch.data(), static_cast<int>(batch.size()), rows_used, st);
        mark_used(batch.data(), static_cast<int>(batch.size()), st);
      }
      // Copies in plan transfer order (== insert order), then prefetches; an
      // expert the plan computes on the GPU is launched right after its copy so
      // that a later copy into the same slot (same-layer eviction) waits for it.
      auto copy_and_maybe_compute = [&](uint32_t ref, int64_t slot, bool demand) {
        issue_copy(ref, slot, st);
        s.bytes_h2d += static_cast<int64_t>(slot_bytes);
        if (demand && assign_of(ref) == HM_ASSIGN_GPU_TRANSFER) {
          const int e = ref_expert(ref);
          wait_ready(slot, st);
          hm_group g{static_cast<int32_t>(slot), h_offsets[e], h_counts[e], 0};
          ffn(&g, 1, rows_used, st);
          mark_used(&g, 1, st);
          ++s.n_gpu;
          s.bytes_gpu += static_cast<int64_t>(slot_bytes);
        }
      };
      for (size_t i = 0; i < rec.demand.size(); ++i) {
        copy_and_maybe_compute(rec.demand[i].first, checked_slot(rec.demand[i].first, rec.demand_slots[i]), true);
        ++s.n_transfer;
      }
      // transfers that entered no cache slot (capacity 0: engine.py:318 inserts
      // only when capacity > 0) still run where the plan put them: through the
      // staging slot, one at a time (each copy waits for the previous reader)
      if (rec.demand.size() < static_cast<size_t>(std::count_if(
                                  rec.plan.events.begin(), rec.plan.events.end(),
                                  [](const Event &e) { return e.kind == HM_KIND_TRANSFER; }))) {
        std::vector<const Event *> xf;
        for (const Event &e : rec.plan.events)
          if (e.kind == HM_KIND_TRANSFER) xf.push_back(&e);
        std::stable_sort(xf.begin(), xf.end(), [](const Event *a, const Event *b) { return a->start < b->start; });
        for (const Event *e : xf) {
          bool inserted = false;
          for (auto &d : rec.demand) inserted = inserted || d.first == e->ref;
          if (inserted) continue;
          copy_and_maybe_compute(e->ref, staging_slot(), true);
          ++s.n_transfer;
        }
      }
      for (size_t i = 0; i < rec.chosen.size(); ++i) {
        copy_and_maybe_compute(rec.chosen[i].first, checked_slot(rec.chosen[i].first, rec.chosen_slots[i]), false);
        ++s.n_prefetch;
      }
      if (pre_tail) {
        ++tail_seq;
        tail_gate.on = true;
        ok(hm_combine_tail_gated(out, dv_h_out, host_mask, pos, w, T, Kp, H, cfg.residual ? x : nullptr, y, nullptr,
                                 scores_dev, layer, N, 0, 0.0, dv_flag + 4, tail_seq, vs));
      }
    };
    if (!cpu_refs.empty()) {
      if (!mirror_rows)
        RT_CUDA(cudaEventSynchronize(ev_rows));
      else
        wait_rows_flag(st);
      const double c0 = now_us();
      bool all_single = true;
      for (uint32_t r : cpu_refs) all_single = all_single && h_counts[ref_expert(r)] == 1;
      if (all_single) {  // decode: the layer's CPU experts in one worker pass
        std::vector<const uint16_t *> imgs, xs;
        std::vector<float *> outs;
        for (uint32_t r : cpu_refs) {
          const size_t rb = h_offsets[ref_expert(r)];
          imgs.push_back(image_ptr(r));
          // a one-token mirror carries the token once (row 0): every routed row is it
          xs.push_back(h_x + (mirror_rows && T == 1 ? 0 : rb) * H);
          outs.push_back(h_out + rb * H);
        }
        const std::function<void()> gpu_first = issue_gpu;
        if (q4) {
          std::vector<const uint8_t *> qimgs;
          for (auto *p : imgs) qimgs.push_back(reinterpret_cast<const uint8_t *>(p));
          cpu_experts_decode_q4(*workers, qimgs.data(), xs.data(), static_cast<int>(imgs.size()), H, I, outs.data(),
                                hbuf, &gpu_first);
        } else {
          cpu_experts_decode(*workers, imgs.data(), xs.data(), static_cast<int>(imgs.size()), H, I, outs.data(),
                             hbuf, &gpu_first);
        }
      } else {
        // prefill: the layer's AMX-sized bf16 experts in one worker pass (GPU
        // launches issued while it starts), the rest one by one in plan CPU order
        std::vector<const uint16_t *> bimgs, bxs;
        std::vector<float *> bouts;
        std::vector<int> bms;
        std::vector<uint32_t> rest;
        static const bool batch = [] {  // HM_PREFILL_BATCH=0: one worker pass per expert (A/B)
          const char *e = std::getenv("HM_PREFILL_BATCH");
          return !e || std::atoi(e) != 0;
        }();
        const bool amx = batch && !q4 && amx_available();
        for (uint32_t r : cpu_refs) {
          const int e = ref_expert(r);
          const size_t rb = h_offsets[e];
          if (amx && h_counts[e] >= 8) {
            bimgs.push_back(image_ptr(r));
            bxs.push_back(h_x + rb * H);
            bouts.push_back(h_out + rb * H);
            bms.push_back(h_counts[e]);
          } else {
            rest.push_back(r);
          }
        }
        if (!bimgs.empty()) {
          const std::function<void()> gpu_first = issue_gpu;
          cpu_experts_amx(*workers, bimgs.data(), bxs.data(), bms.data(), static_cast<int>(bimgs.size()), H, I,
                          bouts.data(), hbuf, &gpu_first);
        } else {
          issue_gpu();
        }
        for (uint32_t r : rest) {  // plan CPU order
          const int e = ref_expert(r);
          const size_t rb = h_offsets[e];
          if (q4)
            cpu_expert_q4(*workers, reinterpret_cast<const uint8_t *>(image_ptr(r)), H, I, h_x + rb * H, h_counts[e],
                          h_out + rb * H, hbuf);
          else
            cpu_expert(*workers, image_ptr(r), H, I, h_x + rb * H, h_counts[e], h_out + rb * H, hbuf);
        }
      }
      s.n_cpu = static_cast<int32_t>(cpu_refs.size());
      s.bytes_cpu = static_cast<int64_t>(cpu_refs.size()) * static_cast<int64_t>(slot_bytes);
      s.t_cpu_us = now_us() - c0;
      if (!zc_out) {
        for (uint32_t r : cpu_refs) {
          const int e = ref_expert(r);
          const size_t rb = h_offsets[e], rc = h_counts[e];
          RT_CUDA(cudaMemcpyAsync(out + rb * H, h_out + rb * H, rc * H * 4, cudaMemcpyHostToDevice, st));
        }
      }
    } else {
      issue_gpu();
    }
    tail_gate.open();
    if (pre_tail) {
      if (stats) *stats = s;
      return;
    }
    if (tail) {
      // one launch: combine (+ residual, host rows zero-copy)
      ok(hm_combine_tail(out, dv_h_out, zc_out && !cpu_refs.empty() ? host_mask : nullptr, pos, w, T, Kp, H,
                         cfg.residual ? x : nullptr, y, nullptr, scores_dev, layer, N, 0, 0.0, vs));
      if (stats) *stats = s;
      return;
    }
    // combine (Eq. 1) with the residual stream, then the GPU copy of S
    if (disp) {  // expert outputs back to their source ranks, then the local combine
      ok(hm_ep_return_rows(ep, out, rows_used, vs));
      ok(hm_combine(retbuf, pos, w, T, Kp, H, cfg.residual ? x : nullptr, y, vs));
    } else if (W > 1 && ep) {  // combine + cross-rank sum + residual: one kernel over peer memory
      ok(hm_ep_combine_allreduce(ep, out, dv_h_out, zc_out && !cpu_refs.empty() ? host_mask : nullptr, pos, w, T, Kp,
                                 H, cfg.residual ? x : nullptr, y, nullptr, vs));
    } else if (W > 1) {
      HM_REQUIRE(y32 != nullptr, HM_EVALUE, "expert parallelism needs hm_runtime_set_ep_output");
      ok(hm_combine_f32(out, pos, w, T, Kp, H, y32, vs));  // partial; the caller all-reduces
    } else {
      ok(hm_combine(out, pos, w, T, Kp, H, cfg.residual ? x : nullptr, y, vs));
    }
    if (stats) *stats = s;
  }
};

}  // namespace hm

extern "C" {

int hm_runtime_create(const hm_runtime_config *cfg, hm_engine *engine, hm_runtime **out) {
  HM_API_BEGIN
  HM_REQUIRE(cfg && engine && out, HM_EVALUE, "null argument");
  *out = reinterpret_cast<hm_runtime *>(new hm::Runtime(*cfg, reinterpret_cast<hm::Engine *>(engine)));
  HM_API_END
}

void hm_runtime_destroy(hm_runtime *rt) { delete reinterpret_cast<hm::Runtime *>(rt); }

int hm_runtime_buffers(hm_runtime *rt, void **pool, void **host_store, size_t *slot_bytes, int64_t *n_slots) {
  HM_API_BEGIN
  auto *r = reinterpret_cast<hm::Runtime *>(rt);
  if (pool) *pool = r->pool;
  if (host_store) *host_store = r->store;
  if (slot_bytes) *slot_bytes = r->slot_bytes;
  if (n_slots) *n_slots = r->n_slots;
  HM_API_END
}

int hm_runtime_image_of(const hm_runtime *rt, int layer, int expert, int64_t *image) {
  HM_API_BEGIN
  *image = reinterpret_cast<const hm::Runtime *>(rt)->image_of(layer, expert);
  HM_API_END
}

int hm_runtime_shared_slot(const hm_runtime *rt, int layer, int chunk, int64_t *slot) {
  HM_API_BEGIN
  *slot = reinterpret_cast<const hm::Runtime *>(rt)->shared_slot(layer, chunk);
  HM_API_END
}

int hm_runtime_forward_layer(hm_runtime *rt, int layer, const uint16_t *x, const float *logits, int T, int ld,
                             uint16_t *y, const int32_t *pred_layers, const int64_t *pred_loads, int n_pred,
                             void *stream, hm_layer_stats *stats) {
  HM_API_BEGIN
  reinterpret_cast<hm::Runtime *>(rt)->forward_layer(layer, x, logits, T, ld, y, pred_layers, pred_loads, n_pred,
                                                    static_cast<cudaStream_t>(stream), stats);
  HM_API_END
}

int hm_runtime_forward_pass(hm_runtime *rt, const uint16_t *x, const float *const *logits, int T, int ld,
                            uint16_t *buf0, uint16_t *buf1, const int64_t *pass_loads, int64_t pass_index,
                            int64_t seed, int horizon, double accuracy, void *stream, hm_layer_stats *stats,
                            hm_pass_result *result, uint16_t **y_out) {
  HM_API_BEGIN
  auto *r = reinterpret_cast<hm::Runtime *>(rt);
  HM_REQUIRE(r->W == 1 || r->ep, HM_EVALUE,
             "expert-parallel passes need the peer-memory exchange (hm_runtime_set_ep_exchange) or forward_layer");
  const bool predicting = pass_loads != nullptr && r->engine->cfg.prefetch;
  const bool live = pass_loads == nullptr && r->engine->cfg.prefetch && r->la_gate != nullptr;
  std::vector<int32_t> pl(static_cast<size_t>(horizon > 0 ? horizon : 1));
  std::vector<int64_t> pload(static_cast<size_t>(horizon > 0 ? horizon : 1) * r->N);
  r->engine->begin_pass();
  const uint16_t *cur = x;
  for (int l = 0; l < r->L; ++l) {
    int n_pred = live ? HM_PREDICT_LIVE : 0;
    if (predicting) {
      const int rc = hm_predict_layers(pass_loads, r->L, r->N, pass_index, l, seed, horizon, accuracy, pl.data(),
                                       pload.data(), &n_pred);
      if (rc != HM_OK) hm::raise(rc, hm::last_error());
    }
    uint16_t *out = (l % 2 == 0) ? buf0 : buf1;
    r->forward_layer(l, cur, logits[l], T, ld, out, pl.data(), pload.data(), n_pred, static_cast<cudaStream_t>(stream),
                     stats ? &stats[l] : nullptr);
    cur = out;
  }
  r->engine->end_pass(result);
  if (y_out) *y_out = const_cast<uint16_t *>(cur);
  HM_API_END
}

int hm_runtime_last_request(const hm_runtime *rt, int64_t *loads, double *scores) {
  HM_API_BEGIN
  auto *r = reinterpret_cast<const hm::Runtime *>(rt);
  for (int e = 0; e < r->N; ++e) {
    if (loads) loads[e] = r->loads[e];
    if (scores) scores[e] = r->scores[e];
  }
  HM_API_END
}

int hm_runtime_device_mrs(hm_runtime *rt, double *host_out) {
  HM_API_BEGIN
  auto *r = reinterpret_cast<hm::Runtime *>(rt);
  RT_CUDA(cudaDeviceSynchronize());
  HM_REQUIRE(r->engine->mrs_ != nullptr, HM_EVALUE, "the runtime's engine has no MRS table");
  RT_CUDA(cudaDeviceSynchronize());
  std::memcpy(host_out, r->engine->mrs_->S.data(), r->engine->mrs_->S.size() * 8);
  HM_API_END
}

int hm_runtime_preload(hm_runtime *rt, const uint32_t *refs, int n) {
  HM_API_BEGIN
  auto *r = reinterpret_cast<hm::Runtime *>(rt);
  for (int i = 0; i < n; ++i) {
    hm::Cache &c = r->engine->cache;
    if (!c.is_resident(refs[i])) c.add_resident(refs[i]);
    const int64_t slot = c.resident.at(refs[i]).slot;
    HM_REQUIRE(slot >= 0 && slot < r->cfg.capacity, HM_EVALUE, "no free HBM slot to preload into");
    r->issue_copy(refs[i], slot, nullptr);
  }
  RT_CUDA(cudaStreamSynchronize(r->copy));
  HM_API_END
}

int hm_runtime_set_ep_output(hm_runtime *rt, float *y32) {
  HM_API_BEGIN
  reinterpret_cast<hm::Runtime *>(rt)->y32 = y32;
  HM_API_END
}

int hm_runtime_set_lookahead(hm_runtime *rt, const uint16_t *gate_w, int ld, int horizon) {
  HM_API_BEGIN
  auto *r = reinterpret_cast<hm::Runtime *>(rt);
  HM_REQUIRE(gate_w == nullptr || (ld >= r->N && horizon >= 0 && r->H % 8 == 0 && r->N <= 256), HM_EVALUE,
             "look-ahead gate shape out of range");
  RT_CUDA(cudaDeviceSynchronize());
  if (r->la_counts) cudaFree(r->la_counts);
  if (r->la_host) cudaFreeHost(r->la_host);
  r->la_counts = nullptr;
  r->la_host = r->la_dv = nullptr;
  r->la_gate = gate_w;
  r->la_ld = ld;
  r->la_hz = gate_w ? horizon : 0;
  const size_t n = static_cast<size_t>(std::max(1, r->la_hz)) * r->N;
  if (gate_w) {
    RT_CUDA(cudaMalloc(&r->la_counts, n * 4));
    RT_CUDA(cudaHostAlloc(&r->la_host, n * 8, cudaHostAllocMapped));
    RT_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void **>(&r->la_dv), r->la_host, 0));
    r->la_layers.assign(std::max(1, r->la_hz), 0);
  }
  HM_API_END
}

int hm_runtime_set_ep_dispatch(hm_runtime *rt, hm_ep *ep) {
  HM_API_BEGIN
  auto *r = reinterpret_cast<hm::Runtime *>(rt);
  HM_REQUIRE(ep && hm_ep_world(ep) == r->W, HM_EVALUE,
             "token-sharded dispatch needs an exchange of the runtime's ep_world (1 exercises it on one rank)");
  uint16_t *xr = nullptr;
  float *rb = nullptr;
  const int rc = hm_ep_dispatch_buffers(ep, &xr, &rb);
  if (rc != HM_OK) hm::raise(rc, hm::last_error());
  if (!r->lcounts) {
    RT_CUDA(cudaMalloc(&r->lcounts, (2 * static_cast<size_t>(r->E) + 1) * 4));
    r->loffsets = r->lcounts + r->E;
    RT_CUDA(cudaMalloc(&r->lsums, static_cast<size_t>(r->N) * 8));
  }
  r->ep = ep;
  r->xrecv = xr;
  r->retbuf = rb;
  r->disp = true;
  HM_API_END
}

int hm_runtime_set_ep_exchange(hm_runtime *rt, hm_ep *ep) {
  HM_API_BEGIN
  reinterpret_cast<hm::Runtime *>(rt)->ep = ep;
  HM_API_END
}

int hm_runtime_set_kernel_timing(hm_runtime *rt, int on) {
  HM_API_BEGIN
  auto *r = reinterpret_cast<hm::Runtime *>(rt);
  r->time_kernels = on != 0;
  r->kused = 0;
  HM_API_END
}

int hm_runtime_set_copy_timing(hm_runtime *rt, int on) {
  HM_API_BEGIN
  auto *r = reinterpret_cast<hm::Runtime *>(rt);
  r->time_copies = on != 0;
  r->cused = 0;
  HM_API_END
}

int hm_runtime_copy_times(hm_runtime *rt, double *total_ms, int64_t *total_bytes, int64_t *n, double *max_ms) {
  HM_API_BEGIN
  auto *r = reinterpret_cast<hm::Runtime *>(rt);
  RT_CUDA(cudaStreamSynchronize(r->copy));
  double tot = 0.0, mx = 0.0;
  for (size_t i = 0; i < r->cused; ++i) {
    float ms = 0.f;
    RT_CUDA(cudaEventElapsedTime(&ms, r->cev[i].first, r->cev[i].second));
    tot += ms;
    mx = ms > mx ? ms : mx;
  }
  if (total_ms) *total_ms = tot;
  if (total_bytes) *total_bytes = static_cast<int64_t>(r->cused) * static_cast<int64_t>(r->slot_bytes);
  if (n) *n = static_cast<int64_t>(r->cused);
  if (max_ms) *max_ms = mx;
  r->cused = 0;
  HM_API_END
}

int hm_runtime_kernel_times(hm_runtime *rt, double *total_ms, int64_t *total_bytes, int64_t *n, double *max_ms) {
  HM_API_BEGIN
  auto *r = reinterpret_cast<hm::Runtime *>(rt);
  double tot = 0.0, mx = 0.0;
  int64_t by = 0;
  for (size_t i = 0; i < r->kused; ++i) {
    RT_CUDA(cudaEventSynchronize(r->kev[i].second));
    float ms = 0.f;
    RT_CUDA(cudaEventElapsedTime(&ms, r->kev[i].first, r->kev[i].second));
    tot += ms;
    mx = ms > mx ? ms : mx;
    by += r->kbytes[i];
  }
  if (total_ms) *total_ms = tot;
  if (total_bytes) *total_bytes = by;
  if (n) *n = static_cast<int64_t>(r->kused);
  if (max_ms) *max_ms = mx;
  r->kused = 0;
  HM_API_END
}

int hm_runtime_sync(hm_runtime *rt) {
  HM_API_BEGIN
  auto *r = reinterpret_cast<hm::Runtime *>(rt);
  RT_CUDA(cudaStreamSynchronize(r->copy));
  HM_API_END
}

}  // extern "C"
