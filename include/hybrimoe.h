/*
 * hybrimoe.h -- C ABI of the B200-native HybriMoE MoE-layer hot path.
 *
 * The reference (`moesim`, /root/reference/pkg/src/moesim) is a pure-Python
 * function API with no FFI; every entry point below replaces one reference
 * function (cited as file:line) and is bound from Python with ctypes by
 * paper_2504_05897_b200/_lib.py.  Conventions:
 *
 *   - every function returns an int status: HM_OK or one of HM_E*;
 *     the message of the last failure on the calling thread is available
 *     through hm_last_error();
 *   - caller-owned flat arrays, opaque handles, no C++ exceptions cross the
 *     ABI, no hidden device synchronisation;
 *   - an ExpertRef (core.py:27-36) is packed as uint32 (layer << 16 | expert)
 *     so that integer order equals the reference's lexicographic tuple order;
 *   - all decision arithmetic is IEEE fp64 evaluated in the reference's
 *     expression order (the library is built with -ffp-contract=off);
 *   - device entry points take a cudaStream_t (passed as void*).
 */
#ifndef HYBRIMOE_H_
#define HYBRIMOE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: map 1:1 onto the reference's exception types ---------- */
#define HM_OK 0
#define HM_EVALUE 1        /* ValueError            (costs.py:70, scheduling.py:169, caching.py:115, prefetch.py:130) */
#define HM_EEVICTION 2     /* EvictionError         (caching.py:26, 96-99) */
#define HM_EPLAN 3         /* PlanInvariantError    (scheduling.py:76-124) */
#define HM_ERUNTIME 4      /* RuntimeError          (scheduling.py:233-234, "scheduler stalled") */
#define HM_ECALIBRATION 5  /* CalibrationError      (costs.py:98) */
#define HM_EASSERT 6       /* AssertionError        (engine.py:373-381, validate replan) */
#define HM_ECUDA 7         /* CUDA runtime failure (no reference counterpart) */

/* devices / kinds / assignments (scheduling.py:33-45) */
#define HM_DEV_CPU 0
#define HM_DEV_GPU 1
#define HM_DEV_PCIE 2
#define HM_KIND_COMPUTE 0
#define HM_KIND_TRANSFER 1
#define HM_ASSIGN_CPU 0
#define HM_ASSIGN_GPU_CACHED 1
#define HM_ASSIGN_GPU_TRANSFER 2

/* cache policies (caching.py:20-23) */
#define HM_POLICY_MRS 0
#define HM_POLICY_LRU 1
#define HM_POLICY_LFU 2

/* scheduling policies (engine.py:66-70) */
#define HM_SCHED_HYBRID 0
#define HM_SCHED_STATIC_SPLIT 1
#define HM_SCHED_FIXED_MAP 2
#define HM_SCHED_GPU_ONDEMAND 3

/* HardwareProfile (costs.py:33-65), field for field. */
typedef struct hm_profile {
  double gpu_time_per_expert;
  double cpu_slope;
  double transfer_bandwidth;
  double transfer_latency;
  int64_t gpu_saturation_load;
  double gpu_slope;
  double cpu_first_expert_penalty;
  double shared_expert_time;
  double non_expert_time;
} hm_profile;

/* ExpertTask (scheduling.py:48-50) */
typedef struct hm_task {
  uint32_t ref;
  int32_t _pad;
  int64_t load;
} hm_task;

/* TimelineEvent (scheduling.py:53-58) */
typedef struct hm_event {
  int32_t device;
  int32_t kind;
  uint32_t ref;
  int32_t _pad;
  double start;
  double end;
} hm_event;

/* one SchedulePlan.assignment entry (scheduling.py:62-67) */
typedef struct hm_assign {
  uint32_t ref;
  int32_t how;
} hm_assign;

/* PrefetchCandidate (prefetch.py:45-51) */
typedef struct hm_candidate {
  uint32_t ref;
  int32_t layer_distance;
  int64_t predicted_load;
  double gain;
  double cost;
} hm_candidate;

typedef struct hm_cache hm_cache;         /* CacheState (core.py:235-265) + HBM slot map */
typedef struct hm_mrs hm_mrs;             /* MrsState (caching.py:30-55) */
typedef struct hm_evaluator hm_evaluator; /* MakespanEvaluator (scheduling.py:433-465) */
typedef struct hm_engine hm_engine;       /* run_pass state machine (engine.py:255-398) */

/* Message of the last failing call on this thread; returns its length. */
int hm_last_error(char *buf, size_t n);
/* Library version string. */
const char *hm_version(void);

/* ---- cost model (costs.py:68-95) ------------------------------------------ */
int hm_profile_check(const hm_profile *p);                                    /* costs.py:47-65 */
int hm_gpu_time(const hm_profile *p, int64_t load, double *out);              /* costs.py:68-74 */
int hm_cpu_time(const hm_profile *p, int64_t load, int64_t pos, double *out); /* costs.py:77-88 */
int hm_transfer_time(const hm_profile *p, double expert_bytes, double *out);  /* costs.py:91-95 */

/* ---- intra-layer scheduler (scheduling.py) -------------------------------- */
/* Output buffers: events[2*n], assign[n]; n = total task count. */
int hm_simulate_schedule(const hm_task *gpu_q, int n_gpu, const hm_task *cpu_q, int n_cpu,
                         const hm_profile *p, double expert_bytes, hm_event *events,
                         int *n_events, hm_assign *assign, int *n_assign,
                         double *makespan); /* scheduling.py:160-270 */
int hm_plan_all_cpu(const hm_task *tasks, int n, const hm_profile *p, hm_event *events,
                    int *n_events, hm_assign *assign, int *n_assign,
                    double *makespan); /* scheduling.py:273-284 */
int hm_plan_all_gpu(const hm_task *cached, int n_cached, const hm_task *uncached,
                    int n_uncached, const hm_profile *p, double expert_bytes,
                    hm_event *events, int *n_events, hm_assign *assign, int *n_assign,
                    double *makespan); /* scheduling.py:287-317 */
int hm_select_plan_tasks(const hm_task *cached, int n_cached, const hm_task *uncached,
                         int n_uncached, const hm_profile *p, double expert_bytes,
                         hm_event *events, int *n_events, hm_assign *assign,
                         int *n_assign, double *makespan); /* scheduling.py:320-335 */
/* select_plan against a native cache: build_queues + _select_plan_tasks. */
int hm_select_plan(const hm_cache *c, int layer, const int64_t *loads, int n,
                   const hm_profile *p, double expert_bytes, hm_event *events,
                   int *n_events, hm_assign *assign, int *n_assign,
                   double *makespan); /* scheduling.py:135-147, 338-350 */
int hm_check_plan(const hm_event *events, int n_events, const hm_assign *assign,
                  int n_assign, double makespan); /* scheduling.py:80-124 */
int hm_pcie_idle_budget(const hm_event *events, int n_events, double makespan,
                        double *out); /* scheduling.py:405-412 */
int hm_oracle_optimal(const hm_task *tasks, int n, const uint8_t *cached,
                      const hm_profile *p, double expert_bytes, int limit,
                      double *out); /* scheduling.py:356-402 */

/* ---- memoised makespans (scheduling.py:433-465) --------------------------- */
int hm_evaluator_create(const hm_profile *p, double expert_bytes, hm_evaluator **out);
void hm_evaluator_destroy(hm_evaluator *e);
int hm_evaluator_makespan(hm_evaluator *e, const int64_t *cached_loads, int n_cached,
                          const int64_t *uncached_loads, int n_uncached, double *out);
int hm_evaluator_size(const hm_evaluator *e, int64_t *out);

/* ---- cache container + policies (core.py:235-265, caching.py:79-128) ------ */
int hm_cache_create(int64_t capacity, hm_cache **out);
void hm_cache_destroy(hm_cache *c);
int hm_cache_capacity(const hm_cache *c, int64_t *out);
int hm_cache_lookup(hm_cache *c, uint32_t ref, int policy, int *hit); /* caching.py:79-91 */
int hm_cache_insert(hm_cache *c, uint32_t ref, int policy, const hm_mrs *mrs,
                    uint32_t *victim, int *has_victim); /* caching.py:111-128 */
int hm_cache_victim(const hm_cache *c, int policy, const hm_mrs *mrs,
                    uint32_t *victim); /* caching.py:94-108 */
int hm_cache_is_resident(const hm_cache *c, uint32_t ref, int *out);
int hm_cache_is_pinned(const hm_cache *c, uint32_t ref, int *out);
int hm_cache_pin(hm_cache *c, uint32_t ref);
int hm_cache_unpin(hm_cache *c, uint32_t ref);
int hm_cache_clear_pinned(hm_cache *c);
int hm_cache_add_resident(hm_cache *c, uint32_t ref);  /* set-like add, no policy metadata */
int hm_cache_remove_resident(hm_cache *c, uint32_t ref);
int hm_cache_clear_resident(hm_cache *c);
int hm_cache_counts(const hm_cache *c, int64_t *n_resident, int64_t *n_pinned);
/* Copy out members (unordered); *n receives the total even if cap is short. */
int hm_cache_resident(const hm_cache *c, uint32_t *out, int64_t cap, int64_t *n);
int hm_cache_pinned(const hm_cache *c, uint32_t *out, int64_t cap, int64_t *n);
/* LRU tick / LFU frequency metadata (core.py:253-259); has=0 when absent. */
int hm_cache_last_access(const hm_cache *c, uint32_t ref, int64_t *out, int *has);
int hm_cache_frequency(const hm_cache *c, uint32_t ref, int64_t *out, int *has);
int hm_cache_set_last_access(hm_cache *c, uint32_t ref, int64_t v);
int hm_cache_set_frequency(hm_cache *c, uint32_t ref, int64_t v);
int hm_cache_tick(const hm_cache *c, int64_t *out);
int hm_cache_next_tick(hm_cache *c, int64_t *out);
/* HBM slot of a resident expert (runtime extension: which slot its weights occupy). */
int hm_cache_slot(const hm_cache *c, uint32_t ref, int64_t *slot);

/* ---- MRS score table (caching.py:30-76) ----------------------------------- */
int hm_mrs_create(int num_layers, int num_routed, double alpha, int p, hm_mrs **out);
void hm_mrs_destroy(hm_mrs *m);
int hm_mrs_update(hm_mrs *m, int layer, const double *scores, int n); /* caching.py:65-76 */
int hm_mrs_get(const hm_mrs *m, uint32_t ref, double *out);
int hm_mrs_set(hm_mrs *m, uint32_t ref, double v);
int hm_mrs_table(const hm_mrs *m, double *out); /* L*N fp64, row-major by layer */
int hm_mrs_params(const hm_mrs *m, double *alpha, int *p, int *num_layers, int *num_routed);
int hm_top_p_filter(const double *scores, int n, int p, double *out); /* caching.py:58-62 */

/* ---- prefetch (prefetch.py:104-143) --------------------------------------- */
/* gain of making `candidate` resident for the predicted layer request. */
int hm_evaluate_gain(uint32_t candidate, int pred_layer, const int64_t *pred_loads, int n,
                     const hm_cache *c, hm_evaluator *ev, double *gain);
int hm_select_prefetches(const hm_candidate *cands, int n, double idle_budget,
                         uint32_t *chosen, int *n_chosen);

/* The prediction model (prefetch.py:54-101) natively: numpy's
 * default_rng([seed, pass, layer, 0x5EED]) stream (SeedSequence + PCG64,
 * random(), integers()) restated draw for draw.  pass_loads [L*N]; writes the
 * predicted loads of layers layer+1..min(layer+horizon, L-1). */
int hm_predict_layers(const int64_t *pass_loads, int L, int N, int64_t pass_index, int layer,
                      int64_t seed, int horizon, double accuracy, int32_t *out_layers,
                      int64_t *out_loads, int *n_out);

/* ---- the per-layer engine step (engine.py:255-398, 401-486) --------------- */
typedef struct hm_engine_config {
  int32_t num_layers;
  int32_t num_routed;
  int32_t num_activated;
  int32_t scheduling;   /* HM_SCHED_* */
  int32_t cache_policy; /* HM_POLICY_* */
  int32_t prefetch;     /* bool */
  int32_t validate;     /* bool */
  int32_t split_point;  /* static_layer_split */
  int64_t capacity;     /* cache slots = floor(ratio * L * N) */
  double expert_bytes;  /* core.py:84-91 */
  int32_t collect;      /* keep the per-layer decision record */
  int32_t _pad;
} hm_engine_config;

/* PassResult (engine.py:159-168) plus the prefetch counters. */
typedef struct hm_pass_result {
  double latency;
  double busy[3]; /* indexed by HM_DEV_* */
  int64_t lookups, hits, inserts, evictions;
  int64_t prefetch_issued, prefetch_hits, prefetch_expired;
} hm_pass_result;

/* The engine borrows the run's cache, MRS state (may be NULL, as in the
 * reference) and evaluator, which must outlive it (engine.py:255-265). */
int hm_engine_create(const hm_engine_config *cfg, const hm_profile *p, hm_cache *cache,
                     hm_mrs *mrs, hm_evaluator *ev, hm_engine **out);
void hm_engine_destroy(hm_engine *e);
/* fixed_frequency_map GPU set (engine.py:195-231); residency is the caller's. */
int hm_engine_set_fixed_pinned(hm_engine *e, const uint32_t *refs, int n);
/* Replace the profile between passes (stage-calibrated profiles: a decode
 * profile and a prefill profile); also resets the evaluator's memo. */
int hm_engine_set_profile(hm_engine *e, const hm_profile *p);
int hm_engine_begin_pass(hm_engine *e);
/* One layer of run_pass in the exact engine.py:288-389 order.  `pred_*` are
 * the predicted future LayerRequests (prefetch.py:54-101), concatenated:
 * pred_layers[n_pred], pred_loads[n_pred*N]; ignored unless prefetch is on. */
int hm_engine_run_layer(hm_engine *e, int layer, const int64_t *loads, const double *scores,
                        int n, const int32_t *pred_layers, const int64_t *pred_loads,
                        int n_pred);
/* End-of-pass expiry (engine.py:392-395) and PassResult. */
int hm_engine_end_pass(hm_engine *e, hm_pass_result *out);
/* Makespan of every layer run in the current pass. */
int hm_engine_layer_makespans(const hm_engine *e, double *out, int cap, int *n);

/* Decision record of the last run layer (valid when cfg.collect or always for
 * the plan).  Sizes first, then the arrays. */
typedef struct hm_layer_record_sizes {
  int32_t n_lookups;
  int32_t n_events;
  int32_t n_assign;
  int32_t n_demand;
  int32_t n_candidates;
  int32_t n_chosen;
  int32_t expired;
  int32_t n_selected;           /* select_prefetches output length */
  int32_t prefetch_evict_error; /* a prefetch insert raised EvictionError */
  int32_t _pad;
  double makespan;
  double budget;
} hm_layer_record_sizes;
int hm_engine_record_sizes(const hm_engine *e, hm_layer_record_sizes *out);
int hm_engine_record(const hm_engine *e, uint32_t *lookup_refs, uint8_t *lookup_hits,
                     hm_event *events, hm_assign *assign, uint32_t *demand_refs,
                     uint32_t *demand_victims, uint8_t *demand_has_victim,
                     hm_candidate *candidates, uint32_t *chosen_refs,
                     uint32_t *chosen_victims, uint8_t *chosen_has_victim,
                     uint32_t *selected_refs);

/* ======================================================================= */
/* Device side (CUDA, sm_100a).  Pointers are device pointers unless noted; */
/* `stream` is a cudaStream_t.  No entry point synchronises the device.      */
/* ======================================================================= */

/* Router (Eq. 1; tracegen.py:137-152; transformers mixtral /
 * deepseek_v2 / qwen2_moe routers).  logits [T, ld] fp32, routed experts in
 * columns [0, N).  Per token: softmax over the N routed logits, top-K by
 * (logit desc, expert index asc) -- the reference's tie rule (core.py:94-97)
 * -- combine weight = probability, renormalised over the K when `renormalize`.
 * Shared experts are appended as always-selected columns N..N+n_shared-1
 * with weight 1, or sigmoid(logits[t, shared_gate_col]) when that is >= 0.
 * Outputs: sel/w [T, K+n_shared], probs [T, N] (routed softmax),
 * counts [N+n_shared] (bincount, tracegen.py:148; zeroed here). */
int hm_router_topk(const float *logits, int T, int N, int ld, int K, int renormalize,
                   int n_shared, int shared_gate_col, int32_t *sel, float *w, float *probs,
                   int32_t *counts, void *stream);
/* Decode-sized layers in one launch (T <= 32, T*(K+S) <= 1024): router,
 * counts, offsets, fp64 score sums, normalised scores, permutation and row
 * gather.  meta_i = [counts E | offsets E+1], meta_d = [score_sum N | scores N]
 * where scores[e] = score_sum[e] / sum_e score_sum (sequential fp64 sums). */
int hm_router_fused_small(const float *logits, int T, int N, int ld, int K, int renormalize,
                          int n_shared, int shared_gate_col, const uint16_t *x, int H, int32_t *sel,
                          float *w, int32_t *pos, int32_t *row_src, uint16_t *xp, int32_t *meta_i,
                          double *meta_d, void *stream);
/* hm_router_fused_small plus a mirror in mapped pinned host memory (device
 * views of cudaHostAlloc(..., cudaHostAllocMapped) buffers): the meta block,
 * optionally the routed rows of xp (host_xp may be NULL; with T == 1 only row
 * 0 -- every routed row is that token), then *host_flag =
 * seq after a system-scope fence -- the host spins on the flag instead of a
 * D2H copy + event wait (the LayerRequest hand-off of engine.py:288-306). */
int hm_router_fused_mirror(const float *logits, int T, int N, int ld, int K, int renormalize,
                           int n_shared, int shared_gate_col, const uint16_t *x, int H, int32_t *sel,
                           float *w, int32_t *pos, int32_t *row_src, uint16_t *xp, int32_t *meta_i,
                           double *meta_d, int32_t *host_meta_i, double *host_meta_d,
                           uint16_t *host_xp, uint32_t *host_flag, uint32_t seq, void *stream);
/* score_sum[e] = sum_t probs[t, e] in fp64, fixed reduction order; the
 * LayerRequest scores are score_sum normalised (tracegen.py:149-150). */
int hm_score_sums(const float *probs, int T, int N, double *score_sum, void *stream);
/* Gate GEMV/GEMM: logits[T, N] = x[T, H] . wg[N, H]^T (bf16 in, fp32 out). */
int hm_router_logits(const uint16_t *x, const uint16_t *wg, int T, int H, int N,
                     float *logits, void *stream);
/* Exclusive scan: offsets[E+1] from counts[E]. */
int hm_offsets(const int32_t *counts, int E, int32_t *offsets, void *stream);
/* Expert-contiguous permutation of the T*Kp selections (token order inside
 * an expert): pos[t*Kp+k] = permuted row, row_src[row] = t*Kp+k. */
int hm_permute(const int32_t *sel, int T, int Kp, int E, const int32_t *offsets,
               int32_t *pos, int32_t *row_src, void *stream);
/* xp[r, :] = x[row_src[r] / Kp, :] */
int hm_gather_rows(const uint16_t *x, const int32_t *row_src, int rows, int Kp, int H,
                   uint16_t *xp, void *stream);

/* Expert weight pool: n_slots expert images of 3*H*I bf16 each --
 *   [0, 2IH)   W13: gate/up rows interleaved in 128-row blocks,
 *   [2IH, 3IH) W2 [H, I] row-major.
 * One group = one expert applied to a contiguous range of permuted rows. */
typedef struct hm_group {
  int32_t slot;
  int32_t row_begin;
  int32_t row_count;
  int32_t _pad;
} hm_group;
#define HM_FFN_AUTO 0 /* <= 4 rows: weight-streaming GEMV; larger: tcgen05 GEMM */
#define HM_FFN_GEMV 1
#define HM_FFN_GEMM 2
#define HM_FFN_GEMV_SPLIT 3 /* the two-launch ffn1 -> ffn2 GEMV pair, whatever HM_GEMV_FUSED says */
#define HM_FFN_GEMV_FUSED 4 /* the persistent one-launch ffn1 -> ffn2 GEMV (measured slower; A/B) */
#define HM_FFN_GEMV_BULK 5  /* the ffn1 -> ffn2 pair with weights staged by the bulk-copy engine */
/* out[rows of g] = W2_g (silu(Wg_g x) * (Wu_g x)) for every group (groups is
 * a HOST array).  h [total_rows, I] bf16 scratch, out [total_rows, H] fp32. */
int hm_expert_ffn(const uint16_t *pool, int n_slots, int H, int I, const hm_group *groups,
                  int n_groups, const uint16_t *xp, int total_rows, uint16_t *h, float *out,
                  int path, void *stream);
/* ---- 4-bit experts (bytes_per_weight 0.5, core.py:55; Marlin,
 * PAPER.md:217).  Weight-only int4, symmetric, one bf16 scale per 128 weights
 * of a row: w = (nibble - 8) * scale.  Image: W13 nibbles [2I][H/2] | W2
 * nibbles [H][I/2] | W13 scales [2I][H/128] | W2 scales [H][I/128], rows in the
 * bf16 image's order; hm_q4_image_bytes gives its size. */
int hm_q4_image_bytes(int H, int I, size_t *bytes);
/* bf16 image (device) -> 4-bit image (device): per (row, 128 weights)
 * scale = bf16(max|w| / 7), nibble = 8 + clamp(rint(w / scale), -8, 7). */
int hm_q4_quantize(const uint16_t *bf16_image, int H, int I, uint8_t *q4_image, void *stream);
int hm_q4_dequantize(const uint8_t *q4_image, int H, int I, uint16_t *bf16_image, void *stream);
/* hm_expert_ffn over a pool of 4-bit images (slot_bytes apart): decode groups
 * (<= 4 rows) on the int4 weight-streaming GEMV; larger groups dequantized into
 * `scratch` (n_scratch bf16 images) and run on the tcgen05 GEMM. */
int hm_expert_ffn_q4(const uint8_t *pool, size_t slot_bytes, int n_slots, int H, int I,
                     const hm_group *groups, int n_groups, const uint16_t *xp, int total_rows,
                     uint16_t *h, float *out, uint16_t *scratch, int n_scratch, int path,
                     void *stream);
/* Micro-benchmark: `reps` back-to-back hm_expert_ffn calls from the library
 * (n_groups experts x rows_per_group rows, slots rotating mod n_slots), timed
 * with events on `stream`; *ms = milliseconds per call. */
int hm_bench_expert_ffn(const uint16_t *pool, int n_slots, int H, int I, int n_groups,
                        int rows_per_group, const uint16_t *xp, uint16_t *h, float *out, int path,
                        int reps, void *stream, float *ms);
/* Pure streaming-read floor: back-to-back launches reading `bytes` each from
 * n_buf rotating buffers at `base` (pair != 0: two dependent launches of 2/3 and
 * 1/3 of the bytes, the ffn1/ffn2 split); *ms = milliseconds per launch (pair).
 * The per-size denominator of the decode GEMV's efficiency. */
int hm_bench_stream_read(const void *base, size_t bytes, int n_buf, int pair, int blocks_per_sm, int reps,
                         void *stream, float *ms);
/* y[t] = residual[t] (optional) + sum_k w[t,k] * out[pos[t,k]]  (Eq. 1 combine). */
int hm_combine(const float *out, const int32_t *pos, const float *w, int T, int Kp, int H,
               const uint16_t *residual, uint16_t *y, void *stream);
/* Expert parallelism helpers: zero the combine weight of every selection whose
 * expert is not homed on `rank` (routed e: e % world; shared column N+c:
 * c % world); fp32 combine without residual; y = bf16(residual + y32). */
int hm_mask_nonhome(const int32_t *sel, float *w, int TKp, int N, int rank, int world,
                    void *stream);
int hm_combine_f32(const float *out, const int32_t *pos, const float *w, int T, int Kp, int H,
                   float *y32, void *stream);
int hm_residual_add(const float *y32, const uint16_t *residual, int T, int H, uint16_t *y,
                    void *stream);
/* Number of kernels this library has launched so far (process-wide). */
long long hm_launch_count(void);
/* GPU-side MRS update (caching.py:58-76): S[layer] <- a*TopP(s) + (1-a)*S[layer],
 * fp64 with explicit round-to-nearest mul/add (bit-identical to the host core). */
int hm_mrs_update_dev(double *S, const double *scores, int layer, int N, int p,
                      double alpha, void *stream);
/* Live look-ahead prediction: for future layers
 * first_layer .. first_layer+hz-1, the gate rows gate_w[layer][0..N) (bf16,
 * [L][ld][H]) applied to the current hidden state x [T, H] and counted through
 * the router's top-K rule -> counts [hz][N] int32 (device); host_counts (device
 * view of mapped memory, int64 [hz][N], optional) receives a fenced copy. */
int hm_lookahead(const uint16_t *x, const uint16_t *gate_w, int first_layer, int hz, int T, int N,
                 int ld, int K, int H, int32_t *counts, int64_t *host_counts, void *stream);
/* Hold `stream` until the host stores `seq` into *flag (device view of mapped
 * pinned memory): lets CUDA events time a group of kernels without the host's
 * launch latency in between (kernel-timing mode of the runtime). */
int hm_gate_wait(const uint32_t *flag, uint32_t seq, void *stream);
/* Decode tail in one launch: hm_combine (Eq. 1 + residual) where positions
 * whose bit is set in host_mask4 (4 x 64 bits, positions < 256; NULL = none)
 * are read zero-copy from host_out (device view of the host worker's mapped
 * output rows), plus, when S != NULL, hm_mrs_update_dev for `layer` (N <= 256). */
int hm_combine_tail(const float *out, const float *host_out, const uint64_t *host_mask4,
                    const int32_t *pos, const float *w, int T, int Kp, int H,
                    const uint16_t *residual, uint16_t *y, double *S, const double *scores, int layer,
                    int N, int p, double alpha, void *stream);

/* ======================================================================= */
/* Host worker (AVX-512 BF16) and the layer executor.                        */
/* ======================================================================= */
typedef struct hm_cpu_pool hm_cpu_pool;
int hm_cpu_pool_create(int nthreads, hm_cpu_pool **out); /* nthreads <= 0: all cores */
void hm_cpu_pool_destroy(hm_cpu_pool *p);
/* out[M, H] fp32 = expert(img)(x[M, H] bf16) on the host; img in slot layout (HOST pointers). */
int hm_cpu_expert(hm_cpu_pool *pool, const uint16_t *img, int H, int I, const uint16_t *x, int M,
                  float *out);
/* 4-bit expert images on the host worker (same rules as hm_cpu_expert). */
int hm_cpu_expert_q4(hm_cpu_pool *pool, const uint8_t *img, int H, int I, const uint16_t *x, int M,
                     float *out);
int hm_cpu_experts_decode_q4(hm_cpu_pool *pool, const uint8_t *const *imgs, const uint16_t *const *xs,
                             int n, int H, int I, float *const *outs);
int hm_cpu_has_avx512bf16(void);
int hm_cpu_has_amx_bf16(void); /* AMX-BF16 present and XTILEDATA granted */
/* Decode-stream tuning: software prefetch distance (elements) and hint (0 none, 1 T0, 2 T1, 3 NTA). */
int hm_cpu_set_prefetch(int dist, int hint);
/* n single-token experts in one worker pass (decode): outs[i][H] = expert(imgs[i])(xs[i][H]). */
/* n multi-token experts (prefill groups, Ms[e] >= 1 tokens each) in one host-worker pass on AMX; outputs
 * equal hm_cpu_expert's per expert (same per-unit arithmetic). */
int hm_cpu_experts_amx(hm_cpu_pool *pool, const uint16_t *const *imgs, const uint16_t *const *xs, const int *Ms,
                       int n, int H, int I, float *const *outs);
int hm_cpu_experts_decode(hm_cpu_pool *pool, const uint16_t *const *imgs, const uint16_t *const *xs, int n,
                          int H, int I, float *const *outs);
/* Best-of-reps host DRAM read bandwidth (GB/s) over `bytes` at p (64-byte aligned). */
/* Decode split granularity in gate/up pairs (0: whole 128-pair blocks); tuning knob. */
int hm_cpu_set_decode_grain(int grain);
/* Decode work balancing: threads that finish their own contiguous range take
 * chunks from the tails of the others' (default on; 0 = static ranges, A/B). */
int hm_cpu_set_decode_steal(int on);
/* Tool hook: enable per-thread phase timestamps of hm_cpu_experts_decode and
 * copy the last call's [thread][start, phase 1 done, barrier passed, phase 2
 * done] (ns since the call) into out. */
int hm_cpu_decode_profile(int enable, int64_t *out, int n_threads);
/* Tool hook: sums over the decode calls made while profiling is enabled --
 * [calls, max worker start (tid >= 1), caller start, max phase-1 end, barrier
 * passed, max phase-2 end, wall] in ns since each call; reset != 0 zeroes them. */
int hm_cpu_decode_profile_accum(int64_t *out7, int reset);
/* Tool hook: histogram of the per-call worker-start delay (<= 5, 20, 100, 1000,
 * > 1000 us) and, per thread, how often it was the slowest to start. */
int hm_cpu_decode_profile_hist(int64_t *out5, int64_t *slowest, int n_threads);
int hm_host_read_bw(hm_cpu_pool *pool, const void *p, size_t bytes, int reps, double *gbs);

typedef struct hm_runtime hm_runtime;
typedef struct hm_runtime_config {
  int32_t num_layers;
  int32_t num_routed;
  int32_t num_activated;
  int32_t hidden;
  int32_t inter;
  int32_t n_shared;        /* always-resident shared-expert chunks per layer (routed dims) */
  int32_t renormalize;     /* renormalise the top-K weights (Mixtral) */
  int32_t shared_gate_col; /* logits column of the Qwen2 shared-expert gate, -1 if none */
  int64_t capacity;        /* routed-expert HBM cache slots = floor(ratio * L * N) */
  int64_t host_images;     /* distinct expert images in the pinned master store */
  int32_t cpu_threads;     /* host worker threads (<= 0: all cores) */
  int32_t max_tokens;      /* largest T of one forward_layer call */
  int32_t gpu_mrs;         /* zero-copy decode: the router computes the layer's new MRS row on the GPU
                              (old row read from the engine's mapped table); the decision core takes it
                              at step (5) instead of its own recurrence */
  int32_t residual;        /* y = x + MoE(x) (1) or y = MoE(x) (0) */
  int32_t ep_rank;         /* expert parallelism: this rank computes experts e with  */
  int32_t ep_world;        /* e % ep_world == ep_rank (shared chunk c: c % ep_world) */
  int32_t weight_bits;     /* 16 (or 0): bf16 expert images; 4: 4-bit images (hm_q4_*) */
  int32_t _pad;
} hm_runtime_config;

typedef struct hm_layer_stats {
  double makespan_planned; /* the plan's makespan (profile units) */
  double t_wait_router_us; /* host wait for the router's LayerRequest */
  double t_decide_us;      /* decision core time */
  double t_cpu_us;         /* host worker time */
  int32_t n_gpu, n_cpu, n_transfer, n_prefetch;
  int64_t bytes_gpu, bytes_cpu, bytes_h2d; /* expert weight bytes per resource */
} hm_layer_stats;

/* The runtime drives `engine` (created with the same shape and capacity); it
 * owns the HBM slot pool (capacity + L*n_shared slots), the pinned master
 * store (host_images expert images; expert (l, e) uses image (l*N+e) mod
 * host_images), a copy stream, per-slot events and the host worker pool. */
int hm_runtime_create(const hm_runtime_config *cfg, hm_engine *engine, hm_runtime **out);
void hm_runtime_destroy(hm_runtime *rt);
int hm_runtime_buffers(hm_runtime *rt, void **pool, void **host_store, size_t *slot_bytes,
                       int64_t *n_slots);
int hm_runtime_image_of(const hm_runtime *rt, int layer, int expert, int64_t *image);
int hm_runtime_shared_slot(const hm_runtime *rt, int layer, int chunk, int64_t *slot);
/* One MoE layer: y[T, H] = x + sum_k w E_k(x) for router logits [T, ld],
 * executing the decision core's plan for this layer (engine.py:288-389).
 * Predictions for the prefetch decision: n_pred LayerRequests (pred_layers
 * [n_pred], pred_loads [n_pred][N], host), or n_pred == HM_PREDICT_LIVE for
 * the live look-ahead on x (hm_runtime_set_lookahead). */
#define HM_PREDICT_LIVE (-1)
int hm_runtime_forward_layer(hm_runtime *rt, int layer, const uint16_t *x, const float *logits,
                             int T, int ld, uint16_t *y, const int32_t *pred_layers,
                             const int64_t *pred_loads, int n_pred, void *stream,
                             hm_layer_stats *stats);
/* A whole pass (all L layers, one call): begin_pass, forward_layer per layer
 * (ping-pong between buf0/buf1; *y_out receives the final buffer), end_pass.
 * logits: L device pointers [T, ld].  pass_loads (HOST, [L*N], optional):
 * the pass's loads for the trace-mode prediction model (hm_predict_layers);
 * without them (and prefetch on) the live look-ahead predicts, if set.
 * stats: optional [L] array.  Under expert parallelism it needs the peer-memory
 * exchange (hm_runtime_set_ep_exchange). */
int hm_runtime_forward_pass(hm_runtime *rt, const uint16_t *x, const float *const *logits, int T,
                            int ld, uint16_t *buf0, uint16_t *buf1, const int64_t *pass_loads,
                            int64_t pass_index, int64_t seed, int horizon, double accuracy,
                            void *stream, hm_layer_stats *stats, hm_pass_result *result,
                            uint16_t **y_out);
/* The LayerRequest (loads, normalised scores) the router produced last. */
int hm_runtime_last_request(const hm_runtime *rt, int64_t *loads, double *scores);
/* The MRS table S [L, N] the decisions use -- one table, mapped into the GPU,
 * whose decode rows the router computes (synchronises the device). */
int hm_runtime_device_mrs(hm_runtime *rt, double *host_out);
int hm_runtime_sync(hm_runtime *rt);
/* Make experts resident (fixed residency of the baseline policies,
 * engine.py:423-434): add them to the cache and copy them into their slots. */
int hm_runtime_preload(hm_runtime *rt, const uint32_t *refs, int n);
/* ---- expert-parallel exchange over peer memory ---------- */
/* One process per GPU; every rank holds the replicated hidden state and its
 * home experts.  hm_ep owns a double-buffered fp32 inbox [2][world][max_rows*H]
 * and per-tile flags on this GPU; peers' buffers are mapped with CUDA IPC
 * (NVLink P2P on an NVSwitch box).  No reference counterpart: multi-GPU is a
 * non-goal of the reference. */
typedef struct hm_ep hm_ep;
int hm_ep_create(int rank, int world, int max_rows, int H, hm_ep **out);
void hm_ep_destroy(hm_ep *ep);
/* Writes two cudaIpcMemHandle_t (64 bytes each) for this rank's buffers. */
int hm_ep_ipc_handles(hm_ep *ep, void *inbox_handle, void *flags_handle);
int hm_ep_open_peer(hm_ep *ep, int peer, const void *inbox_handle, const void *flags_handle);
/* ONE kernel: this rank's partial combine (Eq. 1 over its home experts; rows in
 * host_mask4 read zero-copy from host_out) pushed into every rank's inbox,
 * per-tile flags, then y = residual + sum over ranks in rank order (bf16; y32
 * optional fp32 sum without residual).  Every rank must call it the same
 * number of times with the same T. */
int hm_ep_combine_allreduce(hm_ep *ep, const float *out, const float *host_out,
                            const uint64_t *host_mask4, const int32_t *pos, const float *w, int T,
                            int Kp, int H, const uint16_t *residual, uint16_t *y, float *y32,
                            void *stream);
/* Token-sharded mode ("dispatch: all-to-all(v) of token rows to
 * home ranks ... combine: all-to-all(v) back plus weighted sum"): every rank
 * routes only its own tokens.  hm_ep_enable_dispatch allocates one more IPC
 * region (metadata slots, flags, received rows, returned rows) and writes its
 * 64-byte handle; peers map it with hm_ep_open_peer_dispatch.  Per layer:
 *   hm_ep_dispatch_meta  all-gather of the ranks' per-expert counts [E] and
 *                        fp64 score sums [N]: global LayerRequest (rank-order
 *                        sums), home-rank row layout into dev/host meta
 *                        ([counts E | offsets E+1] int32, [sums N | scores N]
 *                        fp64), then *host_flag = host_seq;
 *   hm_ep_dispatch_rows  all-to-all of the local permuted rows to their
 *                        experts' home ranks (expert e homed on e % world,
 *                        shared chunk c on c % world);
 *   hm_ep_return_rows    all-to-all of the home rank's expert-output rows back
 *                        to their source ranks' permuted positions.
 * Each completes only when every rank's rows for this rank have landed. */
int hm_ep_enable_dispatch(hm_ep *ep, int n_experts_total, int n_routed, int Kp, void *region_handle);
int hm_ep_open_peer_dispatch(hm_ep *ep, int peer, const void *region_handle);
int hm_ep_dispatch_meta(hm_ep *ep, const int32_t *counts, const double *score_sum, int32_t *dev_meta_i,
                        double *dev_meta_d, int32_t *host_meta_i, double *host_meta_d,
                        uint32_t *host_flag, uint32_t host_seq, void *stream);
int hm_ep_dispatch_rows(hm_ep *ep, const uint16_t *xp, const int32_t *sel, const int32_t *row_src,
                        int rows, void *stream);
int hm_ep_return_rows(hm_ep *ep, const float *out, int rows, void *stream);
/* Device pointers of this rank's received-rows (bf16) and returned-rows (fp32) buffers. */
int hm_ep_dispatch_buffers(hm_ep *ep, uint16_t **xrecv, float **ret);
/* NCCL transport of the token-sharded mode (grouped
 * ncclSend/ncclRecv): the baseline of, and the fallback for, the peer-memory
 * kernels when CUDA IPC between the ranks is unavailable.  Rank 0 makes the
 * 128-byte ncclUniqueId, the caller distributes it (control plane), every rank
 * creates its exchange with dispatch mode enabled.  Then, per layer,
 * hm_ep_dispatch_meta = pack + in-place ncclAllGather of the [counts | sums]
 * slots + the same table kernel (its count matrix also mirrored to mapped host
 * memory); hm_ep_dispatch_rows / hm_ep_return_rows = one NCCL group of
 * per-(expert, peer) sends and receives planned on the host from that matrix
 * (hm_ep_a2a_plan), so they must be called after the meta flag was raised.
 * libnccl.so.2 is loaded at run time. */
int hm_ep_nccl_unique_id(void *id128);
int hm_ep_create_nccl(int rank, int world, int max_rows, int H, const void *id128, int n_experts_total,
                      int n_routed, int Kp, hm_ep **out);
int hm_ep_uses_nccl(const hm_ep *ep);
int hm_ep_world(const hm_ep *ep);
/* One rank's all-to-all(v) schedule from the all-gathered count matrix
 * counts_all [world][n_experts_total] (direction 0: dispatch, local permuted
 * rows -> home layouts; 1: return).  Ops in issue order; src_row / dst_row are
 * row indices in the sender's / receiver's buffer.  ops = NULL: count only. */
#define HM_A2A_SEND 0
#define HM_A2A_RECV 1
#define HM_A2A_COPY 2
typedef struct hm_a2a_op {
  int32_t kind, peer;
  int64_t src_row, dst_row, rows;
} hm_a2a_op;
int hm_ep_a2a_plan(const int32_t *counts_all, int world, int n_experts_total, int n_routed, int rank,
                   int direction, hm_a2a_op *ops, int max_ops, int *n_ops);
/* Live prediction: gate_w [L][ld][H] bf16
 * (device; NULL disables) -- layer l's input through the gates of layers
 * l+1..l+horizon gives the predicted loads of forward_layer(n_pred =
 * HM_PREDICT_LIVE) and of forward_pass without pass_loads (prefetch on). */
int hm_runtime_set_lookahead(hm_runtime *rt, const uint16_t *gate_w, int ld, int horizon);
/* Run forward_layer token-sharded through `ep` (dispatch mode enabled): x and
 * logits hold this rank's tokens only (T may be 0).  The exchange's world must
 * be the runtime's ep_world; world 1 runs the whole exchange on one rank. */
int hm_runtime_set_ep_dispatch(hm_runtime *rt, hm_ep *ep);
/* Route forward_layer's expert-parallel combine through `ep` (NULL: partial
 * to hm_runtime_set_ep_output's buffer for an external all-reduce). */
int hm_runtime_set_ep_exchange(hm_runtime *rt, hm_ep *ep);
/* Expert parallelism (ep_world > 1): forward_layer writes this rank's partial
 * sum_k w E_k(x) over its home experts to y32 [T, H] fp32 instead of y; the
 * caller all-reduces y32 across ranks and finishes with hm_residual_add. */
int hm_runtime_set_ep_output(hm_runtime *rt, float *y32);
/* CUDA-event timing of every expert-FFN launch (bench roofline): enable, then
 * read and reset the accumulated launch time / algorithmic bytes. */
int hm_runtime_set_kernel_timing(hm_runtime *rt, int on);
/* Optional CUDA-event timing of every H2D expert copy (demand and prefetch) on
 * the copy stream: achieved PCIe GB/s = total_bytes / total_ms. */
int hm_runtime_set_copy_timing(hm_runtime *rt, int on);
int hm_runtime_copy_times(hm_runtime *rt, double *total_ms, int64_t *total_bytes, int64_t *n,
                          double *max_ms);
int hm_runtime_kernel_times(hm_runtime *rt, double *total_ms, int64_t *total_bytes, int64_t *n,
                            double *max_ms);

#ifdef __cplusplus
}
#endif

#endif /* HYBRIMOE_H_ */
