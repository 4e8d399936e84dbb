// Decision core: the reference's scheduling / caching / prefetch / run_pass
// logic as C++17, bit-identical in fp64 (built with -ffp-contract=off).
//
// Reference: /root/reference/pkg/src/moesim/{costs,scheduling,caching,
// prefetch,engine}.py.  Every function cites the lines it follows.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <new>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <utility>
#include <vector>

#include "common.hpp"

namespace hm {

struct Task {
  uint32_t ref;
  int64_t load;
};

struct Event {
  int32_t device;
  int32_t kind;
  uint32_t ref;
  double start;
  double end;
};

struct Plan {
  std::vector<Event> events;                      // _finalize order
  std::vector<std::pair<uint32_t, int>> assign;   // insertion (commit) order
  double makespan = 0.0;
};

// costs.py:68-95
double gpu_time(const hm_profile &p, int64_t load);
double cpu_time(const hm_profile &p, int64_t load, int64_t pos);
double transfer_time(const hm_profile &p, double expert_bytes);
void check_profile(const hm_profile &p);

// scheduling.py
void check_plan(const Plan &plan);
Plan simulate_schedule(const std::vector<Task> &gpu_q, const std::vector<Task> &cpu_q,
                       const hm_profile &p, double expert_bytes);
Plan plan_all_cpu(std::vector<Task> tasks, const hm_profile &p);
Plan plan_all_gpu(std::vector<Task> cached, std::vector<Task> uncached, const hm_profile &p,
                  double expert_bytes);
Plan select_plan_tasks(const std::vector<Task> &cached, const std::vector<Task> &uncached,
                       const hm_profile &p, double expert_bytes);
double pcie_idle_budget(const Plan &plan);
double oracle_optimal(const std::vector<Task> &tasks, const std::vector<uint8_t> &cached,
                      const hm_profile &p, double expert_bytes, int limit);

// MakespanEvaluator (scheduling.py:433-465)
struct Evaluator {
  hm_profile profile;
  double expert_bytes;
  std::unordered_map<std::string, double> memo;
  std::string kbuf;  // reused lookup key (no allocation on a memo hit)
  double makespan(std::vector<int64_t> cached, std::vector<int64_t> uncached);
};

// MrsState (caching.py:30-76): dense S table over L x N.
// Page-aligned, page-padded storage: a runtime maps the MRS table into the GPU
// (cudaHostRegister) so the router can read the old row; separate tables
// never share a page.
template <typename T>
struct PageAlloc {
  using value_type = T;
  PageAlloc() = default;
  template <typename U>
  PageAlloc(const PageAlloc<U> &) {}
  T *allocate(size_t n) {
    const size_t bytes = (n * sizeof(T) + 4095) / 4096 * 4096;
    void *p = std::aligned_alloc(4096, bytes ? bytes : 4096);
    if (!p) throw std::bad_alloc();
    return static_cast<T *>(p);
  }
  void deallocate(T *p, size_t) { std::free(p); }
  template <typename U>
  bool operator==(const PageAlloc<U> &) const { return true; }
  template <typename U>
  bool operator!=(const PageAlloc<U> &) const { return false; }
};

struct Mrs {
  int L = 0, N = 0;
  double alpha = 0.5;
  int p = 4;
  std::vector<double, PageAlloc<double>> S;
  double get(uint32_t ref) const {
    int l = ref_layer(ref), e = ref_expert(ref);
    if (l < L && e < N) return S[static_cast<size_t>(l) * N + e];
    return 0.0;  // scores.get(e, 0.0)  (caching.py:103)
  }
  void update(int layer, const double *scores, int n);
};
std::vector<double> top_p_filter(const double *scores, int n, int p);

// CacheState (core.py:235-265) + HBM slot map (runtime extension).
struct CacheEntry {
  int64_t last_access = 0;
  int64_t frequency = 0;
  bool has_last_access = false;
  bool has_frequency = false;
  int64_t slot = -1;
};

// Sorted-vector set of refs: the pinned set holds a layer's activated experts
// plus prefetch pins (tens, at most a few hundred), inserted and erased every
// layer -- a hash set paid a node allocation per insert on the decision path.
struct FlatSet {
  std::vector<uint32_t> v;
  size_t count(uint32_t r) const { return std::binary_search(v.begin(), v.end(), r) ? 1 : 0; }
  void insert(uint32_t r) {
    auto it = std::lower_bound(v.begin(), v.end(), r);
    if (it == v.end() || *it != r) v.insert(it, r);
  }
  void erase(uint32_t r) {
    auto it = std::lower_bound(v.begin(), v.end(), r);
    if (it != v.end() && *it == r) v.erase(it);
  }
  void clear() { v.clear(); }
  size_t size() const { return v.size(); }
  bool empty() const { return v.empty(); }
  std::vector<uint32_t>::const_iterator begin() const { return v.begin(); }
  std::vector<uint32_t>::const_iterator end() const { return v.end(); }
};

struct Cache {
  int64_t capacity = 0;
  std::unordered_map<uint32_t, CacheEntry> resident;
  FlatSet pinned;
  std::vector<int64_t> free_slots;  // LIFO of unused HBM slots
  int64_t tick = 0;

  explicit Cache(int64_t cap);
  bool is_resident(uint32_t r) const { return resident.count(r) != 0; }
  bool is_pinned(uint32_t r) const { return pinned.count(r) != 0; }
  int64_t next_tick() { return ++tick; }
  bool lookup(uint32_t ref, int policy);                               // caching.py:79-91
  uint32_t victim(int policy, const Mrs *mrs) const;                   // caching.py:94-108
  bool insert(uint32_t ref, int policy, const Mrs *mrs, uint32_t *v);  // caching.py:111-128
  void add_resident(uint32_t ref);
  void remove_resident(uint32_t ref);
  void clear_resident();
};

// engine.py:255-486
struct LayerRecord {
  std::vector<std::pair<uint32_t, uint8_t>> lookups;
  Plan plan;
  std::vector<std::pair<uint32_t, int64_t>> demand;  // (ref, victim or -1)
  std::vector<int64_t> demand_slots;                 // HBM slot each demand insert landed in
  std::vector<int64_t> chosen_slots;                 // HBM slot of each prefetch insert
  std::vector<hm_candidate> candidates;
  std::vector<uint32_t> selected;                   // select_prefetches output
  std::vector<std::pair<uint32_t, int64_t>> chosen;  // inserted: (ref, victim or -1)
  int prefetch_evict_error = 0;                     // an insert hit EvictionError (engine.py:360-363)
  double budget = 0.0;
  int expired = 0;
};

// The engine borrows the run's CacheState / MrsState / MakespanEvaluator (as
// run_pass does, engine.py:255-265); mrs may be null like the reference's.
struct Engine {
  hm_engine_config cfg;
  hm_profile profile;
  Cache *cache_;
  Mrs *mrs_;
  Evaluator *evaluator_;
  Cache &cache;
  Evaluator &evaluator;
  std::unordered_set<uint32_t> fixed_pinned;
  // prefetch_pins: ref -> used, in insertion order (engine.py:429)
  std::vector<std::pair<uint32_t, bool>> prefetch_pins;
  hm_pass_result res{};
  std::vector<double> layer_makespans;
  LayerRecord rec;
  double tdur = 0.0;
  // Step (5)'s new MRS row as computed on the GPU by the layer's router
  // (runtime zero-copy decode path), consumed instead of the host recurrence
  // for the next run_layer call only; bit-identical by construction
  // (tests/test_kernels_gpu.py::test_mrs_update_dev_bit_exact).
  const double *gpu_mrs_row = nullptr;

  Engine(const hm_engine_config &c, const hm_profile &p, Cache *cache, Mrs *mrs, Evaluator *ev);
  void begin_pass();
  void run_layer(int layer, const int64_t *loads, const double *scores, int n,
                 const int32_t *pred_layers, const int64_t *pred_loads, int n_pred);
  void end_pass(hm_pass_result *out);
  Plan build_plan(int layer, const int64_t *loads, int n);

 private:
  long find_prefetch_pin(uint32_t r) const;
};

}  // namespace hm
