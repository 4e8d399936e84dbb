// extern "C" surface of the decision core (include/hybrimoe.h).  Thin
// marshalling only: every body converts flat arrays to hm:: types, calls the
// core and copies results out; C++ exceptions become status codes.
#include <algorithm>
#include <cstring>

#include "decision.hpp"

// The opaque C handles are the hm:: objects themselves.
static inline hm::Cache *C(hm_cache *c) { return reinterpret_cast<hm::Cache *>(c); }
static inline const hm::Cache *C(const hm_cache *c) { return reinterpret_cast<const hm::Cache *>(c); }
static inline hm::Mrs *M(hm_mrs *m) { return reinterpret_cast<hm::Mrs *>(m); }
static inline const hm::Mrs *M(const hm_mrs *m) { return reinterpret_cast<const hm::Mrs *>(m); }
static inline hm::Evaluator *V(hm_evaluator *e) { return reinterpret_cast<hm::Evaluator *>(e); }
static inline const hm::Evaluator *V(const hm_evaluator *e) { return reinterpret_cast<const hm::Evaluator *>(e); }
static inline hm::Engine *E(hm_engine *e) { return reinterpret_cast<hm::Engine *>(e); }
static inline const hm::Engine *E(const hm_engine *e) { return reinterpret_cast<const hm::Engine *>(e); }

namespace {
std::vector<hm::Task> to_tasks(const hm_task *t, int n) {
  HM_REQUIRE(n >= 0 && (n == 0 || t != nullptr), HM_EVALUE, "bad task array");
  std::vector<hm::Task> v(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) v[i] = {t[i].ref, t[i].load};
  return v;
}
void emit(const hm::Plan &pl, hm_event *ev, int *n_ev, hm_assign *as, int *n_as, double *mk) {
  if (n_ev) *n_ev = static_cast<int>(pl.events.size());
  if (ev)
    for (size_t i = 0; i < pl.events.size(); ++i) {
      const hm::Event &e = pl.events[i];
      ev[i] = hm_event{e.device, e.kind, e.ref, 0, e.start, e.end};
    }
  if (n_as) *n_as = static_cast<int>(pl.assign.size());
  if (as)
    for (size_t i = 0; i < pl.assign.size(); ++i) as[i] = hm_assign{pl.assign[i].first, pl.assign[i].second};
  if (mk) *mk = pl.makespan;
}
hm::Plan from_c(const hm_event *ev, int n_ev, const hm_assign *as, int n_as, double mk) {
  hm::Plan pl;
  for (int i = 0; i < n_ev; ++i) pl.events.push_back({ev[i].device, ev[i].kind, ev[i].ref, ev[i].start, ev[i].end});
  for (int i = 0; i < n_as; ++i) pl.assign.emplace_back(as[i].ref, as[i].how);
  pl.makespan = mk;
  return pl;
}
}  // namespace

extern "C" {

int hm_last_error(char *buf, size_t n) {
  const std::string &m = hm::last_error();
  if (buf && n) {
    size_t k = m.size() < n - 1 ? m.size() : n - 1;
    std::memcpy(buf, m.data(), k);
    buf[k] = 0;
  }
  return static_cast<int>(m.size());
}

const char *hm_version(void) { return "hybrimoe-b200 0.1.0"; }

int hm_profile_check(const hm_profile *p) {
  HM_API_BEGIN
  hm::check_profile(*p);
  HM_API_END
}
int hm_gpu_time(const hm_profile *p, int64_t load, double *out) {
  HM_API_BEGIN
  *out = hm::gpu_time(*p, load);
  HM_API_END
}
int hm_cpu_time(const hm_profile *p, int64_t load, int64_t pos, double *out) {
  HM_API_BEGIN
  *out = hm::cpu_time(*p, load, pos);
  HM_API_END
}
int hm_transfer_time(const hm_profile *p, double expert_bytes, double *out) {
  HM_API_BEGIN
  *out = hm::transfer_time(*p, expert_bytes);
  HM_API_END
}

int hm_simulate_schedule(const hm_task *gq, int ng, const hm_task *cq, int nc, const hm_profile *p,
                         double bytes, hm_event *ev, int *n_ev, hm_assign *as, int *n_as, double *mk) {
  HM_API_BEGIN
  emit(hm::simulate_schedule(to_tasks(gq, ng), to_tasks(cq, nc), *p, bytes), ev, n_ev, as, n_as, mk);
  HM_API_END
}
int hm_plan_all_cpu(const hm_task *t, int n, const hm_profile *p, hm_event *ev, int *n_ev,
                    hm_assign *as, int *n_as, double *mk) {
  HM_API_BEGIN
  emit(hm::plan_all_cpu(to_tasks(t, n), *p), ev, n_ev, as, n_as, mk);
  HM_API_END
}
int hm_plan_all_gpu(const hm_task *c, int nc, const hm_task *u, int nu, const hm_profile *p,
                    double bytes, hm_event *ev, int *n_ev, hm_assign *as, int *n_as, double *mk) {
  HM_API_BEGIN
  emit(hm::plan_all_gpu(to_tasks(c, nc), to_tasks(u, nu), *p, bytes), ev, n_ev, as, n_as, mk);
  HM_API_END
}
int hm_select_plan_tasks(const hm_task *c, int nc, const hm_task *u, int nu, const hm_profile *p,
                         double bytes, hm_event *ev, int *n_ev, hm_assign *as, int *n_as, double *mk) {
  HM_API_BEGIN
  emit(hm::select_plan_tasks(to_tasks(c, nc), to_tasks(u, nu), *p, bytes), ev, n_ev, as, n_as, mk);
  HM_API_END
}
int hm_select_plan(const hm_cache *cache, int layer, const int64_t *loads, int n, const hm_profile *p,
                   double bytes, hm_event *ev, int *n_ev, hm_assign *as, int *n_as, double *mk) {
  HM_API_BEGIN
  std::vector<hm::Task> cached, uncached;
  for (int i = 0; i < n; ++i) {
    if (loads[i] <= 0) continue;
    uint32_t r = hm::pack_ref(layer, i);
    (C(cache)->is_resident(r) ? cached : uncached).push_back({r, loads[i]});
  }
  emit(hm::select_plan_tasks(cached, uncached, *p, bytes), ev, n_ev, as, n_as, mk);
  HM_API_END
}
int hm_check_plan(const hm_event *ev, int n_ev, const hm_assign *as, int n_as, double mk) {
  HM_API_BEGIN
  hm::check_plan(from_c(ev, n_ev, as, n_as, mk));
  HM_API_END
}
int hm_pcie_idle_budget(const hm_event *ev, int n_ev, double mk, double *out) {
  HM_API_BEGIN
  *out = hm::pcie_idle_budget(from_c(ev, n_ev, nullptr, 0, mk));
  HM_API_END
}
int hm_oracle_optimal(const hm_task *t, int n, const uint8_t *cached, const hm_profile *p, double bytes,
                      int limit, double *out) {
  HM_API_BEGIN
  std::vector<uint8_t> c(cached, cached + n);
  *out = hm::oracle_optimal(to_tasks(t, n), c, *p, bytes, limit);
  HM_API_END
}

int hm_evaluator_create(const hm_profile *p, double bytes, hm_evaluator **out) {
  HM_API_BEGIN
  auto *e = new hm::Evaluator();
  e->profile = *p;
  e->expert_bytes = bytes;
  *out = reinterpret_cast<hm_evaluator *>(e);
  HM_API_END
}
void hm_evaluator_destroy(hm_evaluator *e) { delete V(e); }
int hm_evaluator_makespan(hm_evaluator *e, const int64_t *c, int nc, const int64_t *u, int nu, double *out) {
  HM_API_BEGIN
  *out = V(e)->makespan(std::vector<int64_t>(c, c + nc), std::vector<int64_t>(u, u + nu));
  HM_API_END
}
int hm_evaluator_size(const hm_evaluator *e, int64_t *out) {
  HM_API_BEGIN
  *out = static_cast<int64_t>(V(e)->memo.size());
  HM_API_END
}

int hm_cache_create(int64_t capacity, hm_cache **out) {
  HM_API_BEGIN
  *out = reinterpret_cast<hm_cache *>(new hm::Cache(capacity));
  HM_API_END
}
void hm_cache_destroy(hm_cache *c) { delete C(c); }
int hm_cache_capacity(const hm_cache *c, int64_t *out) {
  HM_API_BEGIN
  *out = C(c)->capacity;
  HM_API_END
}
int hm_cache_lookup(hm_cache *c, uint32_t ref, int policy, int *hit) {
  HM_API_BEGIN
  *hit = C(c)->lookup(ref, policy) ? 1 : 0;
  HM_API_END
}
int hm_cache_insert(hm_cache *c, uint32_t ref, int policy, const hm_mrs *mrs, uint32_t *victim, int *has) {
  HM_API_BEGIN
  uint32_t v = 0;
  bool h = C(c)->insert(ref, policy, M(mrs), &v);
  *has = h ? 1 : 0;
  if (victim) *victim = h ? v : 0;
  HM_API_END
}
int hm_cache_victim(const hm_cache *c, int policy, const hm_mrs *mrs, uint32_t *victim) {
  HM_API_BEGIN
  *victim = C(c)->victim(policy, M(mrs));
  HM_API_END
}
int hm_cache_is_resident(const hm_cache *c, uint32_t ref, int *out) {
  HM_API_BEGIN
  *out = C(c)->is_resident(ref) ? 1 : 0;
  HM_API_END
}
int hm_cache_is_pinned(const hm_cache *c, uint32_t ref, int *out) {
  HM_API_BEGIN
  *out = C(c)->is_pinned(ref) ? 1 : 0;
  HM_API_END
}
int hm_cache_pin(hm_cache *c, uint32_t ref) {
  HM_API_BEGIN
  C(c)->pinned.insert(ref);
  HM_API_END
}
int hm_cache_unpin(hm_cache *c, uint32_t ref) {
  HM_API_BEGIN
  C(c)->pinned.erase(ref);
  HM_API_END
}
int hm_cache_clear_pinned(hm_cache *c) {
  HM_API_BEGIN
  C(c)->pinned.clear();
  HM_API_END
}
int hm_cache_add_resident(hm_cache *c, uint32_t ref) {
  HM_API_BEGIN
  C(c)->add_resident(ref);
  HM_API_END
}
int hm_cache_remove_resident(hm_cache *c, uint32_t ref) {
  HM_API_BEGIN
  C(c)->remove_resident(ref);
  HM_API_END
}
int hm_cache_clear_resident(hm_cache *c) {
  HM_API_BEGIN
  C(c)->clear_resident();
  HM_API_END
}
int hm_cache_counts(const hm_cache *c, int64_t *nr, int64_t *np) {
  HM_API_BEGIN
  if (nr) *nr = static_cast<int64_t>(C(c)->resident.size());
  if (np) *np = static_cast<int64_t>(C(c)->pinned.size());
  HM_API_END
}
int hm_cache_resident(const hm_cache *c, uint32_t *out, int64_t cap, int64_t *n) {
  HM_API_BEGIN
  int64_t i = 0;
  for (auto &kv : C(c)->resident) {
    if (out && i < cap) out[i] = kv.first;
    ++i;
  }
  *n = i;
  HM_API_END
}
int hm_cache_pinned(const hm_cache *c, uint32_t *out, int64_t cap, int64_t *n) {
  HM_API_BEGIN
  int64_t i = 0;
  for (uint32_t r : C(c)->pinned) {
    if (out && i < cap) out[i] = r;
    ++i;
  }
  *n = i;
  HM_API_END
}
int hm_cache_last_access(const hm_cache *c, uint32_t ref, int64_t *out, int *has) {
  HM_API_BEGIN
  auto it = C(c)->resident.find(ref);
  *has = (it != C(c)->resident.end() && it->second.has_last_access) ? 1 : 0;
  *out = *has ? it->second.last_access : 0;
  HM_API_END
}
int hm_cache_frequency(const hm_cache *c, uint32_t ref, int64_t *out, int *has) {
  HM_API_BEGIN
  auto it = C(c)->resident.find(ref);
  *has = (it != C(c)->resident.end() && it->second.has_frequency) ? 1 : 0;
  *out = *has ? it->second.frequency : 0;
  HM_API_END
}
int hm_cache_set_last_access(hm_cache *c, uint32_t ref, int64_t v) {
  HM_API_BEGIN
  auto it = C(c)->resident.find(ref);
  HM_REQUIRE(it != C(c)->resident.end(), HM_EVALUE, "last_access only tracks resident experts");
  it->second.last_access = v;
  it->second.has_last_access = true;
  HM_API_END
}
int hm_cache_set_frequency(hm_cache *c, uint32_t ref, int64_t v) {
  HM_API_BEGIN
  auto it = C(c)->resident.find(ref);
  HM_REQUIRE(it != C(c)->resident.end(), HM_EVALUE, "frequency only tracks resident experts");
  it->second.frequency = v;
  it->second.has_frequency = true;
  HM_API_END
}
int hm_cache_tick(const hm_cache *c, int64_t *out) {
  HM_API_BEGIN
  *out = C(c)->tick;
  HM_API_END
}
int hm_cache_next_tick(hm_cache *c, int64_t *out) {
  HM_API_BEGIN
  *out = C(c)->next_tick();
  HM_API_END
}
int hm_cache_slot(const hm_cache *c, uint32_t ref, int64_t *slot) {
  HM_API_BEGIN
  auto it = C(c)->resident.find(ref);
  *slot = it == C(c)->resident.end() ? -1 : it->second.slot;
  HM_API_END
}

int hm_mrs_create(int L, int N, double alpha, int p, hm_mrs **out) {
  HM_API_BEGIN
  HM_REQUIRE(!(alpha < 0.0) && !(alpha > 1.0), HM_EVALUE, "alpha must be in [0, 1]");
  HM_REQUIRE(p >= 1, HM_EVALUE, "p must be >= 1");
  HM_REQUIRE(L >= 1 && N >= 1 && L < 65536 && N < 65536, HM_EVALUE, "bad MRS shape");
  auto *m = new hm::Mrs();
  m->L = L;
  m->N = N;
  m->alpha = alpha;
  m->p = p;
  m->S.assign(static_cast<size_t>(L) * N, 1.0 / static_cast<double>(N));
  *out = reinterpret_cast<hm_mrs *>(m);
  HM_API_END
}
void hm_mrs_destroy(hm_mrs *m) { delete M(m); }
int hm_mrs_update(hm_mrs *m, int layer, const double *s, int n) {
  HM_API_BEGIN
  M(m)->update(layer, s, n);
  HM_API_END
}
int hm_mrs_get(const hm_mrs *m, uint32_t ref, double *out) {
  HM_API_BEGIN
  *out = M(m)->get(ref);
  HM_API_END
}
int hm_mrs_set(hm_mrs *m, uint32_t ref, double v) {
  HM_API_BEGIN
  int l = hm::ref_layer(ref), e = hm::ref_expert(ref);
  hm::Mrs *mm = M(m);
  HM_REQUIRE(l < mm->L && e < mm->N, HM_EVALUE, "ExpertRef outside the MRS table");
  mm->S[static_cast<size_t>(l) * mm->N + e] = v;
  HM_API_END
}
int hm_mrs_table(const hm_mrs *m, double *out) {
  HM_API_BEGIN
  std::memcpy(out, M(m)->S.data(), M(m)->S.size() * sizeof(double));
  HM_API_END
}
int hm_mrs_params(const hm_mrs *m, double *alpha, int *p, int *L, int *N) {
  HM_API_BEGIN
  if (alpha) *alpha = M(m)->alpha;
  if (p) *p = M(m)->p;
  if (L) *L = M(m)->L;
  if (N) *N = M(m)->N;
  HM_API_END
}
int hm_top_p_filter(const double *s, int n, int p, double *out) {
  HM_API_BEGIN
  std::vector<double> f = hm::top_p_filter(s, n, p);
  std::memcpy(out, f.data(), f.size() * sizeof(double));
  HM_API_END
}

int hm_evaluate_gain(uint32_t cand, int pl, const int64_t *loads, int n, const hm_cache *c, hm_evaluator *ev,
                     double *gain) {
  HM_API_BEGIN
  HM_REQUIRE(!C(c)->is_resident(cand), HM_EVALUE, hm::ref_str(cand) + " is already resident");
  std::vector<int64_t> bc, bu, wc, wu;
  for (int i = 0; i < n; ++i) {
    if (loads[i] <= 0) continue;
    uint32_t r = hm::pack_ref(pl, i);
    bool res = C(c)->is_resident(r);
    (res ? bc : bu).push_back(loads[i]);
    (res || r == cand ? wc : wu).push_back(loads[i]);
  }
  double base = V(ev)->makespan(bc, bu);
  double with_it = V(ev)->makespan(wc, wu);
  *gain = base - with_it;
  HM_API_END
}
int hm_select_prefetches(const hm_candidate *cands, int n, double budget, uint32_t *chosen, int *n_chosen) {
  HM_API_BEGIN
  HM_REQUIRE(!(budget < 0), HM_EVALUE, "idle_budget must be >= 0");
  std::vector<const hm_candidate *> ord;
  for (int i = 0; i < n; ++i)
    if (cands[i].gain > 0) ord.push_back(&cands[i]);
  std::stable_sort(ord.begin(), ord.end(), [](const hm_candidate *a, const hm_candidate *b) {
    if (a->gain != b->gain) return a->gain > b->gain;
    if (a->layer_distance != b->layer_distance) return a->layer_distance < b->layer_distance;
    return a->ref < b->ref;
  });
  double spent = 0.0;
  int k = 0;
  for (auto *c : ord) {
    if (spent + c->cost > budget) break;
    spent += c->cost;
    chosen[k++] = c->ref;
  }
  *n_chosen = k;
  HM_API_END
}

int hm_engine_create(const hm_engine_config *cfg, const hm_profile *p, hm_cache *cache, hm_mrs *mrs,
                     hm_evaluator *ev, hm_engine **out) {
  HM_API_BEGIN
  HM_REQUIRE(cache != nullptr && ev != nullptr, HM_EVALUE, "engine needs a cache and an evaluator");
  *out = reinterpret_cast<hm_engine *>(new hm::Engine(*cfg, *p, C(cache), M(mrs), V(ev)));
  HM_API_END
}
void hm_engine_destroy(hm_engine *e) { delete E(e); }
int hm_engine_set_fixed_pinned(hm_engine *e, const uint32_t *refs, int n) {
  HM_API_BEGIN
  hm::Engine *en = E(e);
  en->fixed_pinned.clear();
  for (int i = 0; i < n; ++i) en->fixed_pinned.insert(refs[i]);
  HM_API_END
}
int hm_engine_set_profile(hm_engine *e, const hm_profile *p) {
  HM_API_BEGIN
  hm::check_profile(*p);
  hm::Engine *en = E(e);
  en->profile = *p;
  en->evaluator.profile = *p;
  en->evaluator.memo.clear();  // memoised makespans belong to the old profile
  HM_API_END
}

int hm_engine_begin_pass(hm_engine *e) {
  HM_API_BEGIN
  E(e)->begin_pass();
  HM_API_END
}
int hm_engine_run_layer(hm_engine *e, int layer, const int64_t *loads, const double *scores, int n,
                        const int32_t *pred_layers, const int64_t *pred_loads, int n_pred) {
  HM_API_BEGIN
  E(e)->run_layer(layer, loads, scores, n, pred_layers, pred_loads, n_pred);
  HM_API_END
}
int hm_engine_end_pass(hm_engine *e, hm_pass_result *out) {
  HM_API_BEGIN
  E(e)->end_pass(out);
  HM_API_END
}
int hm_engine_layer_makespans(const hm_engine *e, double *out, int cap, int *n) {
  HM_API_BEGIN
  const hm::Engine *en = E(e);
  int k = static_cast<int>(en->layer_makespans.size());
  for (int i = 0; i < k && i < cap; ++i) out[i] = en->layer_makespans[i];
  *n = k;
  HM_API_END
}
int hm_engine_record_sizes(const hm_engine *e, hm_layer_record_sizes *o) {
  HM_API_BEGIN
  const hm::LayerRecord &r = E(e)->rec;
  o->n_lookups = static_cast<int32_t>(r.lookups.size());
  o->n_events = static_cast<int32_t>(r.plan.events.size());
  o->n_assign = static_cast<int32_t>(r.plan.assign.size());
  o->n_demand = static_cast<int32_t>(r.demand.size());
  o->n_candidates = static_cast<int32_t>(r.candidates.size());
  o->n_chosen = static_cast<int32_t>(r.chosen.size());
  o->expired = r.expired;
  o->n_selected = static_cast<int32_t>(r.selected.size());
  o->prefetch_evict_error = r.prefetch_evict_error;
  o->makespan = r.plan.makespan;
  o->budget = r.budget;
  HM_API_END
}
int hm_engine_record(const hm_engine *e, uint32_t *lookup_refs, uint8_t *lookup_hits, hm_event *events,
                     hm_assign *assign, uint32_t *demand_refs, uint32_t *demand_victims,
                     uint8_t *demand_has_victim, hm_candidate *candidates, uint32_t *chosen_refs,
                     uint32_t *chosen_victims, uint8_t *chosen_has_victim, uint32_t *selected_refs) {
  HM_API_BEGIN
  const hm::LayerRecord &r = E(e)->rec;
  for (size_t i = 0; i < r.selected.size(); ++i)
    if (selected_refs) selected_refs[i] = r.selected[i];
  for (size_t i = 0; i < r.lookups.size(); ++i) {
    if (lookup_refs) lookup_refs[i] = r.lookups[i].first;
    if (lookup_hits) lookup_hits[i] = r.lookups[i].second;
  }
  emit(r.plan, events, nullptr, assign, nullptr, nullptr);
  for (size_t i = 0; i < r.demand.size(); ++i) {
    if (demand_refs) demand_refs[i] = r.demand[i].first;
    if (demand_victims) demand_victims[i] = r.demand[i].second < 0 ? 0u : static_cast<uint32_t>(r.demand[i].second);
    if (demand_has_victim) demand_has_victim[i] = r.demand[i].second >= 0;
  }
  for (size_t i = 0; i < r.candidates.size(); ++i)
    if (candidates) candidates[i] = r.candidates[i];
  for (size_t i = 0; i < r.chosen.size(); ++i) {
    if (chosen_refs) chosen_refs[i] = r.chosen[i].first;
    if (chosen_victims) chosen_victims[i] = r.chosen[i].second < 0 ? 0u : static_cast<uint32_t>(r.chosen[i].second);
    if (chosen_has_victim) chosen_has_victim[i] = r.chosen[i].second >= 0;
  }
  HM_API_END
}

}  // extern "C"
