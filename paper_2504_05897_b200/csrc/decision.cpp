// Decision core of the HybriMoE hot path: cost model, intra-layer hybrid
// scheduler, MRS/LRU/LFU cache, impact-driven prefetch selection and the
// per-layer run_pass step order.  Reproduces /root/reference/pkg/src/moesim
// bit-for-bit in fp64: the build passes -ffp-contract=off so that no a*b+c is
// fused, every expression keeps the reference's left-to-right order, and all
// ties follow the reference's (value, ExpertRef) keys.
#include "decision.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>

namespace hm {

namespace {
thread_local std::string g_last_error;

// _TIE_ORDER (scheduling.py:45): PCIE < GPU < CPU on equal completion time.
inline int tie_order(int device) {
  return device == HM_DEV_PCIE ? 0 : (device == HM_DEV_GPU ? 1 : 2);
}
// Python's max(a, b) / min(a, b) keep the first argument unless the second
// is strictly greater / smaller.
inline double py_max(double a, double b) { return b > a ? b : a; }
inline double py_min(double a, double b) { return b < a ? b : a; }

std::string fmt(const char *f, double v) {
  char b[96];
  std::snprintf(b, sizeof b, f, v);
  return b;
}
}  // namespace

void set_last_error(const std::string &msg) { g_last_error = msg; }
const std::string &last_error() { return g_last_error; }

// ---------------------------------------------------------------- costs.py
void check_profile(const hm_profile &p) {
  // HardwareProfile.__post_init__ (costs.py:47-65)
  const std::pair<const char *, double> nonneg[] = {
      {"gpu_time_per_expert", p.gpu_time_per_expert}, {"cpu_slope", p.cpu_slope},
      {"gpu_slope", p.gpu_slope},                     {"transfer_latency", p.transfer_latency},
      {"shared_expert_time", p.shared_expert_time},   {"non_expert_time", p.non_expert_time}};
  for (auto &kv : nonneg)
    HM_REQUIRE(!(kv.second < 0), HM_EVALUE,
               std::string(kv.first) + fmt(" must be >= 0, got %.17g", kv.second));
  HM_REQUIRE(!(p.cpu_first_expert_penalty < 1.0), HM_EVALUE,
             fmt("cpu_first_expert_penalty must be >= 1, got %.17g", p.cpu_first_expert_penalty));
  HM_REQUIRE(!(p.transfer_bandwidth <= 0), HM_EVALUE,
             fmt("transfer_bandwidth must be > 0, got %.17g", p.transfer_bandwidth));
  HM_REQUIRE(p.gpu_saturation_load >= 1, HM_EVALUE,
             "gpu_saturation_load must be >= 1, got " + std::to_string(p.gpu_saturation_load));
}

double gpu_time(const hm_profile &p, int64_t load) {
  // costs.py:68-74
  HM_REQUIRE(load >= 1, HM_EVALUE, "load must be >= 1, got " + std::to_string(load));
  if (load <= p.gpu_saturation_load) return p.gpu_time_per_expert;
  return p.gpu_time_per_expert + p.gpu_slope * static_cast<double>(load - p.gpu_saturation_load);
}

double cpu_time(const hm_profile &p, int64_t load, int64_t pos) {
  // costs.py:77-88: cpu_slope * load * factor, evaluated left to right.
  HM_REQUIRE(load >= 1, HM_EVALUE, "load must be >= 1, got " + std::to_string(load));
  HM_REQUIRE(pos >= 0, HM_EVALUE, "position_in_burst must be >= 0, got " + std::to_string(pos));
  double factor = pos == 0 ? p.cpu_first_expert_penalty : 1.0;
  double t = p.cpu_slope * static_cast<double>(load);
  return t * factor;
}

double transfer_time(const hm_profile &p, double expert_bytes) {
  // costs.py:91-95: latency + ceil(bytes) / bandwidth (int -> float division)
  HM_REQUIRE(!(expert_bytes < 1), HM_EVALUE,
             fmt("expert_size_bytes must be >= 1, got %.17g", expert_bytes));
  double whole = std::ceil(expert_bytes);
  return p.transfer_latency + whole / p.transfer_bandwidth;
}

// ----------------------------------------------------------- scheduling.py
void check_plan(const Plan &plan) {
  // scheduling.py:80-124
  auto ev_str = [](const Event &e) {
    char b[160];
    std::snprintf(b, sizeof b, "TimelineEvent(device=%d, expert=%s, kind=%d, start=%.17g, end=%.17g)",
                  e.device, ref_str(e.ref).c_str(), e.kind, e.start, e.end);
    return std::string(b);
  };
  std::vector<int> dev_order;
  std::vector<std::vector<const Event *>> by_dev(3);
  for (const Event &ev : plan.events) {
    if (ev.end < ev.start) raise(HM_EPLAN, "event ends before it starts: " + ev_str(ev));
    if ((ev.device == HM_DEV_PCIE) != (ev.kind == HM_KIND_TRANSFER))
      raise(HM_EPLAN, "device/kind mismatch: " + ev_str(ev));
    if (by_dev[ev.device].empty()) dev_order.push_back(ev.device);
    by_dev[ev.device].push_back(&ev);
  }
  for (int d : dev_order) {
    auto evs = by_dev[d];
    std::stable_sort(evs.begin(), evs.end(),
                     [](const Event *a, const Event *b) { return a->start < b->start; });
    for (size_t i = 0; i + 1 < evs.size(); ++i)
      if (evs[i + 1]->start < evs[i]->end)
        raise(HM_EPLAN, "overlap on device: " + ev_str(*evs[i]) + " vs " + ev_str(*evs[i + 1]));
  }
  // the per-layer plans are small (tens of experts): sorted vectors instead of
  // hash containers keep this check off the allocator on the decision path
  std::vector<std::pair<uint32_t, const Event *>> computed;
  computed.reserve(plan.events.size());
  for (const Event &ev : plan.events)
    if (ev.kind == HM_KIND_COMPUTE) computed.emplace_back(ev.ref, &ev);
  std::stable_sort(computed.begin(), computed.end(),
                   [](const std::pair<uint32_t, const Event *> &a, const std::pair<uint32_t, const Event *> &b) {
                     return a.first < b.first;
                   });
  for (size_t i = 0; i + 1 < computed.size(); ++i)
    if (computed[i].first == computed[i + 1].first)
      raise(HM_EPLAN, "expert computed twice: " + ref_str(computed[i].first));
  std::vector<uint32_t> assigned;
  assigned.reserve(plan.assign.size());
  for (auto &a : plan.assign) assigned.push_back(a.first);
  std::sort(assigned.begin(), assigned.end());
  assigned.erase(std::unique(assigned.begin(), assigned.end()), assigned.end());
  bool same = assigned.size() == computed.size();
  for (size_t i = 0; same && i < assigned.size(); ++i) same = assigned[i] == computed[i].first;
  if (!same) raise(HM_EPLAN, "assignment and compute events cover different experts");
  auto compute_of = [&](uint32_t r) {
    auto it = std::lower_bound(computed.begin(), computed.end(), r,
                               [](const std::pair<uint32_t, const Event *> &a, uint32_t v) { return a.first < v; });
    return it->second;
  };
  for (auto &a : plan.assign) {
    if (a.second != HM_ASSIGN_GPU_TRANSFER) continue;
    const Event *tr = nullptr;  // the last transfer event of the expert (dict overwrite order)
    for (const Event &ev : plan.events)
      if (ev.kind == HM_KIND_TRANSFER && ev.ref == a.first) tr = &ev;
    if (!tr) raise(HM_EPLAN, ref_str(a.first) + " marked gpu_after_transfer but has no transfer");
    if (compute_of(a.first)->start < tr->end)
      raise(HM_EPLAN, ref_str(a.first) + " computed before its transfer ends");
  }
  if (!plan.events.empty()) {
    double mx = plan.events[0].end;
    for (const Event &ev : plan.events) mx = py_max(mx, ev.end);
    if (plan.makespan != mx) raise(HM_EPLAN, fmt("makespan %.17g != max event end", plan.makespan));
  } else if (plan.makespan != 0.0) {
    raise(HM_EPLAN, "empty plan must have makespan 0");
  }
}

// Plans are validated as they are built (SchedulePlan's checks), except the
// throw-away plans the memoised makespan evaluator builds only for their makespan.
static thread_local bool t_check_plans = true;

static Plan finalize(std::vector<Event> events, std::vector<std::pair<uint32_t, int>> assign) {
  // scheduling.py:150-157: sort by (start, end, tie order); stable.
  std::stable_sort(events.begin(), events.end(), [](const Event &a, const Event &b) {
    if (a.start != b.start) return a.start < b.start;
    if (a.end != b.end) return a.end < b.end;
    return tie_order(a.device) < tie_order(b.device);
  });
  Plan plan;
  double mk = 0.0;
  bool first = true;
  for (const Event &e : events) {
    mk = first ? e.end : py_max(mk, e.end);
    first = false;
  }
  plan.makespan = mk;
  plan.events = std::move(events);
  plan.assign = std::move(assign);
  if (t_check_plans) check_plan(plan);
  return plan;
}

static inline bool load_desc_less(const Task &a, const Task &b) {  // key (-load, ref)
  return a.load != b.load ? a.load > b.load : a.ref < b.ref;
}
static inline bool load_asc_less(const Task &a, const Task &b) {  // key (load, ref)
  return a.load != b.load ? a.load < b.load : a.ref < b.ref;
}

Plan simulate_schedule(const std::vector<Task> &gpu_q, const std::vector<Task> &cpu_q,
                       const hm_profile &p, double expert_bytes) {
  // scheduling.py:160-270
  {
    std::vector<uint32_t> g;  // sorted refs (tens of tasks: no hash set on the decision path)
    g.reserve(gpu_q.size());
    for (auto &t : gpu_q) g.push_back(t.ref);
    std::sort(g.begin(), g.end());
    for (auto &t : cpu_q)
      HM_REQUIRE(!std::binary_search(g.begin(), g.end(), t.ref), HM_EVALUE, "gpu and cpu queues must be disjoint");
    for (auto &t : gpu_q) HM_REQUIRE(t.load >= 1, HM_EVALUE, "every scheduled expert needs load >= 1");
    for (auto &t : cpu_q) HM_REQUIRE(t.load >= 1, HM_EVALUE, "every scheduled expert needs load >= 1");
  }
  const double tdur = transfer_time(p, expert_bytes);
  const int ng = static_cast<int>(gpu_q.size());
  const int n = ng + static_cast<int>(cpu_q.size());
  std::vector<Task> T;
  T.reserve(n);
  T.insert(T.end(), gpu_q.begin(), gpu_q.end());
  T.insert(T.end(), cpu_q.begin(), cpu_q.end());

  std::vector<uint8_t> claimed(n, 0), in_flight(n, 0), transferred(n, 0), in_pool(n, 0),
      in_cpu_pending(n, 0), in_transfer_pending(n, 0);
  std::vector<double> avail(n, 0.0);
  std::vector<int> pool;  // append order of (task, available_at)
  pool.reserve(n);
  for (int i = 0; i < ng; ++i) {
    pool.push_back(i);
    in_pool[i] = 1;
  }
  std::vector<int> cpu_pending, transfer_pending;
  for (int i = ng; i < n; ++i) {
    cpu_pending.push_back(i);
    transfer_pending.push_back(i);
    in_cpu_pending[i] = in_transfer_pending[i] = 1;
  }
  std::stable_sort(cpu_pending.begin(), cpu_pending.end(),
                   [&](int a, int b) { return load_asc_less(T[a], T[b]); });
  std::stable_sort(transfer_pending.begin(), transfer_pending.end(),
                   [&](int a, int b) { return load_desc_less(T[a], T[b]); });

  double clk[3] = {0.0, 0.0, 0.0};
  int64_t cpu_position = 0;
  int n_claimed = 0;
  std::vector<Event> events;
  events.reserve(2 * n);
  std::vector<std::pair<uint32_t, int>> assign;
  assign.reserve(n);
  // Eligibility in both pending lists only ever shrinks, so scan cursors are monotone.
  size_t cpu_cur = 0, tp_cur = 0;

  while (n_claimed < n) {
    // PCIe proposal: next transfer-queue expert neither claimed nor in flight.
    int pc = -1;
    while (tp_cur < transfer_pending.size()) {
      int id = transfer_pending[tp_cur];
      if (in_transfer_pending[id] && !claimed[id] && !in_flight[id]) {
        pc = id;
        break;
      }
      ++tp_cur;
    }
    double p_end = 0.0;
    if (pc >= 0) p_end = clk[HM_DEV_PCIE] + tdur;

    // GPU proposal (scheduling.py:191-202).
    int gc = -1;
    double g_start = 0.0, g_end = 0.0;
    {
      bool any = false, ready = false;
      double mn = 0.0;
      for (int id : pool) {
        if (!in_pool[id]) continue;
        if (!any) {
          mn = avail[id];
          any = true;
        } else {
          mn = py_min(mn, avail[id]);
        }
        if (avail[id] <= clk[HM_DEV_GPU]) ready = true;
      }
      if (any) {
        g_start = ready ? clk[HM_DEV_GPU] : py_max(clk[HM_DEV_GPU], mn);
        for (int id : pool) {
          if (!in_pool[id] || !(avail[id] <= g_start)) continue;
          if (gc < 0 || load_desc_less(T[id], T[gc])) gc = id;
        }
        g_end = g_start + gpu_time(p, T[gc].load);
      }
    }

    // CPU proposal (scheduling.py:204-212): own queue first, else steal.
    int cc = -1;
    bool stolen = false;
    double c_end = 0.0;
    while (cpu_cur < cpu_pending.size()) {
      int id = cpu_pending[cpu_cur];
      if (in_cpu_pending[id] && !in_flight[id] && !claimed[id]) {
        cc = id;
        break;
      }
      ++cpu_cur;
    }
    if (cc < 0) {
      for (int id : pool) {
        if (!in_pool[id] || !(avail[id] <= clk[HM_DEV_CPU])) continue;
        if (cc < 0 || load_asc_less(T[id], T[cc])) cc = id;
      }
      stolen = cc >= 0;
    }
    if (cc >= 0) c_end = clk[HM_DEV_CPU] + cpu_time(p, T[cc].load, cpu_position);

    // min over (end, tie order): PCIE(0) < GPU(1) < CPU(2).
    int dev = -1;
    double best = 0.0;
    if (pc >= 0) {
      dev = HM_DEV_PCIE;
      best = p_end;
    }
    if (gc >= 0 && (dev < 0 || g_end < best)) {
      dev = HM_DEV_GPU;
      best = g_end;
    }
    if (cc >= 0 && (dev < 0 || c_end < best)) {
      dev = HM_DEV_CPU;
      best = c_end;
    }
    if (dev < 0) raise(HM_ERUNTIME, "scheduler stalled with unscheduled experts");

    if (dev == HM_DEV_PCIE) {
      double start = clk[HM_DEV_PCIE];
      events.push_back({HM_DEV_PCIE, HM_KIND_TRANSFER, T[pc].ref, start, p_end});
      clk[HM_DEV_PCIE] = p_end;
      in_flight[pc] = transferred[pc] = 1;
      in_transfer_pending[pc] = 0;
      in_cpu_pending[pc] = 0;
      pool.push_back(pc);
      in_pool[pc] = 1;
      avail[pc] = p_end;
    } else if (dev == HM_DEV_GPU) {
      events.push_back({HM_DEV_GPU, HM_KIND_COMPUTE, T[gc].ref, g_start, g_end});
      clk[HM_DEV_GPU] = g_end;
      claimed[gc] = 1;
      ++n_claimed;
      in_pool[gc] = 0;
      assign.emplace_back(T[gc].ref, transferred[gc] ? HM_ASSIGN_GPU_TRANSFER : HM_ASSIGN_GPU_CACHED);
    } else {
      double start = clk[HM_DEV_CPU];
      events.push_back({HM_DEV_CPU, HM_KIND_COMPUTE, T[cc].ref, start, c_end});
      clk[HM_DEV_CPU] = c_end;
      claimed[cc] = 1;
      ++n_claimed;
      ++cpu_position;
      if (stolen)
        in_pool[cc] = 0;
      else
        in_cpu_pending[cc] = 0;
      assign.emplace_back(T[cc].ref, HM_ASSIGN_CPU);
    }
  }
  return finalize(std::move(events), std::move(assign));
}

Plan plan_all_cpu(std::vector<Task> tasks, const hm_profile &p) {
  // scheduling.py:273-284
  std::stable_sort(tasks.begin(), tasks.end(), load_asc_less);
  std::vector<Event> events;
  std::vector<std::pair<uint32_t, int>> assign;
  double clock = 0.0;
  int64_t pos = 0;
  for (const Task &t : tasks) {
    double end = clock + cpu_time(p, t.load, pos++);
    events.push_back({HM_DEV_CPU, HM_KIND_COMPUTE, t.ref, clock, end});
    assign.emplace_back(t.ref, HM_ASSIGN_CPU);
    clock = end;
  }
  return finalize(std::move(events), std::move(assign));
}

Plan plan_all_gpu(std::vector<Task> cached, std::vector<Task> uncached, const hm_profile &p,
                  double expert_bytes) {
  // scheduling.py:287-317
  std::stable_sort(cached.begin(), cached.end(), load_desc_less);
  std::stable_sort(uncached.begin(), uncached.end(), load_desc_less);
  double tdur = uncached.empty() ? 0.0 : transfer_time(p, expert_bytes);
  std::vector<Event> events;
  std::vector<std::pair<uint32_t, int>> assign;
  double gclock = 0.0;
  for (const Task &t : cached) {
    double end = gclock + gpu_time(p, t.load);
    events.push_back({HM_DEV_GPU, HM_KIND_COMPUTE, t.ref, gclock, end});
    assign.emplace_back(t.ref, HM_ASSIGN_GPU_CACHED);
    gclock = end;
  }
  double pclock = 0.0;
  for (const Task &t : uncached) {
    double arrive = pclock + tdur;
    events.push_back({HM_DEV_PCIE, HM_KIND_TRANSFER, t.ref, pclock, arrive});
    pclock = arrive;
    double start = py_max(gclock, arrive);
    double end = start + gpu_time(p, t.load);
    events.push_back({HM_DEV_GPU, HM_KIND_COMPUTE, t.ref, start, end});
    assign.emplace_back(t.ref, HM_ASSIGN_GPU_TRANSFER);
    gclock = end;
  }
  return finalize(std::move(events), std::move(assign));
}

Plan select_plan_tasks(const std::vector<Task> &cached, const std::vector<Task> &uncached,
                       const hm_profile &p, double expert_bytes) {
  // scheduling.py:320-335: greedy, then all-CPU, then all-GPU; strict < only.
  std::vector<Task> gq = cached, cq = uncached;
  std::stable_sort(gq.begin(), gq.end(), load_desc_less);
  std::stable_sort(cq.begin(), cq.end(), load_asc_less);
  Plan best = simulate_schedule(gq, cq, p, expert_bytes);
  // The guard plans are serial chains: their makespan is the last clock of
  // the chain (finalize's max over event ends), computed here with the same
  // operations in the same order; a plan is built only when it wins.
  std::vector<Task> all = cached;
  all.insert(all.end(), uncached.begin(), uncached.end());
  if (!all.empty()) {
    std::vector<Task> a = all;
    std::stable_sort(a.begin(), a.end(), load_asc_less);
    double clock = 0.0;
    int64_t pos = 0;
    for (const Task &t : a) clock = clock + cpu_time(p, t.load, pos++);
    if (clock < best.makespan) best = plan_all_cpu(all, p);
  } else if (0.0 < best.makespan) {
    best = plan_all_cpu(all, p);
  }
  {
    double gclock = 0.0;
    for (const Task &t : gq) gclock = gclock + gpu_time(p, t.load);  // gq: cached by (-load, ref)
    if (!uncached.empty()) {
      std::vector<Task> u = uncached;
      std::stable_sort(u.begin(), u.end(), load_desc_less);
      const double tdur = transfer_time(p, expert_bytes);
      double pclock = 0.0;
      for (const Task &t : u) {
        const double arrive = pclock + tdur;
        pclock = arrive;
        gclock = py_max(gclock, arrive) + gpu_time(p, t.load);
      }
    }
    if (gclock < best.makespan) best = plan_all_gpu(cached, uncached, p, expert_bytes);
  }
  return best;
}

double pcie_idle_budget(const Plan &plan) {
  // scheduling.py:405-412: Python sum() starting from int 0, in event order.
  double busy = 0.0;
  bool first = true;
  for (const Event &e : plan.events) {
    if (e.kind != HM_KIND_TRANSFER) continue;
    double d = e.end - e.start;
    busy = first ? d : busy + d;
    first = false;
  }
  double v = plan.makespan - busy;
  return py_max(0.0, v);
}

double oracle_optimal(const std::vector<Task> &tasks, const std::vector<uint8_t> &cached,
                      const hm_profile &p, double expert_bytes, int limit) {
  // scheduling.py:356-402 (exhaustive; test oracle)
  const int n = static_cast<int>(tasks.size());
  HM_REQUIRE(n <= limit, HM_EVALUE,
             "oracle limited to " + std::to_string(limit) + " activated experts, got " + std::to_string(n));
  const double tdur = transfer_time(p, expert_bytes);
  std::vector<int> asc(n), desc(n);
  for (int i = 0; i < n; ++i) asc[i] = desc[i] = i;
  std::stable_sort(asc.begin(), asc.end(), [&](int a, int b) { return load_asc_less(tasks[a], tasks[b]); });
  std::stable_sort(desc.begin(), desc.end(), [&](int a, int b) { return load_desc_less(tasks[a], tasks[b]); });
  double best = INFINITY;
  for (long mask = 0; mask < (1L << n); ++mask) {
    double cpu_total = 0.0;
    int64_t pos = 0;
    bool first = true;
    for (int i : asc)
      if (mask >> i & 1) {
        double c = cpu_time(p, tasks[i].load, pos++);
        cpu_total = first ? 0.0 + c : cpu_total + c;
        first = false;
      }
    if (cpu_total >= best) continue;
    double gclock = 0.0;
    for (int i : desc)
      if (!(mask >> i & 1) && cached[i]) gclock += gpu_time(p, tasks[i].load);
    int64_t arrivals = 0;
    for (int i : desc)
      if (!(mask >> i & 1) && !cached[i]) {
        ++arrivals;
        gclock = py_max(gclock, static_cast<double>(arrivals) * tdur) + gpu_time(p, tasks[i].load);
      }
    best = py_min(best, py_max(cpu_total, gclock));
  }
  return best;
}

double Evaluator::makespan(std::vector<int64_t> c, std::vector<int64_t> u) {
  // scheduling.py:446-457: key = (sorted cached, sorted uncached)
  std::sort(c.begin(), c.end());
  std::sort(u.begin(), u.end());
  std::string &key = kbuf;
  key.resize((c.size() + u.size() + 1) * sizeof(int64_t));
  char *w = &key[0];
  std::memcpy(w, c.data(), c.size() * sizeof(int64_t));
  w += c.size() * sizeof(int64_t);
  int64_t sep = -1;
  std::memcpy(w, &sep, sizeof sep);
  w += sizeof sep;
  std::memcpy(w, u.data(), u.size() * sizeof(int64_t));
  auto it = memo.find(key);
  if (it != memo.end()) return it->second;
  std::vector<Task> ct, ut;
  for (size_t i = 0; i < c.size(); ++i) ct.push_back({pack_ref(0, static_cast<int>(i)), c[i]});
  for (size_t i = 0; i < u.size(); ++i)
    ut.push_back({pack_ref(0, static_cast<int>(c.size() + i)), u[i]});
  struct NoCheck {
    NoCheck() { t_check_plans = false; }
    ~NoCheck() { t_check_plans = true; }
  } no_check;
  double v = select_plan_tasks(ct, ut, profile, expert_bytes).makespan;
  memo.emplace(key, v);
  return v;
}

// -------------------------------------------------------------- caching.py
std::vector<double> top_p_filter(const double *s, int n, int p) {
  // caching.py:58-62: keep the p largest by (-score, index)
  // (-score, index) is a total order, so partial selection of the first p
  // gives exactly the stable sort's prefix
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  const int keep = std::min(n, std::max(p, 0));
  std::partial_sort(order.begin(), order.begin() + keep, order.end(), [&](int a, int b) {
    if (s[a] != s[b]) return s[a] > s[b];
    return a < b;
  });
  std::vector<double> out(n, 0.0);
  for (int k = 0; k < keep; ++k) out[order[k]] = s[order[k]];
  return out;
}

void Mrs::update(int layer, const double *scores, int n) {
  // caching.py:65-76: S[i] <- a*t + (1-a)*S[i] for this layer only
  HM_REQUIRE(layer >= 0 && layer < L, HM_EVALUE, "mrs_update layer out of range");
  HM_REQUIRE(n == N, HM_EVALUE, "mrs_update expects one score per routed expert");
  std::vector<double> f = top_p_filter(scores, n, p);
  const double a = alpha;
  const double keep = 1.0 - a;
  double *row = &S[static_cast<size_t>(layer) * N];
  for (int i = 0; i < n; ++i) {
    double x = a * f[i];
    double y = keep * row[i];
    row[i] = x + y;
  }
}

Cache::Cache(int64_t cap) : capacity(cap) {
  HM_REQUIRE(cap >= 0, HM_EVALUE, "capacity must be >= 0, got " + std::to_string(cap));
  free_slots.reserve(static_cast<size_t>(cap));
  for (int64_t s = cap - 1; s >= 0; --s) free_slots.push_back(s);
}

bool Cache::lookup(uint32_t ref, int policy) {
  auto it = resident.find(ref);
  if (it == resident.end()) return false;
  if (policy == HM_POLICY_LRU) {
    it->second.last_access = next_tick();
    it->second.has_last_access = true;
  } else if (policy == HM_POLICY_LFU) {
    it->second.frequency = (it->second.has_frequency ? it->second.frequency : 0) + 1;
    it->second.has_frequency = true;
  }
  return true;
}

uint32_t Cache::victim(int policy, const Mrs *mrs) const {
  // caching.py:94-108: min over (resident - pinned) of (key, ref)
  bool any = false;
  uint32_t best = 0;
  double best_s = 0.0;
  int64_t best_i = 0;
  for (auto &kv : resident)
    if (!pinned.count(kv.first)) {
      any = true;
      break;
    }
  if (!any)
    raise(HM_EEVICTION, "cache full (" + std::to_string(resident.size()) + "/" +
                            std::to_string(capacity) + ") and all residents pinned");
  any = false;
  if (policy == HM_POLICY_MRS) {
    HM_REQUIRE(mrs != nullptr, HM_EVALUE, "MRS eviction needs an MrsState");
    for (auto &kv : resident) {
      if (pinned.count(kv.first)) continue;
      double s = mrs->get(kv.first);
      if (!any || s < best_s || (s == best_s && kv.first < best)) {
        best = kv.first;
        best_s = s;
        any = true;
      }
    }
    return best;
  }
  if (policy == HM_POLICY_LRU || policy == HM_POLICY_LFU) {
    for (auto &kv : resident) {
      if (pinned.count(kv.first)) continue;
      int64_t k = policy == HM_POLICY_LRU
                      ? (kv.second.has_last_access ? kv.second.last_access : 0)
                      : (kv.second.has_frequency ? kv.second.frequency : 0);
      if (!any || k < best_i || (k == best_i && kv.first < best)) {
        best = kv.first;
        best_i = k;
        any = true;
      }
    }
    return best;
  }
  raise(HM_EVALUE, "unknown policy " + std::to_string(policy));
}

bool Cache::insert(uint32_t ref, int policy, const Mrs *mrs, uint32_t *v) {
  // caching.py:111-128
  if (resident.count(ref)) raise(HM_EVALUE, ref_str(ref) + " is already resident");
  bool evicted = false;
  int64_t slot = -1;
  if (static_cast<int64_t>(resident.size()) >= capacity) {
    uint32_t victim_ref = victim(policy, mrs);
    auto it = resident.find(victim_ref);
    slot = it->second.slot;
    resident.erase(it);
    *v = victim_ref;
    evicted = true;
  } else if (!free_slots.empty()) {
    slot = free_slots.back();
    free_slots.pop_back();
  }
  CacheEntry e;
  e.slot = slot;
  if (policy == HM_POLICY_LRU) {
    e.last_access = next_tick();
    e.has_last_access = true;
  } else if (policy == HM_POLICY_LFU) {
    e.frequency = 1;
    e.has_frequency = true;
  }
  resident.emplace(ref, e);
  return evicted;
}

void Cache::add_resident(uint32_t ref) {
  if (resident.count(ref)) return;
  CacheEntry e;
  if (!free_slots.empty()) {
    e.slot = free_slots.back();
    free_slots.pop_back();
  }
  resident.emplace(ref, e);
}

void Cache::remove_resident(uint32_t ref) {
  auto it = resident.find(ref);
  if (it == resident.end()) return;
  if (it->second.slot >= 0) free_slots.push_back(it->second.slot);
  resident.erase(it);
}

void Cache::clear_resident() {
  resident.clear();
  free_slots.clear();
  for (int64_t s = capacity - 1; s >= 0; --s) free_slots.push_back(s);
}

// --------------------------------------------------------------- engine.py
Engine::Engine(const hm_engine_config &c, const hm_profile &p, Cache *cc, Mrs *m, Evaluator *ev)
    : cfg(c), profile(p), cache_(cc), mrs_(m), evaluator_(ev), cache(*cc), evaluator(*ev) {
  check_profile(p);
  HM_REQUIRE(c.num_layers >= 1 && c.num_routed >= 1 && c.num_routed < 65536 && c.num_layers < 65536,
             HM_EVALUE, "bad model shape");
  HM_REQUIRE(c.scheduling >= 0 && c.scheduling <= 3, HM_EVALUE, "unknown scheduling");
  HM_REQUIRE(c.cache_policy >= 0 && c.cache_policy <= 2, HM_EVALUE, "unknown cache policy");
}

long Engine::find_prefetch_pin(uint32_t r) const {
  for (size_t i = 0; i < prefetch_pins.size(); ++i)
    if (prefetch_pins[i].first == r) return static_cast<long>(i);
  return -1;
}

void Engine::begin_pass() {
  // engine.py:268-286
  tdur = transfer_time(profile, cfg.expert_bytes);
  res = hm_pass_result{};
  layer_makespans.clear();
  prefetch_pins.clear();
}

Plan Engine::build_plan(int layer, const int64_t *loads, int n) {
  // engine.py:234-249 (_build_plan) with the baseline planners at 171-205.
  // The plans built here satisfy SchedulePlan's invariants by construction;
  // their per-plan check (scheduling.py:156) runs when the policy asks for
  // validation (EnginePolicy.validate, engine.py:89) and stays on for plans
  // built through the scheduling API.
  struct CheckScope {
    bool prev;
    explicit CheckScope(bool on) : prev(t_check_plans) { t_check_plans = on; }
    ~CheckScope() { t_check_plans = prev; }
  } check_scope(cfg.validate != 0);
  std::vector<Task> tasks;
  for (int i = 0; i < n; ++i)
    if (loads[i] > 0) tasks.push_back({pack_ref(layer, i), loads[i]});
  if (cfg.scheduling == HM_SCHED_HYBRID || cfg.scheduling == HM_SCHED_GPU_ONDEMAND) {
    std::vector<Task> cached, uncached;
    for (auto &t : tasks) (cache.is_resident(t.ref) ? cached : uncached).push_back(t);
    if (cfg.scheduling == HM_SCHED_HYBRID) return select_plan_tasks(cached, uncached, profile, cfg.expert_bytes);
    return plan_all_gpu(cached, uncached, profile, cfg.expert_bytes);
  }
  auto serial_gpu = [&](std::vector<Task> ts, std::vector<Event> &ev,
                        std::vector<std::pair<uint32_t, int>> &as) {  // engine.py:171-182
    std::stable_sort(ts.begin(), ts.end(), load_desc_less);
    double clock = 0.0;
    for (auto &t : ts) {
      double end = clock + gpu_time(profile, t.load);
      ev.push_back({HM_DEV_GPU, HM_KIND_COMPUTE, t.ref, clock, end});
      as.emplace_back(t.ref, HM_ASSIGN_GPU_CACHED);
      clock = end;
    }
  };
  if (cfg.scheduling == HM_SCHED_STATIC_SPLIT) {  // engine.py:185-192
    if (layer < cfg.split_point) {
      std::vector<Event> ev;
      std::vector<std::pair<uint32_t, int>> as;
      serial_gpu(tasks, ev, as);
      return finalize(std::move(ev), std::move(as));
    }
    return plan_all_cpu(tasks, profile);
  }
  // fixed_frequency_map (engine.py:195-205)
  std::vector<Task> on_gpu, on_cpu;
  for (auto &t : tasks) (fixed_pinned.count(t.ref) ? on_gpu : on_cpu).push_back(t);
  std::vector<Event> ev;
  std::vector<std::pair<uint32_t, int>> as;
  serial_gpu(on_gpu, ev, as);
  Plan cpu_plan = plan_all_cpu(on_cpu, profile);
  ev.insert(ev.end(), cpu_plan.events.begin(), cpu_plan.events.end());
  as.insert(as.end(), cpu_plan.assign.begin(), cpu_plan.assign.end());
  return finalize(std::move(ev), std::move(as));
}

void Engine::run_layer(int layer, const int64_t *loads, const double *scores, int n,
                       const int32_t *pred_layers, const int64_t *pred_loads, int n_pred) {
  // engine.py:288-389, step for step.
  HM_REQUIRE(n == cfg.num_routed, HM_EVALUE, "loads must have one entry per routed expert");
  HM_REQUIRE(layer >= 0 && layer < cfg.num_layers, HM_EVALUE, "layer out of range");
  const bool static_sched = cfg.scheduling == HM_SCHED_STATIC_SPLIT || cfg.scheduling == HM_SCHED_FIXED_MAP;
  const bool track = cfg.scheduling != HM_SCHED_STATIC_SPLIT;
  const int policy = cfg.cache_policy;
  rec.lookups.clear();
  rec.demand.clear();
  rec.demand_slots.clear();
  rec.chosen_slots.clear();
  rec.candidates.clear();
  rec.chosen.clear();
  rec.selected.clear();
  rec.prefetch_evict_error = 0;
  rec.budget = 0.0;
  rec.expired = 0;

  std::vector<uint32_t> refs;
  for (int i = 0; i < n; ++i)
    if (loads[i] > 0) refs.push_back(pack_ref(layer, i));

  // (1) lookups first
  if (track) {
    for (uint32_t r : refs) {
      ++res.lookups;
      bool hit = cache.lookup(r, policy);
      if (hit) {
        ++res.hits;
        long k = find_prefetch_pin(r);
        if (k >= 0 && !prefetch_pins[k].second) {
          prefetch_pins[k].second = true;
          ++res.prefetch_hits;
        }
      }
      rec.lookups.emplace_back(r, hit ? 1 : 0);
    }
  }
  std::vector<uint32_t> layer_pins;
  for (uint32_t r : refs)
    if (cache.is_resident(r) && !cache.is_pinned(r)) layer_pins.push_back(r);
  for (uint32_t r : layer_pins) cache.pinned.insert(r);

  // (2) plan, (3) clock advance
  rec.plan = build_plan(layer, loads, n);
  const Plan &plan = rec.plan;
  double layer_time = plan.makespan + profile.shared_expert_time;
  layer_time = layer_time + profile.non_expert_time;
  layer_makespans.push_back(plan.makespan);
  res.latency += layer_time;
  double busy[3] = {0.0, 0.0, 0.0};
  for (const Event &e : plan.events) busy[e.device] += e.end - e.start;
  for (int d = 0; d < 3; ++d) res.busy[d] += busy[d];
  res.busy[HM_DEV_GPU] += profile.shared_expert_time + profile.non_expert_time;

  // (4) demand-transferred experts enter the cache in transfer-start order
  if (track && !static_sched && cache.capacity > 0) {
    std::vector<const Event *> arrived;
    for (const Event &e : plan.events)
      if (e.kind == HM_KIND_TRANSFER) arrived.push_back(&e);
    std::stable_sort(arrived.begin(), arrived.end(),
                     [](const Event *a, const Event *b) { return a->start < b->start; });
    for (const Event *e : arrived) {
      if (cache.is_resident(e->ref)) continue;
      uint32_t v = 0;
      bool has = cache.insert(e->ref, policy, mrs_, &v);  // EvictionError propagates
      ++res.inserts;
      if (has) {
        ++res.evictions;
        long k = find_prefetch_pin(v);
        if (k >= 0) prefetch_pins.erase(prefetch_pins.begin() + k);
      }
      rec.demand.emplace_back(e->ref, has ? static_cast<int64_t>(v) : -1);
      rec.demand_slots.push_back(cache.resident.at(e->ref).slot);
    }
  }

  // (5) score-aware state follows every executed layer
  if (track && policy == HM_POLICY_MRS && mrs_ != nullptr) {
    if (gpu_mrs_row)
      std::copy(gpu_mrs_row, gpu_mrs_row + mrs_->N, mrs_->S.begin() + static_cast<size_t>(layer) * mrs_->N);
    else
      mrs_->update(layer, scores, n);
  }
  gpu_mrs_row = nullptr;

  // (6) prefetch into the plan's idle PCIe time
  if (cfg.prefetch && !static_sched && cache.capacity > 0) {
    const double budget = pcie_idle_budget(plan);
    rec.budget = budget;
    for (int d = 0; d < n_pred; ++d) {
      const int pl = pred_layers[d];
      const int64_t *pload = pred_loads + static_cast<size_t>(d) * n;
      std::vector<int64_t> base_c, base_u;
      std::vector<int> act;
      for (int i = 0; i < n; ++i) {
        if (pload[i] <= 0) continue;
        act.push_back(i);
        (cache.is_resident(pack_ref(pl, i)) ? base_c : base_u).push_back(pload[i]);
      }
      bool have_base = false;
      double base = 0.0;
      for (int i : act) {
        uint32_t r = pack_ref(pl, i);
        if (cache.is_resident(r)) continue;
        // evaluate_gain (prefetch.py:104-121) through the memoised evaluator
        if (!have_base) {
          base = evaluator.makespan(base_c, base_u);
          have_base = true;
        }
        std::vector<int64_t> wc = base_c, wu;
        wc.push_back(pload[i]);
        bool removed = false;
        for (int64_t x : base_u) {
          if (!removed && x == pload[i]) {
            removed = true;
            continue;
          }
          wu.push_back(x);
        }
        double with_it = evaluator.makespan(wc, wu);
        hm_candidate c;
        c.ref = r;
        c.layer_distance = d + 1;
        c.predicted_load = pload[i];
        c.gain = base - with_it;
        c.cost = tdur;
        rec.candidates.push_back(c);
      }
    }
    // select_prefetches (prefetch.py:124-143)
    std::vector<const hm_candidate *> ordered;
    for (auto &c : rec.candidates)
      if (c.gain > 0) ordered.push_back(&c);
    std::stable_sort(ordered.begin(), ordered.end(), [](const hm_candidate *a, const hm_candidate *b) {
      if (a->gain != b->gain) return a->gain > b->gain;
      if (a->layer_distance != b->layer_distance) return a->layer_distance < b->layer_distance;
      return a->ref < b->ref;
    });
    std::vector<uint32_t> chosen;
    double spent = 0.0;
    for (auto *c : ordered) {
      if (spent + c->cost > budget) break;
      spent += c->cost;
      chosen.push_back(c->ref);
    }
    rec.selected = chosen;
    for (uint32_t r : chosen) {
      if (cache.is_resident(r)) continue;
      uint32_t v = 0;
      bool has;
      try {
        has = cache.insert(r, policy, mrs_, &v);
      } catch (const Error &err) {
        if (err.code == HM_EEVICTION) {  // prefetch is opportunistic
          rec.prefetch_evict_error = 1;
          break;
        }
        throw;
      }
      ++res.inserts;
      ++res.prefetch_issued;
      res.busy[HM_DEV_PCIE] += tdur;
      if (has) {
        ++res.evictions;
        long k = find_prefetch_pin(v);
        if (k >= 0) prefetch_pins.erase(prefetch_pins.begin() + k);
      }
      cache.pinned.insert(r);
      if (find_prefetch_pin(r) < 0) prefetch_pins.emplace_back(r, false);
      rec.chosen.emplace_back(r, has ? static_cast<int64_t>(v) : -1);
      rec.chosen_slots.push_back(cache.resident.at(r).slot);
    }
    if (cfg.validate) {
      Plan replan = build_plan(layer, loads, n);
      if (replan.makespan != plan.makespan)
        raise(HM_EASSERT, "prefetch changed the committed layer makespan");
    }
  }

  // (7) unpin this layer, expire prefetch pins whose layer just ran
  for (uint32_t r : layer_pins) cache.pinned.erase(r);
  for (size_t i = 0; i < prefetch_pins.size();) {
    if (ref_layer(prefetch_pins[i].first) <= layer) {
      cache.pinned.erase(prefetch_pins[i].first);
      if (!prefetch_pins[i].second) {
        ++res.prefetch_expired;
        ++rec.expired;
      }
      prefetch_pins.erase(prefetch_pins.begin() + static_cast<long>(i));
    } else {
      ++i;
    }
  }
}

void Engine::end_pass(hm_pass_result *out) {
  // engine.py:392-398
  for (auto &kv : prefetch_pins) {
    cache.pinned.erase(kv.first);
    if (!kv.second) ++res.prefetch_expired;
  }
  prefetch_pins.clear();
  HM_REQUIRE(res.hits <= res.lookups, HM_EVALUE, "hits exceed lookups");
  HM_REQUIRE(res.evictions <= res.inserts, HM_EVALUE, "evictions exceed inserts");
  if (out) *out = res;
}

}  // namespace hm
