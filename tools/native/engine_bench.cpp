// Decision-core latency per decode layer through the C ABI (no Python):
// hm_engine_run_layer on DeepSeek-, Mixtral- and Qwen2-shaped decode requests
// (K one-hot loads, softmax-like scores), a 25 % cache warmed by one prefill-like
// pass.  g++ -O2 -I include tools/native/engine_bench.cpp -L paper_2504_05897_b200 -lhybrimoe
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "hybrimoe.h"

static void run(const char *name, int L, int N, int K, double eb, double cpu_slope) {
  hm_profile p{4e-5, cpu_slope, 55e9, 0.0, 256, 0.0, 1.2, 0.0, 0.0};
  const int64_t cap = static_cast<int64_t>(std::floor(0.25 * L * N));
  hm_cache *c;
  hm_mrs *m;
  hm_evaluator *ev;
  hm_engine *e;
  hm_cache_create(cap, &c);
  hm_mrs_create(L, N, 0.5, 2 * K, &m);
  hm_evaluator_create(&p, eb, &ev);
  hm_engine_config cfg{L, N, K, HM_SCHED_HYBRID, HM_POLICY_MRS, 0, 0, L / 4, cap, eb, 1, 0};
  hm_engine_create(&cfg, &p, c, m, ev, &e);
  std::mt19937_64 rng(1);
  std::vector<int64_t> loads(N);
  std::vector<double> scores(N);
  auto req = [&](int tokens) {
    std::fill(loads.begin(), loads.end(), 0);
    double tot = 0;
    for (int i = 0; i < N; ++i) tot += (scores[i] = std::exp(std::normal_distribution<double>(0, 1)(rng)));
    for (int i = 0; i < N; ++i) scores[i] /= tot;
    for (int t = 0; t < tokens; ++t) {
      int picked = 0;
      while (picked < K) {
        int i = static_cast<int>(rng() % N);
        if (tokens == 1 && loads[i]) continue;
        ++loads[i];
        ++picked;
      }
    }
  };
  hm_engine_begin_pass(e);
  for (int l = 0; l < L; ++l) {
    req(1024);
    hm_engine_run_layer(e, l, loads.data(), scores.data(), N, nullptr, nullptr, 0);
  }
  hm_pass_result pr;
  hm_engine_end_pass(e, &pr);
  std::vector<double> ts;
  for (int s = 0; s < 200; ++s) {
    hm_engine_begin_pass(e);
    for (int l = 0; l < L; ++l) {
      req(1);
      auto t0 = std::chrono::steady_clock::now();
      int rc = hm_engine_run_layer(e, l, loads.data(), scores.data(), N, nullptr, nullptr, 0);
      ts.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
      if (rc) { std::printf("rc %d\n", rc); return; }
    }
    hm_engine_end_pass(e, &pr);
  }
  std::sort(ts.begin(), ts.end());
  std::printf("%-9s decode layer: median %.2f us, p90 %.2f us\n", name, ts[ts.size() / 2], ts[ts.size() * 9 / 10]);
  hm_engine_destroy(e);
  hm_evaluator_destroy(ev);
  hm_mrs_destroy(m);
  hm_cache_destroy(c);
}

int main() {
  run("mixtral", 32, 8, 2, 352321536.0, 2.5e-4);
  run("deepseek", 26, 64, 6, 17301504.0, 1.2e-5);
  run("qwen2", 28, 64, 8, 55050240.0, 4e-5);
}
