// Host worker thread pool and CPU expert kernel (see host_worker.cpp).
#pragma once

#include <atomic>
#include <memory>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "common.hpp"

namespace hm {

// Fixed pool; run(fn) executes fn(tid, n) on every thread (the caller is tid 0).
// Workers spin for a short while before sleeping, so the back-to-back expert
// launches of a decode layer do not pay a futex wake-up each; barrier() is a
// spin barrier usable inside a job (every thread must call it).
class ThreadPool {
 public:
  explicit ThreadPool(int n, int spin_us = 3000);
  ~ThreadPool();
  int size() const { return n_; }
  // before_self (optional) runs on the caller after the workers were woken
  // and before the caller joins as tid 0: host work that overlaps the job's
  // start (jobs must tolerate a late tid 0, e.g. by stealing its range)
  void run(const std::function<void(int, int)> &fn, const std::function<void()> *before_self = nullptr);
  void barrier();
  // split barrier: arrive() returns the phase token; passed(token) tells
  // whether every thread has arrived; wait(token) blocks until then.  Lets a
  // thread do useful work (prefetch its next phase) while it waits.
  uint32_t arrive();
  bool passed(uint32_t token) const;
  void wait(uint32_t token);
  // Work ranges with stealing (one cache line per thread and phase): thread t
  // owns [front, back) of some index space, takes chunks from the front;
  // a thread that ran out takes chunks from the back of the others' ranges.
  struct alignas(64) Range {
    std::atomic<uint64_t> fb{0};  // (front << 32) | back
  };
  Range *ranges(int phase) { return &ranges_[static_cast<size_t>(phase) * n_]; }

 private:
  void loop(int tid);
  int n_;
  int spin_us_;
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_;
  const std::function<void(int, int)> *job_ = nullptr;
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> pending_{0};
  std::atomic<int> bar_count_{0};
  std::atomic<uint32_t> bar_sense_{0};
  std::atomic<bool> stop_{false};
  std::unique_ptr<Range[]> ranges_;
};

// AMX path for multi-token experts (prefill); amx_available() requests the
// XTILEDATA permission on first use.
bool amx_available();
void cpu_expert_amx(ThreadPool &pool, const uint16_t *img, int H, int I, const uint16_t *x, int M, float *out,
                    std::vector<uint16_t> &scratch);

// n single-token experts at once (decode): one pool run, one barrier.
// before_self: see ThreadPool::run.
void cpu_experts_decode(ThreadPool &pool, const uint16_t *const *imgs, const uint16_t *const *xs, int n, int H,
                        int I, float *const *outs, std::vector<uint16_t> &hbuf,
                        const std::function<void()> *before_self = nullptr);

// n multi-token experts (prefill) in one pool run on AMX (Ms[e] tokens each);
// same per-unit arithmetic as cpu_expert_amx.  before_self: see ThreadPool::run.
void cpu_experts_amx(ThreadPool &pool, const uint16_t *const *imgs, const uint16_t *const *xs, const int *Ms, int n,
                     int H, int I, float *const *outs, std::vector<uint16_t> &scratch,
                     const std::function<void()> *before_self = nullptr);

// 4-bit expert images (include/hybrimoe.h, hm_q4_*): decode GEMV on the
// nibbles; multi-token groups dequantize 32-row units and run on AMX.
void cpu_experts_decode_q4(ThreadPool &pool, const uint8_t *const *imgs, const uint16_t *const *xs, int n, int H,
                           int I, float *const *outs, std::vector<uint16_t> &hbuf,
                           const std::function<void()> *before_self = nullptr);
void cpu_expert_q4(ThreadPool &pool, const uint8_t *img, int H, int I, const uint16_t *x, int M, float *out,
                   std::vector<uint16_t> &scratch);

// out[M, H] fp32 = W2 (silu(Wg x) * (Wu x)) for one expert image (slot layout).
void cpu_expert(ThreadPool &pool, const uint16_t *img, int H, int I, const uint16_t *x, int M, float *out,
                std::vector<uint16_t> &hbuf);

}  // namespace hm
