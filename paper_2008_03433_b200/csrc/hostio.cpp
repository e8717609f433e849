// Host-side runtime services (see hostio.h).
#include "hostio.h"

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace tb {

void cuda_check(cudaError_t e, const char* what);  // engine.cpp

// ---------------------------------------------------------------------------
// device memory pool
// ---------------------------------------------------------------------------
void prepare_device_pool(int device) {
  static std::mutex mu;
  static std::vector<bool> done;
  std::lock_guard<std::mutex> g(mu);
  if ((int)done.size() <= device) done.resize(device + 1, false);
  if (done[device]) return;
  cudaMemPool_t pool;
  cuda_check(cudaDeviceGetDefaultMemPool(&pool, device), "cudaDeviceGetDefaultMemPool");
  uint64_t keep = UINT64_MAX;
  cuda_check(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep),
             "cudaMemPoolSetAttribute");
  done[device] = true;
}

cudaStream_t& alloc_stream() {
  static thread_local cudaStream_t s = nullptr;
  return s;
}

// ---------------------------------------------------------------------------
// pinned slab
// ---------------------------------------------------------------------------
namespace {
constexpr size_t kBlock = 256;
constexpr size_t kSlabBlocks = 1024;  // 256 KB arenas
std::mutex g_slab_mu;
std::vector<void*> g_free_blocks;
}  // namespace

void* pinned_block_get() {
  std::lock_guard<std::mutex> g(g_slab_mu);
  if (g_free_blocks.empty()) {
    void* arena = nullptr;
    cuda_check(cudaMallocHost(&arena, kBlock * kSlabBlocks), "cudaMallocHost");
    for (size_t i = 0; i < kSlabBlocks; ++i)
      g_free_blocks.push_back(static_cast<char*>(arena) + (kSlabBlocks - 1 - i) * kBlock);
  }
  void* p = g_free_blocks.back();
  g_free_blocks.pop_back();
  std::memset(p, 0, kBlock);
  return p;
}

void pinned_block_put(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> g(g_slab_mu);
  g_free_blocks.push_back(p);
}

// ---------------------------------------------------------------------------
// pinned buffer pool
// ---------------------------------------------------------------------------
namespace {
std::mutex g_pool_mu;
std::vector<std::pair<size_t, void*>> g_pool_free;   // (capacity, pointer)
std::vector<std::pair<void*, size_t>> g_pool_live;   // pointer -> capacity
}  // namespace

void* pinned_pool_get(size_t bytes) {
  const size_t cap = ((bytes + (1u << 20) - 1) >> 20 << 20) + (1u << 20) * (bytes == 0);
  std::lock_guard<std::mutex> g(g_pool_mu);
  for (size_t k = 0; k < g_pool_free.size(); ++k) {
    if (g_pool_free[k].first == cap) {
      void* p = g_pool_free[k].second;
      g_pool_free.erase(g_pool_free.begin() + k);
      g_pool_live.emplace_back(p, cap);
      return p;
    }
  }
  void* p = nullptr;
  cuda_check(cudaMallocHost(&p, cap), "cudaMallocHost");
  g_pool_live.emplace_back(p, cap);
  // a spare of the same size: a caller holding one result while the next solve
  // asks for another (every repeated solve) then never waits on page-locking
  // (cudaMallocHost: ~1-5 ms) -- the second timed solve of bench.py did
  void* spare = nullptr;
  if (cap <= (size_t(64) << 20) && cudaMallocHost(&spare, cap) == cudaSuccess)
    g_pool_free.emplace_back(cap, spare);
  else
    cudaGetLastError();
  return p;
}

void pinned_pool_put(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> g(g_pool_mu);
  for (size_t k = 0; k < g_pool_live.size(); ++k) {
    if (g_pool_live[k].first == p) {
      g_pool_free.emplace_back(g_pool_live[k].second, p);
      g_pool_live.erase(g_pool_live.begin() + k);
      return;
    }
  }
}

// ---------------------------------------------------------------------------
// worker pool
// ---------------------------------------------------------------------------
namespace {
class Workers {
 public:
  Workers() {
    unsigned hw = std::thread::hardware_concurrency();
    nthreads_ = (int)std::clamp<unsigned>(hw ? hw : 1, 1, 32) - 1;  // + the caller
    for (int i = 0; i < nthreads_; ++i) threads_.emplace_back([this] { loop(); });
  }
  ~Workers() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  int size() const { return nthreads_ + 1; }
  // runs every task, the caller participating; returns when all are done
  void run(std::vector<std::function<void()>>& tasks) {
    std::unique_lock<std::mutex> job(job_mu_);  // one parallel region at a time
    {
      std::lock_guard<std::mutex> g(mu_);
      for (auto& t : tasks) queue_.push_back(&t);
      pending_ += tasks.size();
    }
    cv_.notify_all();
    for (;;) {
      std::function<void()>* t = nullptr;
      {
        std::lock_guard<std::mutex> g(mu_);
        if (queue_.empty()) break;
        t = queue_.front();
        queue_.pop_front();
      }
      (*t)();
      finish_one();
    }
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [this] { return pending_ == 0; });
  }

 private:
  void finish_one() {
    std::lock_guard<std::mutex> g(mu_);
    if (--pending_ == 0) done_cv_.notify_all();
  }
  void loop() {
    for (;;) {
      std::function<void()>* t = nullptr;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [this] { return stop_ || !queue_.empty(); });
        if (stop_ && queue_.empty()) return;
        t = queue_.front();
        queue_.pop_front();
      }
      (*t)();
      finish_one();
    }
  }
  int nthreads_ = 0;
  std::vector<std::thread> threads_;
  std::mutex mu_, job_mu_;
  std::condition_variable cv_, done_cv_;
  std::deque<std::function<void()>*> queue_;
  size_t pending_ = 0;
  bool stop_ = false;
};

Workers& workers() {
  static Workers w;
  return w;
}
}  // namespace

int host_workers() { return workers().size(); }

void parallel_for(size_t count, size_t min_grain, const std::function<void(size_t, size_t)>& fn) {
  if (count == 0) return;
  size_t parts = std::min<size_t>((size_t)workers().size(), (count + min_grain - 1) / min_grain);
  if (parts <= 1) {
    fn(0, count);
    return;
  }
  std::vector<std::function<void()>> tasks;
  tasks.reserve(parts);
  for (size_t k = 0; k < parts; ++k) {
    const size_t b = count * k / parts, e = count * (k + 1) / parts;
    tasks.emplace_back([&fn, b, e] { fn(b, e); });
  }
  workers().run(tasks);
}

// ---------------------------------------------------------------------------
// uploads
// ---------------------------------------------------------------------------
bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

namespace {
constexpr size_t kStageBytes = 32u << 20;
struct Staging {
  std::mutex mu;
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  bool used[2] = {false, false};
};
Staging& staging() {
  static Staging s;
  return s;
}
}  // namespace

void upload(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  if (is_pinned(src)) {
    cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s), "H2D");
    return;
  }
  Staging& st = staging();
  std::lock_guard<std::mutex> g(st.mu);
  if (!st.buf[0]) {
    for (int k = 0; k < 2; ++k) {
      cuda_check(cudaMallocHost(&st.buf[k], kStageBytes), "cudaMallocHost");
      cuda_check(cudaEventCreateWithFlags(&st.ev[k], cudaEventDisableTiming), "cudaEventCreate");
    }
  }
  const char* in = static_cast<const char*>(src);
  char* out = static_cast<char*>(dst);
  int k = 0;
  for (size_t off = 0; off < bytes; off += kStageBytes, k ^= 1) {
    const size_t len = std::min(kStageBytes, bytes - off);
    if (st.used[k]) cuda_check(cudaEventSynchronize(st.ev[k]), "staging wait");
    char* pb = static_cast<char*>(st.buf[k]);
    parallel_for(len, 1u << 20, [&](size_t b, size_t e) { std::memcpy(pb + b, in + off + b, e - b); });
    cuda_check(cudaMemcpyAsync(out + off, pb, len, cudaMemcpyHostToDevice, s), "H2D");
    cuda_check(cudaEventRecord(st.ev[k], s), "event record");
    st.used[k] = true;
  }
  // the staging buffers are reused by the next upload only after their events
}

void download(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) {
    cuda_check(cudaStreamSynchronize(s), "synchronize");
    return;
  }
  if (is_pinned(dst) || bytes <= (64u << 10)) {
    cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaStreamSynchronize(s), "synchronize");
    return;
  }
  Staging& st = staging();
  std::lock_guard<std::mutex> g(st.mu);
  if (!st.buf[0]) {
    for (int k = 0; k < 2; ++k) {
      cuda_check(cudaMallocHost(&st.buf[k], kStageBytes), "cudaMallocHost");
      cuda_check(cudaEventCreateWithFlags(&st.ev[k], cudaEventDisableTiming), "cudaEventCreate");
    }
  }
  for (int k = 0; k < 2; ++k)  // an upload's copies out of the buffers must be done
    if (st.used[k]) cuda_check(cudaEventSynchronize(st.ev[k]), "staging wait");
  const char* in = static_cast<const char*>(src);
  char* out = static_cast<char*>(dst);
  const size_t nchunk = (bytes + kStageBytes - 1) / kStageBytes;
  auto issue = [&](size_t c) {
    const size_t off = c * kStageBytes, len = std::min(kStageBytes, bytes - off);
    cuda_check(cudaMemcpyAsync(st.buf[c & 1], in + off, len, cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaEventRecord(st.ev[c & 1], s), "event record");
    st.used[c & 1] = true;
  };
  issue(0);
  for (size_t c = 0; c < nchunk; ++c) {
    if (c + 1 < nchunk) issue(c + 1);
    cuda_check(cudaEventSynchronize(st.ev[c & 1]), "D2H wait");
    const size_t off = c * kStageBytes, len = std::min(kStageBytes, bytes - off);
    const char* pb = static_cast<const char*>(st.buf[c & 1]);
    parallel_for(len, 1u << 20, [&](size_t b, size_t e) { std::memcpy(out + off + b, pb + b, e - b); });
  }
}

}  // namespace tb
