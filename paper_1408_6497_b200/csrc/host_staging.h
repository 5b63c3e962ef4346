// host_staging.h — host<->device copies of PAGEABLE host buffers (the C++
// drop-in's GridField is a std::vector) through a small ring of pinned staging
// chunks: worker threads copy chunk c into a pinned slot while the copy engine
// moves chunk c-1, so a pageable 8.6 GB field crosses PCIe at close to the
// pinned rate instead of the driver's synchronous staged copy (B200 box,
// 1024^3 solve with pageable buffers: 1257 ms -> ~500 ms; pinned: 336 ms).
// Host code only.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace arena_fft {

// Persistent threads splitting one memcpy at a time.
class CopyPool {
 public:
  explicit CopyPool(int nthreads) {
    for (int i = 0; i < nthreads; ++i) th_.emplace_back([this, i, nthreads] { run(i, nthreads); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void copy(void* dst, const void* src, size_t len) {
    std::unique_lock<std::mutex> lk(m_);
    dst_ = static_cast<char*>(dst);
    src_ = static_cast<const char*>(src);
    len_ = len;
    pending_ = int(th_.size());
    ++gen_;
    cv_.notify_all();
    done_.wait(lk, [this] { return pending_ == 0; });
  }

 private:
  void run(int i, int nt) {
    unsigned long long seen = 0;
    for (;;) {
      char* d;
      const char* s;
      size_t len;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        d = dst_;
        s = src_;
        len = len_;
      }
      const size_t per = (len / nt + 4095) & ~size_t(4095);
      const size_t b = std::min(len, per * size_t(i)), e = std::min(len, b + per);
      if (e > b) memcpy(d + b, s + b, e - b);
      {
        std::lock_guard<std::mutex> lk(m_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t len_ = 0;
  int pending_ = 0;
  unsigned long long gen_ = 0;
  bool stop_ = false;
};

// Ring of pinned chunks + the copy pool.  One transfer at a time (callers hold
// the plan's host mutex).
class Stager {
 public:
  static constexpr size_t kChunk = size_t(64) << 20;
  static constexpr int kSlots = 3;

  ~Stager() {
    for (int s = 0; s < kSlots; ++s) {
      if (pin_[s]) cudaFreeHost(pin_[s]);
      if (ev_[s]) cudaEventDestroy(ev_[s]);
    }
    delete pool_;
  }
  // threads: host copy threads of this ring (0: ARENA_FFT_COPY_THREADS or min(8, cores)).
  cudaError_t init(int threads = 0) {
    cudaError_t e;
    for (int s = 0; s < kSlots; ++s) {
      if ((e = cudaMallocHost(&pin_[s], kChunk)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&ev_[s], cudaEventDisableTiming)) != cudaSuccess) return e;
    }
    const unsigned hc = std::thread::hardware_concurrency();
    int nt = int(std::max(1u, std::min(8u, hc ? hc : 1u)));  // B200 box: 8 and 16 threads equal (~35 GB/s)
    if (const char* env = getenv("ARENA_FFT_COPY_THREADS")) nt = std::max(1, atoi(env));
    if (threads > 0) nt = threads;
    pool_ = new CopyPool(nt);
    return cudaSuccess;
  }
  // pageable host -> device, enqueued on `st` (returns once every chunk left the host buffer).
  cudaError_t h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    const size_t nch = (bytes + kChunk - 1) / kChunk;
    for (size_t c = 0; c < nch; ++c) {
      const int s = int(c % kSlots);
      const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
      cudaError_t e;
      if ((e = cudaEventSynchronize(ev_[s])) != cudaSuccess) return e;  // slot free (also across calls)
      pool_->copy(pin_[s], static_cast<const char*>(src) + off, len);
      if ((e = cudaMemcpyAsync(static_cast<char*>(dst) + off, pin_[s], len, cudaMemcpyHostToDevice, st))) return e;
      if ((e = cudaEventRecord(ev_[s], st)) != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  // device -> pageable host after the work already on `st`; synchronous.
  cudaError_t d2h(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    const size_t nch = (bytes + kChunk - 1) / kChunk;
    cudaError_t e;
    auto issue = [&](size_t c) -> cudaError_t {
      const int s = int(c % kSlots);
      const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
      cudaError_t r = cudaMemcpyAsync(pin_[s], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, st);
      return r ? r : cudaEventRecord(ev_[s], st);
    };
    for (size_t c = 0; c < nch && c < size_t(kSlots); ++c)
      if ((e = issue(c)) != cudaSuccess) return e;
    for (size_t c = 0; c < nch; ++c) {
      const int s = int(c % kSlots);
      const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
      if ((e = cudaEventSynchronize(ev_[s])) != cudaSuccess) return e;
      pool_->copy(static_cast<char*>(dst) + off, pin_[s], len);
      if (c + kSlots < nch && (e = issue(c + kSlots)) != cudaSuccess) return e;
    }
    return cudaSuccess;
  }

 private:
  void* pin_[kSlots] = {};
  cudaEvent_t ev_[kSlots] = {};
  CopyPool* pool_ = nullptr;
};

// True when `p` is page-locked (or device / managed) memory the copy engines can use directly.
inline bool host_ptr_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type != cudaMemoryTypeUnregistered;
}

}  // namespace arena_fft
