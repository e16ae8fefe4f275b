// Host runtime: context, stream-ordered device memory, launch accounting, profiling.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <chrono>
#include <cstdlib>
#include <map>
#include <tuple>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/sconv_b200.h"

namespace sconvb {

// Internal error carrying a C-ABI status; converted at the boundary (capi.cu).
struct Error : std::runtime_error {
  sconv_status status;
  Error(sconv_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};
[[noreturn]] inline void fail(sconv_status s, const std::string& m) { throw Error(s, m); }
inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    if (e == cudaErrorMemoryAllocation) fail(SCONV_ERR_OOM, std::string(what) + ": " + cudaGetErrorString(e));
    fail(SCONV_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}
#define SCONV_CUDA(expr) ::sconvb::cuda_check((expr), #expr)

struct Ctx;

// Stream-ordered device allocation (cudaMallocAsync on the context stream; the pool keeps
// freed memory cached so steady-state layers do not hit the driver).
class DevBuf {
 public:
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      ptr_ = o.ptr_;
      bytes_ = o.bytes_;
      stream_ = o.stream_;
      o.ptr_ = nullptr;
      o.bytes_ = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t bytes, cudaStream_t s) {
    release();
    stream_ = s;
    if (bytes == 0) return;
    SCONV_CUDA(cudaMallocAsync(&ptr_, bytes, s));
    bytes_ = bytes;
  }
  // grow-only reuse for scratch
  void reserve(size_t bytes, cudaStream_t s) {
    if (bytes <= bytes_ && s == stream_) return;
    alloc(bytes, s);
  }
  void release() {
    if (ptr_) cudaFreeAsync(ptr_, stream_);
    ptr_ = nullptr;
    bytes_ = 0;
  }
  template <class T = void>
  T* get() const {
    return static_cast<T*>(ptr_);
  }
  size_t bytes() const { return bytes_; }

 private:
  void* ptr_ = nullptr;
  size_t bytes_ = 0;
  cudaStream_t stream_ = nullptr;
};

struct ProfileEntry {
  int64_t launches = 0;
  double total_ms = 0.0;
};

struct TuneKey {
  int c_in, c_out, dtype;
  bool operator<(const TuneKey& o) const {
    return std::tie(c_in, c_out, dtype) < std::tie(o.c_in, o.c_out, o.dtype);
  }
};

struct Ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  std::string err;
  int64_t launches = 0;

  // profiling (CUDA events around every launch on the context stream)
  bool profiling = false;
  std::string profile_only;  // non-empty: time only launches with this label
  struct Pending {
    std::string name;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  std::map<std::string, ProfileEntry> profile;
  std::vector<std::string> profile_names;  // stable order for the C API
  std::vector<std::pair<std::string, double>> last_records;  // individual launches since last clear

  // scratch (grow-only, stream ordered)
  DevBuf scratch_sort, scratch_misc, flush_buf;
  DevBuf gather_buf, gemm_out, plan_dev;
  DevBuf fused_counter;  // dynamic tile queue of the fused kernel
  DevBuf fused_ws;       // split work items' fp32 partials (fused kernel)
  // (sconv_ctx_destroy releases every DevBuf above before destroying the stream)
  // Pinned host staging, carved into fixed regions, used ONLY for device->host readbacks that
  // are followed by a stream sync (map sizes / flags). Host->device inputs of a map build are
  // generated on the device instead: lazy (network) map builds end without a sync, so a
  // staging region reused by the next build could be overwritten before its copy ran.
  static constexpr size_t kPinFlagsBytes = 8192, kPinReadbackBytes = 16384, kPinPlanBytes = 1 << 20;
  unsigned char* pinned = nullptr;
  void* pin_flags() { return pinned; }
  void* pin_readback() { return pinned + kPinFlagsBytes; }
  void* pin_plan() { return pinned + kPinFlagsBytes + kPinReadbackBytes; }

  std::map<TuneKey, std::pair<int, int>> tuned;  // (T_g, T_s)
  // gather IMT-lookup counter (SPEC.md:340 counter; acceptance #6), on when count_lookups
  bool count_lookups = false;
  unsigned long long* lookup_counter = nullptr;  // device, allocated with the context
  unsigned* done = nullptr;  // zero-initialised "last CTA" counter, reset by its user kernel
  unsigned* done_counter() { return done; }
  // bucket-sort state: histogram (kept zeroed by its scan kernel) + starts + cursors
  int* sort_state = nullptr;
  int* sort_hist() { return sort_state; }

  cudaEvent_t take_event();
  void resolve_profile();

  // host-side phase trace (SCONV_HOST_TRACE=1): (label, us since the trace epoch), buffered
  // and printed by the network forward at its end (printing inline would distort the times)
  std::vector<std::pair<const char*, double>> htrace;
  std::chrono::steady_clock::time_point htrace_t0 = std::chrono::steady_clock::now();
  static bool htrace_on() {
    static const bool on = [] {
      const char* e = std::getenv("SCONV_HOST_TRACE");
      return e && e[0] == '1';
    }();
    return on;
  }
  void hmark(const char* what) {
    if (htrace_on())
      htrace.emplace_back(what, std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - htrace_t0).count());
  }

  template <class F>
  void launch(const char* name, F&& f) {
    cudaEvent_t a = nullptr, b = nullptr;
    const bool timed = profiling && (profile_only.empty() || profile_only == name);
    if (timed) {
      a = take_event();
      b = take_event();
      SCONV_CUDA(cudaEventRecord(a, stream));
    }
    f();
    SCONV_CUDA(cudaGetLastError());
    ++launches;
    if (timed) {
      SCONV_CUDA(cudaEventRecord(b, stream));
      pending.push_back({name, a, b});
    }
  }
  void sync() { SCONV_CUDA(cudaStreamSynchronize(stream)); }
};

}  // namespace sconvb

struct sconv_ctx : sconvb::Ctx {};
