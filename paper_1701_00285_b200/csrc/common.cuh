// Internal runtime of libmlk: error handling, context, device buffers, timed launches.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdlib>

#include <cstdint>
#include <cstdio>
#include <deque>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mlk.h"

namespace mlk {

// An error carrying an mlk_status; thrown inside the library, converted at the ABI edge.
struct Error : std::runtime_error {
  mlk_status status;
  Error(mlk_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

void set_last_error(const std::string& msg);

#define MLK_REQUIRE(cond, msg)                                                  \
  do {                                                                          \
    if (!(cond)) throw ::mlk::Error(MLK_ERR_INVALID_ARG, std::string(msg));     \
  } while (0)

inline void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    throw Error(MLK_ERR_OUT_OF_MEMORY, std::string(what) + ": " + cudaGetErrorString(e));
  }
  throw Error(MLK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CUDA_CHECK(x) ::mlk::cuda_check((x), #x)

struct KStat {
  int64_t launches = 0;
  double ms = 0.0;
};

struct Ctx {
  int device = 0, nranks = 1, rank = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  bool timing = false;
  std::map<std::string, KStat> stats;
  struct Pending {
    std::string name;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  // device memory free when the context first needed a scratch budget (cudaMemGetInfo is
  // slow and erratic -- 0.3 to 14 ms per call on B200 while NVML is polled -- so it is queried
  // once per context, not per call)
  int64_t free_at_first_use = -1;  // cudaMemGetInfo once per context (it stalls under NVML polling)
  int64_t live_at_first_use = 0;
  cudaStream_t copy_stream = nullptr;  // mlk_cw_export_async (created on first use)
  cudaStream_t aux_stream = nullptr;   // asynchronous basis merge levels (created on first use)
  cudaEvent_t copy_ready = nullptr;
  void* comm = nullptr;                // ncclComm_t of mlk_ctx_create with a unique id (comm.cu)
  int64_t scratch_budget_bytes();
  // grow-only scratch buffers kept across calls (ctx.cu): the symmetric C a kernels' partials
  // (up to a few x 10 GB) are re-used instead of re-allocated per product -- a stream-ordered
  // allocation of that size, when the pool must map memory, stalled the step by up to 80 ms (r02)
  std::map<std::string, std::pair<void*, size_t>> scratch_cache;
  double* scratch(const char* key, size_t doubles);

  cudaEvent_t get_event();
  void flush_timing();  // synchronize and fold pending events into stats
};

// Times a launch region with CUDA events on the context stream when timing is enabled.
struct TimedLaunch {
  Ctx& c;
  const char* name;
  cudaEvent_t a = nullptr;
  TimedLaunch(Ctx& ctx, const char* n) : c(ctx), name(n) {
    if (c.timing) {
      a = c.get_event();
      CUDA_CHECK(cudaEventRecord(a, c.stream));
    }
  }
  // never throws: it also runs while an exception unwinds the launch sequence; a failed
  // record drops the sample (the error itself surfaces at the next check_launch / CUDA_CHECK)
  ~TimedLaunch() {
    if (!c.timing || a == nullptr) return;
    cudaEvent_t b = nullptr;
    if (!c.event_pool.empty()) {  // pooled (set_timing pre-creates them): no driver call here
      b = c.event_pool.back();
      c.event_pool.pop_back();
    } else if (cudaEventCreate(&b) != cudaSuccess) {
      b = nullptr;
    }
    if (b == nullptr || cudaEventRecord(b, c.stream) != cudaSuccess) {
      if (b) c.event_pool.push_back(b);
      c.event_pool.push_back(a);
      return;
    }
    try {
      c.pending.push_back({name, a, b});
    } catch (...) {
      cudaEventDestroy(b);
    }
  }
};

extern std::atomic<int64_t> g_launches;

inline void check_launch(const char* name) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(MLK_ERR_CUDA, std::string("launch ") + name + ": " + cudaGetErrorString(e));
}

// Host -> device copy that returns immediately: small transfers are staged through a
// process-wide pinned ring buffer (a chunk is reused only after the event recorded behind its
// copy has completed), large ones go straight to cudaMemcpyAsync.  Pageable cudaMemcpyAsync
// would block the host until the stream reaches the copy.  dst: device memory of the current
// device; src: host memory.
void upload_async(void* dst, const void* src, size_t bytes, cudaStream_t s);

// bytes held by live DevBufs in this process (the scratch budget subtracts what handles keep)
extern std::atomic<int64_t> g_live_bytes;

// Stream-ordered device buffer.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(size_t count, cudaStream_t stream) { alloc(count, stream); }
  void alloc(size_t count, cudaStream_t stream) {
    release();
    s = stream;
    n = count;
    if (count) {
      if (cudaMallocAsync((void**)&p, count * sizeof(T), stream) != cudaSuccess) {
        // memory freed on another stream is reusable only once that free has completed:
        // drain the device and retry once before reporting out-of-memory
        cudaGetLastError();
        CUDA_CHECK(cudaDeviceSynchronize());
        CUDA_CHECK(cudaMallocAsync((void**)&p, count * sizeof(T), stream));
      }
      g_live_bytes.fetch_add((int64_t)(count * sizeof(T)), std::memory_order_relaxed);
    }
  }
  void zero() {
    if (n) CUDA_CHECK(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void upload(const T* host, size_t count) {
    if (count) upload_async(p, host, count * sizeof(T), s);
  }
  void upload(const std::vector<T>& v) {
    if (v.size() > n) alloc(v.size(), s);
    upload(v.data(), v.size());
  }
  std::vector<T> download(size_t count) const {
    std::vector<T> h(count);
    if (count) {
      CUDA_CHECK(cudaMemcpyAsync(h.data(), p, count * sizeof(T), cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
    }
    return h;
  }
  void release() {
    if (p) {
      cudaFreeAsync(p, s);
      g_live_bytes.fetch_sub((int64_t)(n * sizeof(T)), std::memory_order_relaxed);
    }
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    p = o.p; n = o.n; s = o.s;
    o.p = nullptr; o.n = 0;
    return *this;
  }
};

// True if ptr is device or managed memory usable by the current device.
bool is_device_ptr(const void* ptr);

// Read-only view of a host-or-device input as a device pointer (copied if on the host).
template <typename T>
struct DevIn {
  DevBuf<T> staged;
  const T* p = nullptr;
  DevIn(const T* src, size_t count, cudaStream_t s) {
    if (src == nullptr || count == 0) { p = src; return; }
    if (is_device_ptr(src)) { p = src; return; }
    staged.alloc(count, s);
    staged.upload(src, count);
    p = staged.p;
  }
};

// Write target: device pointer directly, or a staging buffer copied back by finish().
template <typename T>
struct DevOut {
  DevBuf<T> staged;
  T* dst;
  T* p;
  size_t count;
  cudaStream_t s;
  bool host;
  DevOut(T* out, size_t cnt, cudaStream_t stream) : dst(out), count(cnt), s(stream) {
    host = out != nullptr && cnt > 0 && !is_device_ptr(out);
    if (host) {
      staged.alloc(cnt, stream);
      p = staged.p;
    } else {
      p = out;
    }
  }
  void finish() {
    if (host) CUDA_CHECK(cudaMemcpyAsync(dst, p, count * sizeof(T), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Host-side phase timer, printed to stderr when MLK_TRACE is set (diagnostics only).
struct HostTrace {
  const char* what;
  bool on;
  std::chrono::steady_clock::time_point t0, last;
  explicit HostTrace(const char* w) : what(w), on(std::getenv("MLK_TRACE") != nullptr) {
    t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char* phase) {
    if (!on) return;
    auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[mlk] %s.%s %.3f ms\n", what, phase,
                 std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
  }
};

int num_sms(int device);
int64_t device_total_bytes(int device);  // cudaDeviceProp::totalGlobalMem, cached

}  // namespace mlk

struct mlk_ctx_s {
  mlk::Ctx c;
};
