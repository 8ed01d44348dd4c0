#include <cstdlib>
// Context, error reporting, per-kernel timing and host-only helpers of the C ABI.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <queue>

#include "api.cuh"
#include "common.cuh"

namespace mlk {

static thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};

void set_last_error(const std::string& msg) { g_last_error = msg; }

bool is_device_ptr(const void* ptr) {
  cudaPointerAttributes attr;
  cudaError_t e = cudaPointerGetAttributes(&attr, ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

int num_sms(int device) {
  static int cached[64] = {0};
  if (device >= 0 && device < 64 && cached[device]) return cached[device];
  int v = 0;
  CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  if (device >= 0 && device < 64) cached[device] = v;
  return v;
}

int64_t device_total_bytes(int device) {
  static int64_t cached[64] = {0};
  if (device >= 0 && device < 64 && cached[device]) return cached[device];
  cudaDeviceProp prop;
  CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
  if (device >= 0 && device < 64) cached[device] = (int64_t)prop.totalGlobalMem;
  return (int64_t)prop.totalGlobalMem;
}

namespace {
struct PinnedRing {
  static constexpr size_t kCap = (size_t)64 << 20;
  char* base = nullptr;
  size_t head = 0;
  int device = -1;
  struct Chunk {
    size_t off, len;
    cudaEvent_t ev;
  };
  std::deque<Chunk> live;
  std::vector<cudaEvent_t> pool;
  std::mutex mu;
};
PinnedRing g_ring[64];
}  // namespace

void upload_async(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  int dev = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  if (bytes == 0) return;
  if (bytes > PinnedRing::kCap / 4 || dev < 0 || dev >= 64) {
    CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
    return;
  }
  PinnedRing& r = g_ring[dev];
  std::lock_guard<std::mutex> lock(r.mu);
  if (!r.base) {
    CUDA_CHECK(cudaHostAlloc((void**)&r.base, PinnedRing::kCap, cudaHostAllocPortable));
    r.device = dev;
  }
  const size_t len = (bytes + 255) & ~(size_t)255;
  if (r.head + len > PinnedRing::kCap) r.head = 0;
  // wait for EVERY live chunk overlapping [head, head + len): after two wraps of the ring the
  // overlapping chunks need not be at the front of the deque (live holds the tail of one lap
  // followed by the start of the next, and copies on different streams complete out of order).
  // Checking only the front let a new upload overwrite staged job descriptors whose copy had not
  // run yet -- an illegal address in the next kernel (cfg5 basis, r01f / r01h).
  for (const auto& ch : r.live)
    if (ch.off < r.head + len && r.head < ch.off + ch.len) CUDA_CHECK(cudaEventSynchronize(ch.ev));
  // retire every completed chunk
  for (auto it = r.live.begin(); it != r.live.end();) {
    if (cudaEventQuery(it->ev) == cudaSuccess) {
      r.pool.push_back(it->ev);
      it = r.live.erase(it);
    } else {
      ++it;
    }
  }
  cudaGetLastError();  // cudaEventQuery's cudaErrorNotReady is not an error here
  char* stage = r.base + r.head;
  std::memcpy(stage, src, bytes);
  CUDA_CHECK(cudaMemcpyAsync(dst, stage, bytes, cudaMemcpyHostToDevice, s));
  cudaEvent_t ev;
  if (!r.pool.empty()) {
    ev = r.pool.back();
    r.pool.pop_back();
  } else {
    CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  CUDA_CHECK(cudaEventRecord(ev, s));
  r.live.push_back({r.head, len, ev});
  r.head += len;
}

std::atomic<int64_t> g_live_bytes{0};

// What was free at the context's first query, less what live handles (W, BSR values, shards,
// scratch) have taken since.  cudaMemGetInfo itself runs once per context: under NVML polling
// (the bench's clock sampler, nvidia-smi on the box) a call stalled the host by up to 500 ms,
// and one call per mlk_build_basis made cfg4 steps of 830 ms take up to 1330 ms (r02 spk).
int64_t ctx_avail_bytes(Ctx& c) {
  if (c.free_at_first_use < 0) {
    size_t freeb = 0, totalb = 0;
    CUDA_CHECK(cudaMemGetInfo(&freeb, &totalb));
    c.free_at_first_use = (int64_t)freeb;
    c.live_at_first_use = g_live_bytes.load();
  }
  return c.free_at_first_use - (g_live_bytes.load() - c.live_at_first_use);
}

int64_t Ctx::scratch_budget_bytes() {
  // a third of what is available, at least 256 MB so small problems never starve
  const int64_t avail = ctx_avail_bytes(*this);
  static const int64_t forced = [] {
    const char* e = std::getenv("MLK_SCRATCH_BUDGET_MB");  // diagnostics: force small batches
    return e ? (int64_t)std::atoll(e) << 20 : (int64_t)0;
  }();
  if (forced > 0) return forced;
  return std::max<int64_t>(avail / 3, (int64_t)256 << 20);
}

double* Ctx::scratch(const char* key, size_t doubles) {
  auto& e = scratch_cache[key];
  const size_t bytes = std::max<size_t>(doubles, 1) * sizeof(double);
  if (e.first && e.second >= bytes) return static_cast<double*>(e.first);
  if (e.first) {
    CUDA_CHECK(cudaFreeAsync(e.first, stream));
    g_live_bytes.fetch_sub((int64_t)e.second, std::memory_order_relaxed);
    e = {nullptr, 0};
  }
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes, stream) != cudaSuccess) {
    cudaGetLastError();
    CUDA_CHECK(cudaDeviceSynchronize());
    CUDA_CHECK(cudaMallocAsync(&p, bytes, stream));
  }
  g_live_bytes.fetch_add((int64_t)bytes, std::memory_order_relaxed);
  e = {p, bytes};
  return static_cast<double*>(p);
}

cudaEvent_t Ctx::get_event() {
  if (!event_pool.empty()) {
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CUDA_CHECK(cudaEventCreate(&e));
  return e;
}

void Ctx::flush_timing() {
  if (pending.empty()) return;
  CUDA_CHECK(cudaStreamSynchronize(stream));
  for (auto& p : pending) {
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, p.a, p.b));
    KStat& s = stats[p.name];
    s.launches += 1;
    s.ms += ms;
    event_pool.push_back(p.a);
    event_pool.push_back(p.b);
  }
  pending.clear();
}

void partition_lpt(const double* cost, int64_t n, int nranks, int32_t* owner) {
  std::vector<int64_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return cost[a] > cost[b]; });
  // min-heap of (load, rank); ties resolved to the lower rank
  using E = std::pair<double, int>;
  std::priority_queue<E, std::vector<E>, std::greater<E>> heap;
  for (int r = 0; r < nranks; r++) heap.push({0.0, r});
  for (int64_t k : idx) {
    E e = heap.top();
    heap.pop();
    owner[k] = e.second;
    e.first += cost[k];
    heap.push(e);
  }
}

void shard_plan(const int64_t* val_off, const int32_t* owner, int64_t n, int nranks, int64_t* shard_off,
                int64_t* shard_len) {
  for (int r = 0; r < nranks; r++) shard_len[r] = 0;
  for (int64_t k = 0; k < n; k++) {
    shard_off[k] = shard_len[owner[k]];
    shard_len[owner[k]] += val_off[k + 1] - val_off[k];
  }
}

}  // namespace mlk

using namespace mlk;

extern "C" {

const char* mlk_last_error(void) { return g_last_error.c_str(); }

const char* mlk_version(void) { return "mlk 0.1 (sm_100a, FP64 DMMA)"; }

int64_t mlk_launch_count(void) { return g_launches.load(); }

mlk_status mlk_ctx_create(int device, int nranks, int rank, const void* nccl_unique_id, void* cuda_stream,
                          mlk_ctx* out) {
  MLK_API_BEGIN
  MLK_REQUIRE(out != nullptr, "out is NULL");
  *out = nullptr;
  MLK_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "need 0 <= rank < nranks");
  int ndev = 0;
  CUDA_CHECK(cudaGetDeviceCount(&ndev));
  MLK_REQUIRE(device >= 0 && device < ndev, "invalid device ordinal");
  CUDA_CHECK(cudaSetDevice(device));
  {
    // keep freed stream-ordered memory in the pool across synchronisations (the default
    // threshold 0 returns it to the OS at every sync and re-maps it at the next allocation)
    cudaMemPool_t pool;
    CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    // Reuse of a block freed on another stream (the auxiliary stream of the basis merges, stream 0
    // of the handle frees) must not depend on whether that free happens to have completed when the
    // allocation is requested ("opportunistic" reuse): when it had not, the allocator took other
    // blocks, a later large request (cfg4: the 13.7 GB S / V buffers, the 1 GB W) found no block
    // and the pool grew -- 150-600 ms of driver time in ~1 step of 5 (cfg4 steps of 830 ms
    // measured 970-1470 ms, r02 spk; MLK_SLOW_MS showed the stalls inside cudaMallocAsync).
    // With internal dependencies only, every step takes the same blocks.
    if (std::getenv("MLK_POOL_OPPORTUNISTIC") == nullptr) {
      int off = 0;
      CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowOpportunistic, &off));
    }
  }
  auto* h = new mlk_ctx_s();
  h->c.device = device;
  h->c.nranks = nranks;
  h->c.rank = rank;
  if (cuda_stream) {
    h->c.stream = (cudaStream_t)cuda_stream;
  } else {
    cudaError_t e = cudaStreamCreateWithFlags(&h->c.stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete h;
      cuda_check(e, "cudaStreamCreate");
    }
    h->c.own_stream = true;
  }
  if (nccl_unique_id) {
    try {
      h->c.comm = comm_create(nranks, rank, nccl_unique_id);
    } catch (...) {
      if (h->c.own_stream) cudaStreamDestroy(h->c.stream);
      delete h;
      throw;
    }
  }
  *out = h;
  MLK_API_END
}

void mlk_ctx_destroy(mlk_ctx ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->c.device);
  cudaStreamSynchronize(ctx->c.stream);
  for (auto& p : ctx->c.pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : ctx->c.event_pool) cudaEventDestroy(e);
  for (auto& s : ctx->c.scratch_cache)
    if (s.second.first) cudaFreeAsync(s.second.first, ctx->c.stream);
  cudaStreamSynchronize(ctx->c.stream);
  if (ctx->c.aux_stream) {
    cudaStreamSynchronize(ctx->c.aux_stream);
    cudaStreamDestroy(ctx->c.aux_stream);
  }
  if (ctx->c.copy_stream) {
    cudaStreamSynchronize(ctx->c.copy_stream);
    cudaStreamDestroy(ctx->c.copy_stream);
    cudaEventDestroy(ctx->c.copy_ready);
  }
  if (ctx->c.comm) {
    try {
      comm_destroy(ctx->c.comm);
    } catch (...) {
    }
  }
  if (ctx->c.own_stream) cudaStreamDestroy(ctx->c.stream);
  delete ctx;
}

mlk_status mlk_ctx_wait_copies(mlk_ctx ctx) {
  MLK_API_BEGIN
  MLK_REQUIRE(ctx, "ctx is NULL");
  CUDA_CHECK(cudaSetDevice(ctx->c.device));
  if (ctx->c.copy_stream) CUDA_CHECK(cudaStreamSynchronize(ctx->c.copy_stream));
  MLK_API_END
}

void* mlk_ctx_stream(mlk_ctx ctx) { return ctx ? (void*)ctx->c.stream : nullptr; }

mlk_status mlk_ctx_set_timing(mlk_ctx ctx, int enable) {
  MLK_API_BEGIN
  MLK_REQUIRE(ctx, "ctx is NULL");
  ctx->c.flush_timing();
  ctx->c.timing = enable != 0;
  // pre-create the events of a few steps' timed launches, so that recording them inside a
  // timed region never waits on cudaEventCreate
  while (enable && ctx->c.event_pool.size() < 8192) {
    cudaEvent_t e;
    CUDA_CHECK(cudaEventCreate(&e));
    ctx->c.event_pool.push_back(e);
  }
  MLK_API_END
}

mlk_status mlk_ctx_reset_stats(mlk_ctx ctx) {
  MLK_API_BEGIN
  MLK_REQUIRE(ctx, "ctx is NULL");
  ctx->c.flush_timing();
  ctx->c.stats.clear();
  MLK_API_END
}

mlk_status mlk_ctx_kernel_stats(mlk_ctx ctx, int idx, int* count, char* name, int name_len,
                                int64_t* launches, double* ms) {
  MLK_API_BEGIN
  MLK_REQUIRE(ctx, "ctx is NULL");
  CUDA_CHECK(cudaSetDevice(ctx->c.device));
  ctx->c.flush_timing();
  if (count) *count = (int)ctx->c.stats.size();
  if (name == nullptr && launches == nullptr && ms == nullptr) return MLK_OK;
  MLK_REQUIRE(idx >= 0 && idx < (int)ctx->c.stats.size(), "stat index out of range");
  auto it = ctx->c.stats.begin();
  std::advance(it, idx);
  if (name && name_len > 0) {
    std::strncpy(name, it->first.c_str(), name_len - 1);
    name[name_len - 1] = 0;
  }
  if (launches) *launches = it->second.launches;
  if (ms) *ms = it->second.ms;
  MLK_API_END
}

mlk_status mlk_partition_lpt(const double* cost, int64_t n, int32_t nranks, int32_t* owner) {
  MLK_API_BEGIN
  MLK_REQUIRE(n >= 0 && nranks >= 1, "invalid sizes");
  MLK_REQUIRE(n == 0 || (cost && owner), "NULL pointer");
  for (int64_t k = 0; k < n; k++) MLK_REQUIRE(cost[k] >= 0.0, "negative cost");
  partition_lpt(cost, n, nranks, owner);
  MLK_API_END
}

mlk_status mlk_shard_plan(const int64_t* val_off, const int32_t* owner, int64_t n, int32_t nranks,
                          int64_t* shard_off, int64_t* shard_len) {
  MLK_API_BEGIN
  MLK_REQUIRE(n >= 0 && nranks >= 1, "invalid sizes");
  MLK_REQUIRE(val_off && shard_len && (n == 0 || (owner && shard_off)), "NULL pointer");
  for (int64_t k = 0; k < n; k++) MLK_REQUIRE(owner[k] >= 0 && owner[k] < nranks, "owner out of range");
  shard_plan(val_off, owner, n, nranks, shard_off, shard_len);
  MLK_API_END
}

}  // extern "C"
