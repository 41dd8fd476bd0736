// host.cu — host-buffer engine: the reference's blocking call shape
// (run_flavor(method, Flavor("cuda"), data, b) -> pair, kernels.py:591-640)
// on host memory, as one native call.
//
// An engine owns, per device: a non-blocking stream, two staging slots (pinned
// host + device, up to `chunk` bytes per operand each, allocated at 1 MiB and
// grown on the first larger input), grow-on-demand leaf partials
// and retire counters, a pinned result pair, and a small memcpy thread pool.
//
// tf_host_reduce(engine, method, dtype, hx, hy, n, leaf_log2, out_pair_host):
//   * n fits one chunk: stage -> H2D per operand -> tf_reduce (fused; its
//     last CTA stores the pair into mapped pinned memory) -> stream sync;
//   * larger: leaf-aligned chunks; H2D copies on a copy stream, leaf kernels
//     (tf_reduce_leaves into partials + c*chunk_leaves) on the compute stream,
//     two slots: the DMA of chunk c+1 overlaps the leaves of chunk c, and the
//     pool fills the other pinned slot meanwhile; tf_merge_tree
//     closes the tree.  Chunks are whole leaves, so the partials and the tree
//     are exactly those of tf_reduce on the whole array: bit-identical.
//   * page-locked inputs (cudaHostAlloc / cudaHostRegister) skip the staging
//     copy and DMA straight from the caller's memory; device pointers skip the
//     copies altogether.
//   * pageable staging is pipelined in 2 MiB pieces (the DMA of piece i
//     overlaps the pool's copy of piece i+1);
//   * small inputs (<= 128 KiB pageable / 256 KiB page-locked per operand)
//     skip the DMA: the kernel reads them over PCIe from page-locked memory.
// Calls on one engine are serialised by its mutex; the call blocks until the
// pair is in out_pair_host.
#include <cuda_runtime.h>
#include <sched.h>
#include <xmmintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges cost nothing unless a tool is attached

#include "status.h"

namespace tfb {
namespace {

// NVTX range for the host-side stages (ncu --nvtx / Nsight timelines).
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
};

// Fixed-size pool: copy(dst, src, bytes) splits the range into one piece per
// worker (plus the calling thread) and returns when all pieces are done.
// Workers spin for up to kSpinUs after a job (the next piece of a pipelined
// stage usually follows within microseconds) and then sleep on a condvar.
class CopyPool {
 public:
  static constexpr int kSpinUs = 200;
  explicit CopyPool(int workers) {
    for (int i = 0; i < workers; ++i) workers_.emplace_back([this, i] { run(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_.store(true);
      gen_.fetch_add(1);
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  int threads() const { return static_cast<int>(workers_.size()) + 1; }

  void copy(void* dst, const void* src, size_t bytes) {
    const int parts = threads();
    if (bytes < (size_t(256) << 10) || parts == 1) {
      std::memcpy(dst, src, bytes);
      return;
    }
    dst_ = static_cast<char*>(dst);
    src_ = static_cast<const char*>(src);
    bytes_ = bytes;
    pending_.store(parts - 1, std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> g(m_);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    piece(parts - 1);
    while (pending_.load(std::memory_order_acquire) != 0) pause();
  }

 private:
  static void pause() {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  void piece(int i) {
    const int parts = threads();
    const size_t per = ((bytes_ / parts) + 4095) & ~size_t(4095);
    const size_t lo = std::min(bytes_, per * i);
    const size_t hi = i == parts - 1 ? bytes_ : std::min(bytes_, per * (i + 1));
    if (hi > lo) std::memcpy(dst_ + lo, src_ + lo, hi - lo);
  }
  void run(int i) {
    uint64_t seen = 0;
    for (;;) {
      auto t0 = std::chrono::steady_clock::now();
      int k = 0;
      while (gen_.load(std::memory_order_acquire) == seen) {
        pause();
        if ((++k & 63) == 0 && std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(kSpinUs)) {
          std::unique_lock<std::mutex> lk(m_);
          cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
          break;
        }
      }
      seen = gen_.load(std::memory_order_acquire);
      if (stop_.load()) return;
      piece(i);
      pending_.fetch_sub(1, std::memory_order_release);
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_;
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> pending_{0};
  std::atomic<bool> stop_{false};
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0;
};

// Workers for the hybrid host path: start(job) runs job(worker) on every worker
// asynchronously (the calling thread keeps driving the GPU pipeline); wait()
// returns when all have finished.  Idle workers sleep on a condvar (no spin).
// Each worker clears FTZ/DAZ once: subnormals are in contract.
class LeafPool {
 public:
  explicit LeafPool(int workers) {
    for (int i = 0; i < workers; ++i) workers_.emplace_back([this, i] { run(i); });
  }
  ~LeafPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  int size() const { return static_cast<int>(workers_.size()); }
  void start(std::function<void(int)> job) {
    {
      std::lock_guard<std::mutex> g(m_);
      job_ = std::move(job);
      pending_ = size();
      ++gen_;
    }
    cv_.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [&] { return pending_ == 0; });
  }

 private:
  void run(int i) {
    _mm_setcsr(_mm_getcsr() & ~0x8040u);  // FTZ (bit 15) and DAZ (bit 6) off
    uint64_t seen = 0;
    for (;;) {
      std::function<void(int)> job;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        job = job_;
      }
      job(i);
      {
        std::lock_guard<std::mutex> g(m_);
        if (--pending_ == 0) done_.notify_all();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  std::function<void(int)> job_;
  uint64_t gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

enum class Mem { kPageable, kPinned, kDevice, kOtherDevice };

Mem classify(const void* p, int device) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return Mem::kPageable;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged)
    return a.device == device ? Mem::kDevice : Mem::kOtherDevice;
  if (a.type == cudaMemoryTypeHost) return Mem::kPinned;
  return Mem::kPageable;
}

}  // namespace

struct HostEngine {
  int device = 0;
  size_t chunk = 0;         // bytes per operand per slot, as allocated
  size_t chunk_target = 0;  // slot size large inputs grow to (creation argument)
  cudaStream_t stream = nullptr;   // kernels (and all work of single-chunk calls)
  cudaStream_t cstream = nullptr;  // H2D copies of multi-chunk calls
  char* pin[2] = {nullptr, nullptr};  // [x | y] per slot
  char* dev[2] = {nullptr, nullptr};
  cudaEvent_t h2d_done[2] = {nullptr, nullptr};  // slot's DMA finished (pinned slot reusable)
  cudaEvent_t k_done[2] = {nullptr, nullptr};    // slot's leaf kernel finished (device slot reusable)
  cudaEvent_t entry = nullptr;                   // the caller's stream at entry (device / pinned inputs)
  void* pair_pin = nullptr;  // mapped pinned: the last kernel stores the pair straight into it
  void* rows_pin = nullptr;  // mapped pinned row pairs (rows family), grown on demand
  size_t rows_pin_bytes = 0;
  void* partials = nullptr;
  size_t partials_bytes = 0;
  void* counters = nullptr;
  int64_t counters_len = 0;
  CopyPool* pool = nullptr;
  // staging copies of the hybrid path's GPU share: a small pool (TFB_HYBRID_COPY_THREADS,
  // default 3 incl. the caller) — the full pool's spinning workers take cores from the leaf
  // workers (pageable 2^26 f64 dot 13.8 -> 8.2 ms, profiles/r02_pageable_threads.txt)
  CopyPool* hpool = nullptr;
  LeafPool* leaf_pool = nullptr;   // hybrid host path workers (nullptr: GPU only)
  size_t hybrid_min_bytes = 0;     // per operand; smaller host inputs stay GPU-only
  void* hpairs = nullptr;          // pinned: leaf pairs the host workers computed
  size_t hpairs_bytes = 0;
  int64_t last_gpu_elems = 0, last_cpu_elems = 0;  // split of the last host-path call
  std::mutex mu;
};

namespace {

int cu(cudaError_t e) {
  if (e == cudaSuccess) return TF_OK;
  set_cuda_error(e);
  cudaGetLastError();
  return TF_ECUDA;
}

void release(HostEngine* g) {
  for (int b = 0; b < 2; ++b) {
    if (g->pin[b]) cudaFreeHost(g->pin[b]);
    if (g->dev[b]) cudaFree(g->dev[b]);
    if (g->h2d_done[b]) cudaEventDestroy(g->h2d_done[b]);
    if (g->k_done[b]) cudaEventDestroy(g->k_done[b]);
  }
  if (g->pair_pin) cudaFreeHost(g->pair_pin);
  if (g->rows_pin) cudaFreeHost(g->rows_pin);
  if (g->partials) cudaFree(g->partials);
  if (g->counters) cudaFree(g->counters);
  if (g->entry) cudaEventDestroy(g->entry);
  if (g->stream) cudaStreamDestroy(g->stream);
  if (g->cstream) cudaStreamDestroy(g->cstream);
  delete g->pool;
  delete g->hpool;
  delete g->leaf_pool;
  if (g->hpairs) cudaFreeHost(g->hpairs);
  delete g;
}

// Grow the scratch to at least (pb bytes, cnt counters); counters are zeroed.
int ensure_scratch(HostEngine* g, size_t pb, int64_t cnt) {
  int rc;
  if (pb > g->partials_bytes) {
    if ((rc = cu(cudaStreamSynchronize(g->stream)))) return rc;
    if (g->partials) cudaFree(g->partials);
    g->partials = nullptr;
    g->partials_bytes = 0;
    if ((rc = cu(cudaMalloc(&g->partials, pb)))) return rc;
    g->partials_bytes = pb;
  }
  if (cnt > g->counters_len) {
    if ((rc = cu(cudaStreamSynchronize(g->stream)))) return rc;
    if (g->counters) cudaFree(g->counters);
    g->counters = nullptr;
    g->counters_len = 0;
    if ((rc = cu(cudaMalloc(&g->counters, sizeof(unsigned) * cnt)))) return rc;
    if ((rc = cu(cudaMemsetAsync(g->counters, 0, sizeof(unsigned) * cnt, g->stream)))) return rc;
    g->counters_len = cnt;
  }
  return TF_OK;
}

// Grow the staging slots (first large input, or an explicit leaf larger than a
// slot — leaf_log2 up to 24 — so that a chunk always holds one whole leaf).
int grow_slots(HostEngine* g, size_t bytes) {
  if (bytes <= g->chunk) return TF_OK;
  int rc;
  if ((rc = cu(cudaStreamSynchronize(g->cstream)))) return rc;
  if ((rc = cu(cudaStreamSynchronize(g->stream)))) return rc;
  bytes = (bytes + 4095) & ~size_t(4095);
  for (int b = 0; b < 2; ++b) {
    cudaFreeHost(g->pin[b]);
    cudaFree(g->dev[b]);
    g->pin[b] = nullptr;
    g->dev[b] = nullptr;
  }
  g->chunk = 0;
  for (int b = 0; b < 2; ++b) {
    if ((rc = cu(cudaHostAlloc(reinterpret_cast<void**>(&g->pin[b]), 2 * bytes, cudaHostAllocDefault)))) return rc;
    if ((rc = cu(cudaMalloc(reinterpret_cast<void**>(&g->dev[b]), 2 * bytes)))) return rc;
  }
  g->chunk = bytes;
  return TF_OK;
}

constexpr size_t kPiece = size_t(2) << 20;
// Inputs up to this size per operand are read by the kernel in place from
// page-locked host memory (zero-copy) instead of being DMA'd first.  Pageable
// inputs must be copied into the staging slot first, which the DMA path
// overlaps with the transfer, hence the lower bound (measured crossovers,
// scripts/tiny_latency.py and scripts/host_engine_probe.py).
constexpr size_t kZeroCopyMaxPinned = size_t(256) << 10;
constexpr size_t kZeroCopyMaxPageable = size_t(128) << 10;

// Stage `bytes` of operand k (0 = x, 1 = y) from host `src` into device slot b.
int stage(HostEngine* g, cudaStream_t s, int b, int k, const char* src, size_t bytes, Mem kind, bool wait_slot,
          CopyPool* pool = nullptr) {
  if (!pool) pool = g->pool;
  char* d = g->dev[b] + k * g->chunk;
  if (kind == Mem::kPinned) return cu(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, s));
  if (wait_slot) {
    int rc = cu(cudaEventSynchronize(g->h2d_done[b]));  // the slot's previous DMA has drained
    if (rc) return rc;
  }
  // Pieces: the DMA of piece i overlaps the host copy of piece i+1.
  char* p = g->pin[b] + k * g->chunk;
  for (size_t off = 0; off < bytes; off += kPiece) {
    const size_t m = std::min(kPiece, bytes - off);
    pool->copy(p + off, src + off, m);
    int rc = cu(cudaMemcpyAsync(d + off, p + off, m, cudaMemcpyHostToDevice, s));
    if (rc) return rc;
  }
  return TF_OK;
}


size_t pair_size(int method, int dtype) {
  const int base = method & ~TF_TRACK_PRODUCT;
  return (base == TF_WIDE ? 8 : (dtype == TF_F64 ? 8 : 4)) * 2;
}

// Order the engine's streams after the caller's stream when an operand is device
// or page-locked memory the caller may still be writing.
int after_caller(HostEngine* g, Mem kx, Mem ky, void* after_stream) {
  if (kx == Mem::kPageable && ky == Mem::kPageable) return TF_OK;
  int rc;
  if ((rc = cu(cudaEventRecord(g->entry, static_cast<cudaStream_t>(after_stream))))) return rc;
  if ((rc = cu(cudaStreamWaitEvent(g->stream, g->entry, 0)))) return rc;
  return cu(cudaStreamWaitEvent(g->cstream, g->entry, 0));
}

// The staged path for host operands (pageable or page-locked) of n elements at
// leaf size lg: up to one chunk -> stage + tf_reduce; more -> leaf-aligned
// chunks, the DMA of chunk c+1 (copy stream) overlapping the leaves of chunk c
// (compute stream), then tf_merge_tree.  Chunks are whole leaves, so the result
// is bit-identical to tf_reduce on the whole array.  The pair lands in `out`
// (mapped pinned memory); returns after the streams drained.
int staged_reduce(HostEngine* g, int method, int dtype, const char* cx, const char* cy, int64_t n, int lg,
                  Mem kx, Mem ky, void* out) {
  Range range("staged_reduce");
  const size_t pair_bytes = pair_size(method, dtype);
  const size_t item = dtype == TF_F64 ? 8 : 4;
  const bool dot = cy != nullptr;
  size_t pb = 0;
  int64_t cnt = 0, leaves = 0;
  int rc = tf_workspace_size(method, dtype, 1, n, lg, &pb, &cnt, &leaves);
  if (rc) return rc;
  if ((rc = ensure_scratch(g, std::max<size_t>(pb, pair_bytes), std::max<int64_t>(cnt, 1)))) return rc;
  const int64_t L = int64_t(1) << lg;
  // slot size: the whole input up to the target, never less than one leaf
  const size_t want = std::max(std::min(static_cast<size_t>(n) * item, g->chunk_target),
                               static_cast<size_t>(std::min<int64_t>(L, n)) * item);
  if ((rc = grow_slots(g, want))) return rc;
  const int64_t chunk_leaves = std::max<int64_t>(1, static_cast<int64_t>(g->chunk / (L * item)));
  const int64_t chunk_elems = chunk_leaves * L;
  if (n <= chunk_elems) {
    const size_t bytes = n * item;
    if (n > 0) {
      Range r("h2d");
      if ((rc = stage(g, g->stream, 0, 0, cx, bytes, kx, true))) return rc;
      if (dot && (rc = stage(g, g->stream, 0, 1, cy, bytes, ky, true))) return rc;
      if ((rc = cu(cudaEventRecord(g->h2d_done[0], g->stream)))) return rc;
    }
    rc = tf_reduce(method, dtype, g->dev[0], dot ? g->dev[0] + g->chunk : nullptr, n, lg, out, g->partials,
                   g->partials_bytes, g->counters, g->counters_len, g->stream);
  } else {
    const int64_t nchunks = (n + chunk_elems - 1) / chunk_elems;
    for (int64_t c = 0; c < nchunks && rc == TF_OK; ++c) {
      Range r("chunk");
      const int b = static_cast<int>(c & 1);
      const int64_t lo = c * chunk_elems;
      const int64_t m = std::min(n, lo + chunk_elems) - lo;
      const size_t bytes = m * item;
      // Copies on cstream, leaf kernels on stream: the DMA of chunk c+1 overlaps
      // the leaves of chunk c.  Slot b is reused by chunk c+2 only after
      // kernel c finished (device side) and DMA c drained (host side, pageable).
      if (c >= 2 && (rc = cu(cudaStreamWaitEvent(g->cstream, g->k_done[b], 0)))) break;
      if ((rc = stage(g, g->cstream, b, 0, cx + lo * item, bytes, kx, c >= 2))) break;
      if (dot && (rc = stage(g, g->cstream, b, 1, cy + lo * item, bytes, ky, c >= 2))) break;
      if ((rc = cu(cudaEventRecord(g->h2d_done[b], g->cstream)))) break;
      if ((rc = cu(cudaStreamWaitEvent(g->stream, g->h2d_done[b], 0)))) break;
      rc = tf_reduce_leaves(method, dtype, g->dev[b], dot ? g->dev[b] + g->chunk : nullptr, m, lg,
                            static_cast<char*>(g->partials) + c * chunk_leaves * pair_bytes, g->stream);
      if (rc == TF_OK) rc = cu(cudaEventRecord(g->k_done[b], g->stream));
    }
    if (rc == TF_OK) rc = tf_merge_tree(method, dtype, g->partials, leaves, out, g->stream);
  }
  if (rc) {
    cudaStreamSynchronize(g->cstream);
    cudaStreamSynchronize(g->stream);
    return rc;
  }
  rc = cu(cudaStreamSynchronize(g->stream));
  if (rc == TF_OK) rc = cu(cudaStreamSynchronize(g->cstream));
  return rc;
}

extern "C" int tfb_host_leaves_avx512(int, int, const void*, const void*, int, int64_t, int64_t, void*);
extern "C" int tfb_host_leaves_base(int, int, const void*, const void*, int, int64_t, int64_t, void*);

int host_leaves(int method, int dtype, const void* x, const void* y, int lg, int64_t lo, int64_t hi, void* pairs) {
  // TFB_HOSTLEAF_BASE=1 forces the x86-64 baseline build (tests: both builds give the same bits)
  static const bool avx512 = !getenv("TFB_HOSTLEAF_BASE") && __builtin_cpu_supports("avx512f") &&
                             __builtin_cpu_supports("avx512vl") && __builtin_cpu_supports("avx512dq");
  return avx512 ? tfb_host_leaves_avx512(method, dtype, x, y, lg, lo, hi, pairs)
                : tfb_host_leaves_base(method, dtype, x, y, lg, lo, hi, pairs);
}

extern "C" int tfb_host_rows_avx512(int, int, const void*, const void*, int64_t, int64_t, int64_t, int64_t, int64_t,
                                    int, void*);
extern "C" int tfb_host_rows_base(int, int, const void*, const void*, int64_t, int64_t, int64_t, int64_t, int64_t, int,
                                  void*);

int host_rows(int method, int dtype, const void* x, const void* y, int64_t lo, int64_t hi, int64_t cols, int64_t ldx,
              int64_t ldy, int lg, void* pairs) {
  static const bool avx512 = !getenv("TFB_HOSTLEAF_BASE") && __builtin_cpu_supports("avx512f") &&
                             __builtin_cpu_supports("avx512vl") && __builtin_cpu_supports("avx512dq");
  return avx512 ? tfb_host_rows_avx512(method, dtype, x, y, lo, hi, cols, ldx, ldy, lg, pairs)
                : tfb_host_rows_base(method, dtype, x, y, lo, hi, cols, ldx, ldy, lg, pairs);
}

bool hybrid_methods(const HostEngine* g, int method, int dtype, int lg) {
  if (!g->leaf_pool || g->leaf_pool->size() == 0) return false;
  if (method & TF_TRACK_PRODUCT) return false;  // TwoProduct dots stay on the device
  if (method < 0 || method > TF_KAHAN || (method == TF_WIDE && dtype != TF_F32)) return false;
  return lg >= (dtype == TF_F64 ? 9 : 10);
}

bool hybrid_applies(const HostEngine* g, int method, int dtype, int64_t n, int lg, size_t item) {
  return hybrid_methods(g, method, dtype, lg) && static_cast<size_t>(n) * item >= g->hybrid_min_bytes && (n >> lg) >= 2;
}

// The hybrid host path: the GPU pipeline claims chunks of full leaves from the
// FRONT of the array while the leaf workers claim blocks of full leaves from the
// BACK (work stealing, no calibration); they meet wherever the two rates put
// them.  The host pairs are uploaded into their leaf slots, the partial last
// leaf (if any) is reduced on the GPU, and tf_merge_tree builds the one balanced
// tree over all leaf pairs — bit-identical to tf_reduce for every split.
int hybrid_reduce(HostEngine* g, int method, int dtype, const char* cx, const char* cy, int64_t n, int lg, Mem kx,
                  Mem ky, void* out) {
  Range range("hybrid_reduce");
  const size_t pair_bytes = pair_size(method, dtype);
  const size_t item = dtype == TF_F64 ? 8 : 4;
  const bool dot = cy != nullptr;
  const int64_t L = int64_t(1) << lg;
  const int64_t P = (n + L - 1) / L;
  const int64_t Pfull = n / L;
  size_t pb = 0;
  int64_t cnt = 0, leaves = 0;
  int rc = tf_workspace_size(method, dtype, 1, n, lg, &pb, &cnt, &leaves);
  if (rc) return rc;
  if ((rc = ensure_scratch(g, std::max<size_t>(pb, P * pair_bytes), std::max<int64_t>(cnt, 1)))) return rc;
  if ((rc = grow_slots(g, std::max(std::min(static_cast<size_t>(n) * item, g->chunk_target),
                                    static_cast<size_t>(L) * item))))
    return rc;
  if (static_cast<size_t>(P) * pair_bytes > g->hpairs_bytes) {
    if ((rc = cu(cudaStreamSynchronize(g->stream)))) return rc;
    if (g->hpairs) cudaFreeHost(g->hpairs);
    g->hpairs = nullptr;
    g->hpairs_bytes = 0;
    if ((rc = cu(cudaHostAlloc(&g->hpairs, P * pair_bytes, cudaHostAllocDefault)))) return rc;
    g->hpairs_bytes = P * pair_bytes;
  }
  // Claim granularity: GPU chunks of at most a slot and at most 1/8 of the leaves (a
  // first chunk of half the array would leave the host idle), host blocks of at most
  // 4 MiB per operand and small enough that every worker gets several.
  const int64_t slot_leaves = std::max<int64_t>(1, static_cast<int64_t>(g->chunk / (L * item)));
  const int64_t chunk_leaves = std::max<int64_t>(1, std::min(slot_leaves, (P + 7) / 8));
  const int64_t workers = g->leaf_pool->size();
  const int64_t host_block = std::max<int64_t>(
      1, std::min(static_cast<int64_t>((size_t(4) << 20) / (L * item)), Pfull / (4 * workers)));
  std::mutex cm;
  int64_t front = 0, back = Pfull;  // GPU owns [0, front), host owns [back, Pfull)
  std::atomic<int> host_rc{0};
  char* hp = static_cast<char*>(g->hpairs);
  g->leaf_pool->start([&](int) {
    for (;;) {
      int64_t lo, hi;
      {
        std::lock_guard<std::mutex> lk(cm);
        if (back <= front) return;
        hi = back;
        lo = std::max(front, back - host_block);
        back = lo;
      }
      if (host_leaves(method, dtype, cx, cy, lg, lo, hi, hp + lo * pair_bytes) != 0) host_rc.store(-1);
    }
  });
  // GPU side: chunks from the front; a chunk is claimed only when a staging slot
  // is free (host wait), so the device never runs ahead of the link
  // While it waits for a staging slot the calling thread reduces single leaves from the back
  // too (its core would otherwise idle; TFB_HYBRID_CALLER_WORKS=0: sleep on the event instead).
  static const bool caller_works = !getenv("TFB_HYBRID_CALLER_WORKS") || atoi(getenv("TFB_HYBRID_CALLER_WORKS")) != 0;
  auto wait_slot = [&](int b) -> int {
    if (!caller_works) return cu(cudaEventSynchronize(g->k_done[b]));
    const unsigned csr = _mm_getcsr();
    _mm_setcsr(csr & ~0x8040u);  // FTZ / DAZ off, like the workers
    int r = TF_OK;
    for (;;) {
      const cudaError_t q = cudaEventQuery(g->k_done[b]);
      if (q == cudaSuccess) break;
      if (q != cudaErrorNotReady) {
        r = cu(q);
        break;
      }
      int64_t lo, hi;
      {
        std::lock_guard<std::mutex> lk(cm);
        if (back <= front) {
          lo = hi = 0;
        } else {
          hi = back;
          lo = std::max(front, back - 1);
          back = lo;
        }
      }
      if (hi == lo) {  // nothing left to steal: sleep until the slot is free
        r = cu(cudaEventSynchronize(g->k_done[b]));
        break;
      }
      if (host_leaves(method, dtype, cx, cy, lg, lo, hi, hp + lo * pair_bytes) != 0) host_rc.store(-1);
    }
    _mm_setcsr(csr);
    return r;
  };
  int64_t c = 0;
  for (;; ++c) {
    int64_t lo, hi;
    const int b = static_cast<int>(c & 1);
    if (c >= 2 && (rc = wait_slot(b))) break;
    {
      std::lock_guard<std::mutex> lk(cm);
      if (front >= back) break;
      lo = front;
      hi = std::min(back, front + chunk_leaves);
      front = hi;
    }
    Range r("gpu chunk");
    const size_t bytes = static_cast<size_t>(hi - lo) * L * item;
    if ((rc = stage(g, g->cstream, b, 0, cx + lo * L * item, bytes, kx, false, g->hpool))) break;
    if (dot && (rc = stage(g, g->cstream, b, 1, cy + lo * L * item, bytes, ky, false, g->hpool))) break;
    if ((rc = cu(cudaEventRecord(g->h2d_done[b], g->cstream)))) break;
    if ((rc = cu(cudaStreamWaitEvent(g->stream, g->h2d_done[b], 0)))) break;
    rc = tf_reduce_leaves(method, dtype, g->dev[b], dot ? g->dev[b] + g->chunk : nullptr, (hi - lo) * L, lg,
                          static_cast<char*>(g->partials) + lo * pair_bytes, g->stream);
    if (rc == TF_OK) rc = cu(cudaEventRecord(g->k_done[b], g->stream));
    if (rc) break;
  }
  if (rc) {  // stop the workers' claims, let them drain, then fail
    {
      std::lock_guard<std::mutex> lk(cm);
      back = front;
    }
    g->leaf_pool->wait();
    cudaStreamSynchronize(g->cstream);
    cudaStreamSynchronize(g->stream);
    return rc;
  }
  // the partial last leaf, if any: one more (small) GPU chunk
  if (Pfull < P) {
    const int b = static_cast<int>(c & 1);
    if (c >= 2 && (rc = cu(cudaEventSynchronize(g->k_done[b])))) return rc;
    const int64_t m = n - Pfull * L;
    if ((rc = stage(g, g->cstream, b, 0, cx + Pfull * L * item, m * item, kx, false))) return rc;
    if (dot && (rc = stage(g, g->cstream, b, 1, cy + Pfull * L * item, m * item, ky, false))) return rc;
    if ((rc = cu(cudaEventRecord(g->h2d_done[b], g->cstream)))) return rc;
    if ((rc = cu(cudaStreamWaitEvent(g->stream, g->h2d_done[b], 0)))) return rc;
    rc = tf_reduce_leaves(method, dtype, g->dev[b], dot ? g->dev[b] + g->chunk : nullptr, m, lg,
                          static_cast<char*>(g->partials) + Pfull * pair_bytes, g->stream);
    if (rc == TF_OK) rc = cu(cudaEventRecord(g->k_done[b], g->stream));
    if (rc) return rc;
  }
  g->leaf_pool->wait();
  if (host_rc.load()) return TF_EINVAL_ARG;
  const int64_t host_lo = front;  // == back after both sides stopped
  if (host_lo < Pfull &&
      (rc = cu(cudaMemcpyAsync(static_cast<char*>(g->partials) + host_lo * pair_bytes, hp + host_lo * pair_bytes,
                               static_cast<size_t>(Pfull - host_lo) * pair_bytes, cudaMemcpyHostToDevice,
                               g->stream))))
    return rc;
  if ((rc = tf_merge_tree(method, dtype, g->partials, P, out, g->stream))) return rc;
  if ((rc = cu(cudaStreamSynchronize(g->stream)))) return rc;
  if ((rc = cu(cudaStreamSynchronize(g->cstream)))) return rc;
  g->last_cpu_elems = (Pfull - host_lo) * L;
  g->last_gpu_elems = n - g->last_cpu_elems;
  return TF_OK;
}
}  // namespace
}  // namespace tfb

using tfb::HostEngine;

extern "C" {

int tf_host_engine_create(int device, int threads, size_t chunk_bytes, void** engine) {
  if (!engine) return TF_EINVAL_ARG;
  *engine = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) return tfb::record_cuda_error();
  if (device < 0 || device >= ndev) return TF_EINVAL_ARG;
  if (chunk_bytes == 0) chunk_bytes = size_t(16) << 20;
  // A chunk must hold at least one maximal leaf (2^16 f64 = 512 KiB).
  chunk_bytes = std::max(chunk_bytes, size_t(1) << 20);
  chunk_bytes = (chunk_bytes + 4095) & ~size_t(4095);
  if (threads <= 0) {
    const unsigned hw = std::thread::hardware_concurrency();
    threads = static_cast<int>(std::min(8u, std::max(1u, hw / 2)));
  }
  tfb::DeviceGuard guard(device);
  auto* g = new HostEngine();
  g->device = device;
  // Slots start at 1 MiB (fast creation, small calls never pay for more) and grow
  // to chunk_bytes the first time a larger input arrives.
  g->chunk_target = chunk_bytes;
  g->chunk = std::min(chunk_bytes, size_t(1) << 20);
  int rc = TF_OK;
  auto step = [&](cudaError_t e) {
    if (rc == TF_OK) rc = tfb::cu(e);
  };
  step(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
  step(cudaStreamCreateWithFlags(&g->cstream, cudaStreamNonBlocking));
  for (int b = 0; b < 2 && rc == TF_OK; ++b) {
    step(cudaHostAlloc(reinterpret_cast<void**>(&g->pin[b]), 2 * g->chunk, cudaHostAllocDefault));
    step(cudaMalloc(reinterpret_cast<void**>(&g->dev[b]), 2 * g->chunk));
    step(cudaEventCreateWithFlags(&g->h2d_done[b], cudaEventDisableTiming));
    // k_done is host-waited only by the hybrid path, whose caller should sleep (its core
    // belongs to the host workers), not spin
    step(cudaEventCreateWithFlags(&g->k_done[b], cudaEventDisableTiming | cudaEventBlockingSync));
  }
  step(cudaHostAlloc(&g->pair_pin, 16, cudaHostAllocMapped));
  step(cudaEventCreateWithFlags(&g->entry, cudaEventDisableTiming));
  if (rc != TF_OK) {
    tfb::release(g);
    return rc;
  }
  g->pool = new tfb::CopyPool(threads - 1);
  {
    const char* e = getenv("TFB_HYBRID_COPY_THREADS");
    const int hc = std::max(1, std::min(e ? atoi(e) : 3, threads));
    g->hpool = new tfb::CopyPool(hc - 1);
  }
  // hybrid host path: all cores but the caller's by default (TFB_HYBRID_THREADS,
  // 0 = GPU only), for host inputs >= TFB_HYBRID_MIN_MB (default 8) per operand
  {
    const char* e = getenv("TFB_HYBRID_THREADS");
    int ht = e ? atoi(e) : -1;
    if (ht < 0) {  // the CPUs this process may run on (its affinity mask), minus the caller's
      cpu_set_t set;
      CPU_ZERO(&set);
      const int n = sched_getaffinity(0, sizeof(set), &set) == 0 ? CPU_COUNT(&set)
                                                                  : static_cast<int>(std::thread::hardware_concurrency());
      ht = std::max(1, n) - 1;
    }
    const char* mb = getenv("TFB_HYBRID_MIN_MB");
    g->hybrid_min_bytes = (mb ? static_cast<size_t>(atoll(mb)) : size_t(8)) << 20;
    g->leaf_pool = ht > 0 ? new tfb::LeafPool(ht) : nullptr;
  }
  *engine = g;
  return TF_OK;
}

int tf_host_engine_destroy(void* engine) {
  if (!engine) return TF_OK;
  auto* g = static_cast<HostEngine*>(engine);
  {
    tfb::DeviceGuard guard(g->device);
    std::lock_guard<std::mutex> lk(g->mu);
    cudaStreamSynchronize(g->stream);
  }
  tfb::DeviceGuard guard(g->device);
  tfb::release(g);
  return TF_OK;
}

int tf_host_engine_threads(const void* engine) {
  return engine ? static_cast<const HostEngine*>(engine)->pool->threads() : 0;
}

int tf_host_engine_hybrid(void* engine, int threads, size_t min_bytes) {
  if (!engine) return TF_EINVAL_ARG;
  auto* g = static_cast<HostEngine*>(engine);
  std::lock_guard<std::mutex> lk(g->mu);
  if (threads >= 0) {
    delete g->leaf_pool;
    g->leaf_pool = threads > 0 ? new tfb::LeafPool(threads) : nullptr;
  }
  g->hybrid_min_bytes = min_bytes;
  return TF_OK;
}

int tf_host_engine_last_split(const void* engine, int64_t* gpu_elems, int64_t* host_elems) {
  if (!engine || !gpu_elems || !host_elems) return TF_EINVAL_ARG;
  const auto* g = static_cast<const HostEngine*>(engine);
  *gpu_elems = g->last_gpu_elems;
  *host_elems = g->last_cpu_elems;
  return TF_OK;
}

int tf_host_rows(int method, int dtype, const void* x, const void* y, int64_t rows, int64_t cols, int64_t ldx,
                 int64_t ldy, int leaf_log2, int64_t row_lo, int64_t row_hi, void* out_pairs) {
  if (dtype != TF_F32 && dtype != TF_F64) return TF_EINVAL_DTYPE;
  if (method < 0 || method > TF_KAHAN) return TF_EINVAL_METHOD;
  if (method == TF_WIDE && dtype != TF_F32) return TF_EINVAL_DTYPE;
  if (rows < 0 || cols < 0 || (rows > 1 && (ldx < cols || (y && ldy < cols)))) return TF_EINVAL_SHAPE;
  const int lg = leaf_log2 ? leaf_log2 : tf_leaf_log2(dtype, rows * cols);
  if (lg < (dtype == TF_F64 ? 9 : 10) || lg > 24) return TF_EINVAL_ARG;
  if (row_lo < 0 || row_hi < row_lo || row_hi > rows || (cols > 0 && !x) || !out_pairs) return TF_EINVAL_ARG;
  const unsigned old = _mm_getcsr();
  _mm_setcsr(old & ~0x8040u);
  const int rc = tfb::host_rows(method, dtype, x, y, row_lo, row_hi, cols, ldx, ldy, lg, out_pairs);
  _mm_setcsr(old);
  return rc ? TF_EINVAL_ARG : TF_OK;
}

int tf_host_leaves(int method, int dtype, const void* x, const void* y, int64_t n, int leaf_log2, int64_t leaf_lo,
                   int64_t leaf_hi, void* out_pairs) {
  if (dtype != TF_F32 && dtype != TF_F64) return TF_EINVAL_DTYPE;
  if (method < 0 || method > TF_KAHAN) return TF_EINVAL_METHOD;
  if (method == TF_WIDE && dtype != TF_F32) return TF_EINVAL_DTYPE;
  if (n < 0) return TF_EINVAL_SHAPE;
  const int lg = leaf_log2 ? leaf_log2 : tf_leaf_log2(dtype, n);
  if (lg < (dtype == TF_F64 ? 9 : 10) || lg > 24) return TF_EINVAL_ARG;
  if (leaf_lo < 0 || leaf_hi < leaf_lo || (leaf_hi << lg) > n || !x || !out_pairs) return TF_EINVAL_ARG;
  const unsigned old = _mm_getcsr();
  _mm_setcsr(old & ~0x8040u);
  const int rc = tfb::host_leaves(method, dtype, x, y, lg, leaf_lo, leaf_hi, out_pairs);
  _mm_setcsr(old);
  return rc ? TF_EINVAL_ARG : TF_OK;
}

int tf_host_reduce(void* engine, int method, int dtype, const void* hx, const void* hy, int64_t n,
                   int leaf_log2, void* out_pair_host, void* after_stream) {
  if (!engine || !out_pair_host) return TF_EINVAL_ARG;
  if (dtype != TF_F32 && dtype != TF_F64) return TF_EINVAL_DTYPE;
  if (n < 0) return TF_EINVAL_SHAPE;
  if (n > 0 && !hx) return TF_EINVAL_ARG;
  auto* g = static_cast<HostEngine*>(engine);
  std::lock_guard<std::mutex> lk(g->mu);
  tfb::DeviceGuard guard(g->device);
  tfb::Range range("tf_host_reduce");
  const size_t pair_bytes = tfb::pair_size(method, dtype);
  const size_t item = dtype == TF_F64 ? 8 : 4;
  const bool dot = hy != nullptr;

  size_t pb = 0;
  int64_t cnt = 0, leaves = 0;
  int rc = tf_workspace_size(method, dtype, 1, n, leaf_log2, &pb, &cnt, &leaves);
  if (rc) return rc;
  const int lg = leaf_log2 ? leaf_log2 : tf_leaf_log2(dtype, n);
  if ((rc = tfb::ensure_scratch(g, std::max<size_t>(pb, pair_bytes), std::max<int64_t>(cnt, 1)))) return rc;

  const tfb::Mem kx = n > 0 ? tfb::classify(hx, g->device) : tfb::Mem::kPageable;
  const tfb::Mem ky = dot && n > 0 ? tfb::classify(hy, g->device) : kx;
  if (kx == tfb::Mem::kOtherDevice || ky == tfb::Mem::kOtherDevice) return TF_EINVAL_ARG;
  // Device or page-locked operands may still be in flight on the caller's
  // stream (NULL = the legacy default stream): order the engine's streams after it.
  if ((rc = tfb::after_caller(g, kx, ky, after_stream))) return rc;
  g->last_gpu_elems = n;  // every path below but the hybrid one reduces everything on the GPU
  g->last_cpu_elems = 0;
  if (kx == tfb::Mem::kDevice && ky == tfb::Mem::kDevice) {  // already resident: plain tf_reduce
    rc = tf_reduce(method, dtype, hx, hy, n, leaf_log2, g->pair_pin, g->partials, g->partials_bytes,
                   g->counters, g->counters_len, g->stream);
    if (rc == TF_OK) rc = tfb::cu(cudaStreamSynchronize(g->stream));
    if (rc) {
      cudaStreamSynchronize(g->stream);
      return rc;
    }
    std::memcpy(out_pair_host, g->pair_pin, pair_bytes);
    return TF_OK;
  }
  if (kx == tfb::Mem::kDevice || ky == tfb::Mem::kDevice) return TF_EINVAL_ARG;  // mixed host/device operands
  const auto* cx = static_cast<const char*>(hx);
  const auto* cy = static_cast<const char*>(hy);
  const size_t bytes_all = static_cast<size_t>(n) * item;
  const bool pageable = kx == tfb::Mem::kPageable || (dot && ky == tfb::Mem::kPageable);
  if (n > 0 && bytes_all <= (pageable ? tfb::kZeroCopyMaxPageable : tfb::kZeroCopyMaxPinned)) {
    // Small input: no DMA at all.  The kernel reads the operands over PCIe
    // straight from page-locked host memory (the staging slot, or the caller's
    // own pinned buffer); one launch, one sync.
    const void* dx = hx;
    const void* dy = hy;
    if (kx == tfb::Mem::kPageable) {
      std::memcpy(g->pin[0], cx, bytes_all);
      dx = g->pin[0];
    } else if (cudaHostGetDevicePointer(const_cast<void**>(&dx), const_cast<void*>(hx), 0) != cudaSuccess) {
      cudaGetLastError();
      dx = nullptr;
    }
    if (dot) {
      if (ky == tfb::Mem::kPageable) {
        std::memcpy(g->pin[0] + g->chunk, cy, bytes_all);
        dy = g->pin[0] + g->chunk;
      } else if (cudaHostGetDevicePointer(const_cast<void**>(&dy), const_cast<void*>(hy), 0) != cudaSuccess) {
        cudaGetLastError();
        dy = nullptr;
      }
    }
    if (dx && (!dot || dy)) {
      rc = tf_reduce(method, dtype, dx, dot ? dy : nullptr, n, lg, g->pair_pin, g->partials, g->partials_bytes,
                     g->counters, g->counters_len, g->stream);
      if (rc) {
        cudaStreamSynchronize(g->stream);
        return rc;
      }
      if ((rc = tfb::cu(cudaStreamSynchronize(g->stream)))) return rc;
      std::memcpy(out_pair_host, g->pair_pin, pair_bytes);
      return TF_OK;
    }
  }
  if (tfb::hybrid_applies(g, method, dtype, n, lg, item)) {
    if ((rc = tfb::hybrid_reduce(g, method, dtype, cx, cy, n, lg, kx, ky, g->pair_pin))) return rc;
  } else {
    if ((rc = tfb::staged_reduce(g, method, dtype, cx, cy, n, lg, kx, ky, g->pair_pin))) return rc;
  }
  std::memcpy(out_pair_host, g->pair_pin, pair_bytes);
  return TF_OK;
}

int tf_host_reduce_rows(void* engine, int method, int dtype, const void* hx, const void* hy, int64_t rows,
                        int64_t cols, int64_t ldx, int64_t ldy, int leaf_log2, void* out_pairs_host,
                        void* after_stream) {
  if (!engine || (!out_pairs_host && rows > 0)) return TF_EINVAL_ARG;
  if (dtype != TF_F32 && dtype != TF_F64) return TF_EINVAL_DTYPE;
  if (rows < 0 || cols < 0) return TF_EINVAL_SHAPE;
  if (rows > 1 && (ldx < cols || (hy && ldy < cols))) return TF_EINVAL_SHAPE;
  if (rows == 1)  // one row is the 1-D reduction (chunked within the row)
    return tf_host_reduce(engine, method, dtype, hx, hy, cols, leaf_log2, out_pairs_host, after_stream);
  if (rows == 0) return TF_OK;
  if (cols > 0 && !hx) return TF_EINVAL_ARG;
  auto* g = static_cast<HostEngine*>(engine);
  std::lock_guard<std::mutex> lk(g->mu);
  tfb::DeviceGuard guard(g->device);
  tfb::Range range("tf_host_reduce_rows");
  const size_t pair_bytes = tfb::pair_size(method, dtype);
  const size_t item = dtype == TF_F64 ? 8 : 4;
  const bool dot = hy != nullptr;
  // the leaf size is the WHOLE matrix's (tf_reduce_rows resolves it from rows * cols),
  // so every row block reduces exactly as the single-launch call would
  int rc;
  size_t pb = 0;
  int64_t cnt = 0, leaves = 0;
  if ((rc = tf_workspace_size(method, dtype, rows, cols, leaf_log2, &pb, &cnt, &leaves))) return rc;
  const int lg = leaf_log2 ? leaf_log2 : tf_leaf_log2(dtype, rows * cols);
  if ((rc = tfb::ensure_scratch(g, std::max<size_t>(pb, pair_bytes), std::max<int64_t>(cnt, 1)))) return rc;
  if (static_cast<size_t>(rows) * pair_bytes > g->rows_pin_bytes) {
    if ((rc = tfb::cu(cudaStreamSynchronize(g->stream)))) return rc;
    if (g->rows_pin) cudaFreeHost(g->rows_pin);
    g->rows_pin = nullptr;
    g->rows_pin_bytes = 0;
    const size_t want = static_cast<size_t>(rows) * pair_bytes;
    if ((rc = tfb::cu(cudaHostAlloc(&g->rows_pin, want, cudaHostAllocMapped)))) return rc;
    g->rows_pin_bytes = want;
  }
  const tfb::Mem kx = cols > 0 ? tfb::classify(hx, g->device) : tfb::Mem::kPageable;
  const tfb::Mem ky = dot && cols > 0 ? tfb::classify(hy, g->device) : kx;
  if (kx == tfb::Mem::kOtherDevice || ky == tfb::Mem::kOtherDevice) return TF_EINVAL_ARG;
  if ((rc = tfb::after_caller(g, kx, ky, after_stream))) return rc;
  const size_t row_bytes = static_cast<size_t>(cols) * item;
  g->last_gpu_elems = rows * cols;
  g->last_cpu_elems = 0;
  if (kx == tfb::Mem::kDevice && ky == tfb::Mem::kDevice) {
    rc = tf_reduce_rows(method, dtype, hx, hy, rows, cols, ldx, ldy, lg, g->rows_pin, g->partials,
                        g->partials_bytes, g->counters, g->counters_len, g->stream);
  } else if (kx == tfb::Mem::kDevice || ky == tfb::Mem::kDevice) {
    return TF_EINVAL_ARG;  // mixed host/device operands
  } else if (row_bytes > g->chunk_target) {
    // Rows longer than a staging slot stream through leaf-aligned chunks, one row
    // at a time (the 1-D staged path at the matrix's leaf size, so each row is
    // bit-identical to tf_reduce_rows), instead of sizing the slots to a whole row.
    const auto* cx = static_cast<const char*>(hx);
    const auto* cy = static_cast<const char*>(hy);
    const bool hyb = tfb::hybrid_applies(g, method, dtype, cols, lg, item);
    int64_t gpu_el = 0, host_el = 0;
    for (int64_t r = 0; r < rows && rc == TF_OK; ++r) {
      const char* xr = cx + static_cast<size_t>(r) * ldx * item;
      const char* yr = dot ? cy + static_cast<size_t>(r) * ldy * item : nullptr;
      char* o = static_cast<char*>(g->rows_pin) + static_cast<size_t>(r) * pair_bytes;
      rc = hyb ? tfb::hybrid_reduce(g, method, dtype, xr, yr, cols, lg, kx, ky, o)
               : tfb::staged_reduce(g, method, dtype, xr, yr, cols, lg, kx, ky, o);
      gpu_el += hyb ? g->last_gpu_elems : cols;
      host_el += hyb ? g->last_cpu_elems : 0;
    }
    g->last_gpu_elems = gpu_el;
    g->last_cpu_elems = host_el;
  } else {
    // Row blocks, packed (leading dimension = cols) into the staging slots; the
    // copies of block b+1 (copy stream) overlap the reduction of block b.
    const size_t want = std::min(static_cast<size_t>(rows) * row_bytes, g->chunk_target);
    if ((rc = tfb::grow_slots(g, std::max(want, row_bytes)))) return rc;
    const int64_t block = std::max<int64_t>(1, static_cast<int64_t>(g->chunk / std::max<size_t>(row_bytes, 1)));
    const int64_t nblocks = (rows + block - 1) / block;
    const auto* cx = static_cast<const char*>(hx);
    const auto* cy = static_cast<const char*>(hy);
    tfb::CopyPool* cpool = g->pool;  // the hybrid path stages with its small pool (set below)
    auto stage_block = [&](int b, int k, const char* src, int64_t ld, int64_t r0, int64_t nr, tfb::Mem kind,
                           bool wait) -> int {
      const char* s0 = src + static_cast<size_t>(r0) * ld * item;
      if (ld == cols)
        return tfb::stage(g, g->cstream, b, k, s0, static_cast<size_t>(nr) * row_bytes, kind, wait, cpool);
      char* d = g->dev[b] + k * g->chunk;
      if (kind == tfb::Mem::kPinned)  // pitched DMA packs the rows
        return tfb::cu(cudaMemcpy2DAsync(d, row_bytes, s0, ld * item, row_bytes, nr, cudaMemcpyHostToDevice,
                                         g->cstream));
      if (wait) {
        int e = tfb::cu(cudaEventSynchronize(g->h2d_done[b]));
        if (e) return e;
      }
      char* p = g->pin[b] + k * g->chunk;
      for (int64_t r = 0; r < nr; ++r) cpool->copy(p + r * row_bytes, s0 + static_cast<size_t>(r) * ld * item, row_bytes);
      return tfb::cu(cudaMemcpyAsync(d, p, static_cast<size_t>(nr) * row_bytes, cudaMemcpyHostToDevice, g->cstream));
    };
    // Hybrid (as tf_host_reduce): the GPU claims row blocks from the front, the
    // engine's host workers whole rows from the back (csrc/hostleaf.cpp row
    // reducer: the same leaves and row tree), straight into the mapped row pairs.
    const bool hybrid = tfb::hybrid_methods(g, method, dtype, lg) && rows >= 2 &&
                        static_cast<size_t>(rows) * row_bytes >= g->hybrid_min_bytes;
    if (hybrid && g->hpool) cpool = g->hpool;
    std::mutex cm;
    int64_t front = 0, back = rows;  // GPU owns [0, front), host owns [back, rows)
    std::atomic<int> host_rc{0};
    // everything the workers' lambda captures lives at this scope (they run until wait())
    const int64_t workers = hybrid ? g->leaf_pool->size() : 1;
    const int64_t hb = std::max<int64_t>(
        1, std::min(static_cast<int64_t>((size_t(4) << 20) / std::max<size_t>(row_bytes, 1)), rows / (4 * workers)));
    char* const rp = static_cast<char*>(g->rows_pin);
    if (hybrid) {
      g->leaf_pool->start([&](int) {
        for (;;) {
          int64_t lo, hi;
          {
            std::lock_guard<std::mutex> lk(cm);
            if (back <= front) return;
            hi = back;
            lo = std::max(front, back - hb);
            back = lo;
          }
          if (tfb::host_rows(method, dtype, cx, cy, lo, hi, cols, ldx, ldy, lg, rp + lo * pair_bytes) != 0)
            host_rc.store(-1);
        }
      });
    }
    const int64_t gblock = hybrid ? std::max<int64_t>(1, std::min(block, (rows + 7) / 8)) : block;
    (void)nblocks;
    for (int64_t c = 0; rc == TF_OK; ++c) {
      const int b = static_cast<int>(c & 1);
      if (hybrid && c >= 2) {
        // as in hybrid_reduce: the calling thread reduces whole rows from the back while it
        // waits for the slot (rows of at most ~1 MiB at a time; TFB_HYBRID_CALLER_WORKS=0 sleeps)
        static const bool caller_works =
            !getenv("TFB_HYBRID_CALLER_WORKS") || atoi(getenv("TFB_HYBRID_CALLER_WORKS")) != 0;
        if (!caller_works || row_bytes > (size_t(2) << 20)) {  // a long row would keep the caller from the GPU pipeline
          if ((rc = tfb::cu(cudaEventSynchronize(g->k_done[b])))) break;
        } else {
          const int64_t cb = std::max<int64_t>(1, std::min<int64_t>(hb, (int64_t(1) << 20) / std::max<size_t>(row_bytes, 1)));
          const unsigned csr = _mm_getcsr();
          _mm_setcsr(csr & ~0x8040u);
          for (;;) {
            const cudaError_t q = cudaEventQuery(g->k_done[b]);
            if (q == cudaSuccess) break;
            if (q != cudaErrorNotReady) {
              rc = tfb::cu(q);
              break;
            }
            int64_t lo = 0, hi = 0;
            {
              std::lock_guard<std::mutex> lk(cm);
              if (back > front) {
                hi = back;
                lo = std::max(front, back - cb);
                back = lo;
              }
            }
            if (hi == lo) {
              rc = tfb::cu(cudaEventSynchronize(g->k_done[b]));
              break;
            }
            if (tfb::host_rows(method, dtype, cx, cy, lo, hi, cols, ldx, ldy, lg, rp + lo * pair_bytes) != 0)
              host_rc.store(-1);
          }
          _mm_setcsr(csr);
          if (rc) break;
        }
      }
      int64_t r0, nr;
      {
        std::lock_guard<std::mutex> lk(cm);
        if (front >= back) break;
        r0 = front;
        nr = std::min(back - front, gblock);
        front += nr;
      }
      const bool wait = !hybrid && c >= 2;
      if (wait && (rc = tfb::cu(cudaStreamWaitEvent(g->cstream, g->k_done[b], 0)))) break;
      if ((rc = stage_block(b, 0, cx, ldx, r0, nr, kx, wait))) break;
      if (dot && (rc = stage_block(b, 1, cy, ldy, r0, nr, ky, wait))) break;
      if ((rc = tfb::cu(cudaEventRecord(g->h2d_done[b], g->cstream)))) break;
      if ((rc = tfb::cu(cudaStreamWaitEvent(g->stream, g->h2d_done[b], 0)))) break;
      rc = tf_reduce_rows(method, dtype, g->dev[b], dot ? g->dev[b] + g->chunk : nullptr, nr, cols, cols, cols, lg,
                          static_cast<char*>(g->rows_pin) + static_cast<size_t>(r0) * pair_bytes, g->partials,
                          g->partials_bytes, g->counters, g->counters_len, g->stream);
      if (rc == TF_OK) rc = tfb::cu(cudaEventRecord(g->k_done[b], g->stream));
    }
    if (hybrid) {
      if (rc) {
        std::lock_guard<std::mutex> lk(cm);
        back = front;
      }
      g->leaf_pool->wait();
      if (rc == TF_OK && host_rc.load()) rc = TF_EINVAL_ARG;
    }
    g->last_gpu_elems = front * cols;
    g->last_cpu_elems = (rows - front) * cols;
  }
  if (rc) {
    cudaStreamSynchronize(g->cstream);
    cudaStreamSynchronize(g->stream);
    return rc;
  }
  if ((rc = tfb::cu(cudaStreamSynchronize(g->stream)))) return rc;
  std::memcpy(out_pairs_host, g->rows_pin, static_cast<size_t>(rows) * pair_bytes);
  return TF_OK;
}

}  // extern "C"
