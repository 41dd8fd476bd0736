// tma.cuh — warp-specialised bulk-copy (TMA engine) variant of leaves_kernel.
// Included by reduce.cu after the shared device helpers.
//
// Same partition, same per-thread chains, same trees as leaves_kernel (so the
// results are bit-identical); only the loader differs:
//   * warp 8 (one elected lane) is the producer: for every full leaf it issues
//     cp.async.bulk (global -> shared, completion counted on an mbarrier) of
//     SR consecutive "rows" of 256 vectors (= SR*4 KiB per operand) into a
//     ring of NS stages;
//   * warps 0..7 are the consumers: thread t reads its vector row*256 + t of
//     every row straight from shared memory (conflict-free 16-byte loads),
//     runs the recurrence, and releases the stage (one arrive per warp);
//   * partial last leaves are read from global memory by the consumers with
//     the scalar path (the producer skips them).
// Consumers synchronise among themselves with named barrier 1 only.

namespace tfb {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

constexpr int kTmaConsumers = kThreads;        // 8 consumer warps
constexpr int kTmaThreads = kThreads + 32;     // + 1 producer warp

template <typename T, bool DOT, int NS, int SR>
struct TmaSmem {
  using VT = typename Vec<T>::type;
  static constexpr int kRowVecs = kThreads;                       // vectors per row
  static constexpr int kStageVecs = SR * kRowVecs;                 // per operand
  static constexpr size_t kStageBytes = sizeof(VT) * kStageVecs;   // per operand
  static constexpr size_t kBytes = NS * kStageBytes * (DOT ? 2 : 1) + 2 * NS * sizeof(uint64_t) + 64;
};

template <int M, typename T, bool DOT, int NS, int SR, int MINB = 1>
__global__ void __launch_bounds__(kTmaThreads, MINB) leaves_tma_kernel(
    const T* __restrict__ x, const T* __restrict__ y, int64_t ldx, int64_t ldy, int64_t rows,
    int64_t cols, int leaf_log2, int64_t P, Pair<typename Acc<M, T>::type>* __restrict__ partials,
    unsigned* __restrict__ counters, Pair<typename Acc<M, T>::type>* __restrict__ out,
    const PeerCtx* __restrict__ peer, uint32_t epoch, int chain_pf_kb) {
  using A = typename Acc<M, T>::type;
  using VT = typename Vec<T>::type;
  using L = TmaSmem<T, DOT, NS, SR>;
  constexpr int V = Vec<T>::V;
  extern __shared__ __align__(128) unsigned char tma_smem[];
  VT* sx = reinterpret_cast<VT*>(tma_smem);
  VT* sy = reinterpret_cast<VT*>(tma_smem + NS * L::kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(tma_smem + NS * L::kStageBytes * (DOT ? 2 : 1));
  uint64_t* empty = full + NS;
  __shared__ Pair<A> red[kWarps];
  __shared__ int s_last;

  const int R = (1 << leaf_log2) / (kThreads * V);
  const int64_t Lelems = int64_t(1) << leaf_log2;
  const int64_t units = rows * P;
  const int warp = threadIdx.x >> 5;

  // Cross-call overlap (chain_pf_kb >= 0: launched as a programmatic dependent): a CTA of
  // this grid becomes resident as soon as a CTA of the previous kernel frees its shared
  // memory, asks the L2 for the head of its first leaf (a hint, leaves_kernel's preamble),
  // and only then waits for the previous grid to complete — before any memory access.
  if (chain_pf_kb >= 0) {
    if (chain_pf_kb > 0 && threadIdx.x < 64 && static_cast<int64_t>(blockIdx.x) < units) {
      const int64_t r = blockIdx.x / P;
      const int64_t start = (blockIdx.x - r * P) * Lelems;
      int64_t bytes = (cols - start < Lelems ? cols - start : Lelems) * static_cast<int64_t>(sizeof(T));
      if (bytes > (static_cast<int64_t>(chain_pf_kb) << 10)) bytes = static_cast<int64_t>(chain_pf_kb) << 10;
      bytes &= ~int64_t(15);
      const int op = threadIdx.x & 1;
      const int64_t off = static_cast<int64_t>(threadIdx.x >> 1) * 16384;
      if (off < bytes && (DOT || op == 0)) {
        const char* p = reinterpret_cast<const char*>((op ? y + r * ldy : x + r * ldx) + start) + off;
        const unsigned sz = static_cast<unsigned>(bytes - off < 16384 ? bytes - off : 16384);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(sz) : "memory");
      }
    }
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (chain_pf_kb >= 0) asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == kWarps) {  // ---------------- producer warp ----------------
    if ((threadIdx.x & 31) != 0) return;
    int slot = 0;
    uint32_t phase = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      const int64_t r = u / P, l = u - r * P;
      const int64_t start = l * Lelems;
      if (start + Lelems > cols) continue;  // partial leaf: consumers read it directly
      const T* gx = x + r * ldx + start;
      const T* gy = DOT ? y + r * ldy + start : nullptr;
      for (int r0 = 0; r0 < R; r0 += SR) {
        const int nrow = R - r0 < SR ? R - r0 : SR;
        const uint32_t bytes = static_cast<uint32_t>(nrow * L::kRowVecs * sizeof(VT));
        TFB_CHECK(static_cast<int64_t>(r0 + nrow) * L::kRowVecs * V <= Lelems && start + Lelems <= cols);
        mbar_wait(&empty[slot], phase ^ 1u);
        mbar_arrive_expect_tx(&full[slot], bytes * (DOT ? 2u : 1u));
        bulk_g2s(sx + slot * L::kStageVecs, gx + static_cast<int64_t>(r0) * L::kRowVecs * V, bytes, &full[slot]);
        if constexpr (DOT)
          bulk_g2s(sy + slot * L::kStageVecs, gy + static_cast<int64_t>(r0) * L::kRowVecs * V, bytes,
                   &full[slot]);
        if (++slot == NS) { slot = 0; phase ^= 1u; }
      }
    }
    // This CTA has issued its last bulk copy: once every CTA has, the next kernel of the
    // stream may become resident (a kernel that needs no shared memory could otherwise sit
    // beside this grid from its start and run its prefetch preamble far too early).
    if (chain_pf_kb >= 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    return;
  }

  // ---------------- consumer warps (threads 0..255) ----------------
  const int t = threadIdx.x;
  int slot = 0;
  uint32_t phase = 0;
  unsigned pending = 0;  // leaf pairs of the current row stored but not yet retired
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t r = u / P, l = u - r * P;
    const int64_t start = l * Lelems;
    Pair<A> st = zero_pair<A>();
    if (start + Lelems <= cols) {
      for (int r0 = 0; r0 < R; r0 += SR) {
        const int nrow = R - r0 < SR ? R - r0 : SR;
        mbar_wait(&full[slot], phase);
        const VT* bx = sx + slot * L::kStageVecs + t;
        const VT* by = sy + slot * L::kStageVecs + t;
#pragma unroll 4
        for (int q = 0; q < nrow; ++q) {
          const VT a = bx[q * L::kRowVecs];
          if constexpr (DOT) {
            const VT b = by[q * L::kRowVecs];
#pragma unroll
            for (int j = 0; j < V; ++j) accumulate<M, T, true>(st, vget(a, j), vget(b, j));
          } else {
#pragma unroll
            for (int j = 0; j < V; ++j) accumulate<M, T, false>(st, vget(a, j), T(0));
          }
        }
        __syncwarp();
        if ((t & 31) == 0) mbar_arrive(&empty[slot]);
        if (++slot == NS) { slot = 0; phase ^= 1u; }
      }
    } else {
      st = leaf_chain<M, T, DOT, false, 1>(x + r * ldx, DOT ? y + r * ldy : nullptr, start, cols, R, t);
    }
    st = block_tree<M, A, 1, kTmaConsumers>(st, red, kThreads);
    if (P == 1) {
      finish_root<M, A, 1, kTmaConsumers>(st, out + r, peer, epoch, red);
      continue;
    }
    if (t == 0) partials[u] = st;
    ++pending;
    const int64_t un = u + gridDim.x;
    if (un < units && un / P == r) continue;  // one ticket per row per CTA (reduce.cu:retire_ticket)
    if (t == 0) s_last = (retire_ticket(&counters[r], pending) + pending == static_cast<unsigned>(P));
    pending = 0;
    group_sync<1, kTmaConsumers>();
    if (s_last) {
      acquire_fence();
      Pair<A> root = tree_over<M, A, kThreads, 1>(partials + r * P, P, red);
      if (t == 0) counters[r] = 0u;
      finish_root<M, A, 1, kTmaConsumers>(root, out + r, peer, epoch, red);
    }
    group_sync<1, kTmaConsumers>();
  }
}

}  // namespace tfb
