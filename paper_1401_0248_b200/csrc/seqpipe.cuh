// seqpipe.cuh — the reference's sequential flavors (seq: kernels.py:127-243;
// unroll:k / vec:k lanes: kernels.py:257-541) with their memory latency taken
// off the dependency chain.  Included by reduce.cu after tma.cuh (mbarrier and
// bulk-copy helpers).
//
// The recurrences are inherently serial (one rounding after another, in the
// reference's element order), so one thread (seq) or k threads (lanes) do all
// the arithmetic — but they no longer wait on global memory: a producer thread
// streams the input in 8 KiB chunks with cp.async.bulk (TMA engine) into a
// ring of shared-memory stages guarded by mbarriers, and the consumers read
// each element from shared memory, so the time per element is the recurrence's
// FP-add latency instead of a DRAM round trip per 8 elements.
//
// Elements are consumed in exactly the reference's order: the unaligned head
// (before the first 16-byte boundary) and the tail after the last whole chunk
// come straight from global memory, the chunks in between from the ring.
// x and y must share their offset modulo 16 bytes (the launcher falls back to
// the plain kernels otherwise).

namespace tfb {

constexpr int kSeqStages = 8;
constexpr int kSeqChunkBytes = 8192;  // per operand per stage
constexpr int kSeqThreads = 64;       // warp 0: consumers (lanes 0..k-1); warp 1 lane 0: producer

template <typename T, bool DOT>
struct SeqSmem {
  static constexpr size_t kBytes = size_t(kSeqStages) * kSeqChunkBytes * (DOT ? 2 : 1) + 2 * kSeqStages * 8 + 16;
};

// k == 1: seq flavor (the state is the result).  k in {2,4,8,16}: lane j runs
// elements i*k + j of the blocked prefix nb = n - n % k, the lanes merge left to
// right, lane 0 continues over the tail [nb, n) (lanes_kernel, reduce.cu).
template <int M, typename T, bool DOT>
__global__ void __launch_bounds__(kSeqThreads) seq_pipe_kernel(const T* __restrict__ x, const T* __restrict__ y,
                                                               int64_t n, int k, int64_t head, int64_t nchunks,
                                                               Pair<typename Acc<M, T>::type>* __restrict__ out) {
  using A = typename Acc<M, T>::type;
  constexpr int CE = kSeqChunkBytes / static_cast<int>(sizeof(T));  // elements per chunk (multiple of 16)
  extern __shared__ __align__(128) unsigned char seq_smem[];
  T* sx = reinterpret_cast<T*>(seq_smem);
  T* sy = reinterpret_cast<T*>(seq_smem + size_t(kSeqStages) * kSeqChunkBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(seq_smem + size_t(kSeqStages) * kSeqChunkBytes * (DOT ? 2 : 1));
  uint64_t* empty = full + kSeqStages;
  __shared__ Pair<A> lane_state[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSeqStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t body = head + nchunks * CE;  // [head, body) streams through the ring

  if (threadIdx.x == 32) {  // ---------------- producer ----------------
    int slot = 0;
    uint32_t phase = 0;
    for (int64_t c = 0; c < nchunks; ++c) {
      TFB_CHECK(head + (c + 1) * CE <= n);
      mbar_wait(&empty[slot], phase ^ 1u);
      mbar_arrive_expect_tx(&full[slot], kSeqChunkBytes * (DOT ? 2u : 1u));
      bulk_g2s(sx + slot * CE, x + head + c * CE, kSeqChunkBytes, &full[slot]);
      if constexpr (DOT) bulk_g2s(sy + slot * CE, y + head + c * CE, kSeqChunkBytes, &full[slot]);
      if (++slot == kSeqStages) { slot = 0; phase ^= 1u; }
    }
    return;
  }
  if (threadIdx.x >= 32) return;

  // ---------------- consumers: lanes 0..k-1 of warp 0 ----------------
  const int j = threadIdx.x;
  const bool active = j < k;
  const unsigned mask = k >= 32 ? 0xffffffffu : ((1u << k) - 1u);
  const int64_t nb = k == 1 ? n : n - n % k;  // elements the lanes run (the rest: lane 0 after the merge)
  Pair<A> st = zero_pair<A>();
  if (active) {
    // head (global): elements j, j + k, ... below `head`
    for (int64_t e = j; e < head && e < nb; e += k) accumulate<M, T, DOT>(st, x[e], DOT ? y[e] : T(0));
    int slot = 0;
    uint32_t phase = 0;
    // lane j's first element in every chunk: offset = (j - head) mod k (CE is a multiple of k)
    const int off0 = static_cast<int>(((j - head % k) % k + k) % k);
    for (int64_t c = 0; c < nchunks; ++c) {
      const int64_t base = head + c * CE;
      mbar_wait(&full[slot], phase);
      const T* cx = sx + slot * CE;
      const T* cy = sy + slot * CE;
      if (base + CE <= nb) {
        if (k == 1) {  // seq: 8 elements per step, the next step's loads in flight
          T a[8], b[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            a[q] = cx[q];
            if constexpr (DOT) b[q] = cy[q];
          }
          for (int off = 0; off < CE; off += 8) {
            T a2[8], b2[8];
            const int nxt = off + 8 < CE ? off + 8 : off;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              a2[q] = cx[nxt + q];
              if constexpr (DOT) b2[q] = cy[nxt + q];
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) accumulate<M, T, DOT>(st, a[q], DOT ? b[q] : T(0));
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              a[q] = a2[q];
              if constexpr (DOT) b[q] = b2[q];
            }
          }
        } else {
#pragma unroll 4
          for (int off = off0; off < CE; off += k) accumulate<M, T, DOT>(st, cx[off], DOT ? cy[off] : T(0));
        }
      } else {
        for (int off = off0; off < CE && base + off < nb; off += k)
          accumulate<M, T, DOT>(st, cx[off], DOT ? cy[off] : T(0));
      }
      __syncwarp(mask);
      if (j == 0) mbar_arrive(&empty[slot]);
      if (++slot == kSeqStages) { slot = 0; phase ^= 1u; }
    }
    // tail of the streamed region (global): lane j's elements in [body, nb)
    int64_t e = body + ((j - body % k) % k + k) % k;
    for (; e < nb; e += k) accumulate<M, T, DOT>(st, x[e], DOT ? y[e] : T(0));
  }
  if (k == 1) {
    if (j == 0) out[0] = st;
    return;
  }
  if (active) lane_state[j] = st;
  __syncwarp();
  if (j != 0) return;
  Pair<A> s;
  if constexpr (M == kDirect || M == kWide) {
    s = zero_pair<A>();  // s = 0; s = s + acc[j] for all j   (kernels.py:267-269)
    for (int q = 0; q < k; ++q) s.s = Ar<A>::add(s.s, lane_state[q].s);
  } else {
    s = lane_state[0];
    for (int q = 1; q < k; ++q) s = merge<M, A>(s, lane_state[q]);
  }
  for (int64_t i = nb; i < n; ++i) accumulate<M, T, DOT>(s, x[i], DOT ? y[i] : T(0));
  out[0] = s;
}

}  // namespace tfb
