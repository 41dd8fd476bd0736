// small.cuh — single-cluster reduction for small 1-D inputs (<= 64 one-vector
// leaves, i.e. <= 256 KiB per operand at the auto leaf size).  Included by
// reduce.cu after the shared device helpers.
//
// Same leaves, chains and trees as leaves_kernel + the row tree, so results
// are bit-identical; only the launch shape differs.  One thread-block cluster
// of C = max(1, P2/4) CTAs (P2 = pow2ceil(P) leaves):
//   * CTA c owns leaves [4c, 4c+4); every thread issues the loads of all its
//     chains (one 16-byte vector per operand per leaf) before any arithmetic,
//     so the whole input is a single memory round trip;
//   * the four 256-chain leaf trees run interleaved (warp shuffles, one
//     shared-memory exchange), then the CTA's aligned 4-leaf subtree;
//   * each CTA stores its subtree pair into CTA 0's shared memory (DSMEM),
//     one cluster barrier, CTA 0 finishes the tree over the C pairs.
// No global scratch, no atomics, no second kernel: the multi-launch tail
// (retire ticket or PDL tree) is replaced by one cluster barrier.

#include <cooperative_groups.h>

namespace tfb {

constexpr int kSmallLeaves = 4;       // leaves per CTA
constexpr int kSmallMaxCluster = 16;  // non-portable cluster size (opt-in)
constexpr int64_t kSmallMaxLeaves = int64_t(kSmallLeaves) * kSmallMaxCluster;

template <typename A>
__device__ __forceinline__ Pair<A> shfl_down_pair(const Pair<A>& p, int off) {
  Pair<A> o;
  o.s = __shfl_down_sync(0xffffffffu, p.s, off);
  o.e = __shfl_down_sync(0xffffffffu, p.e, off);
  return o;
}

template <int M, typename T, bool DOT, bool VEC>
__global__ void __launch_bounds__(kThreads) small_cluster_kernel(const T* __restrict__ x,
                                                                 const T* __restrict__ y, int64_t n,
                                                                 int64_t P, int64_t P2,
                                                                 Pair<typename Acc<M, T>::type>* __restrict__ out,
                                                                 int prefetch) {
  namespace cg = cooperative_groups;
  using A = typename Acc<M, T>::type;
  using VT = typename Vec<T>::type;
  constexpr int V = Vec<T>::V;
  constexpr int64_t Lel = int64_t(kThreads) * V;  // one vector per chain (R = 1)
  constexpr int G = kSmallLeaves;
  __shared__ Pair<A> red[G * kWarps];
  __shared__ Pair<A> slots[kSmallMaxCluster];

  cg::cluster_group cluster = cg::this_cluster();
  const int c = static_cast<int>(cluster.block_rank());
  const int C = static_cast<int>(cluster.num_blocks());
  TFB_CHECK(C <= kSmallMaxCluster && int64_t(C) * G >= P && gridDim.x == static_cast<unsigned>(C));
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int gsz = static_cast<int>(P2 < G ? P2 : G);  // leaves of this CTA's subtree
  // Preamble (leaves_kernel has the same): ask the L2 for this CTA's contiguous G leaves
  // before the grid dependency resolves — a hint, no data enters the SM.
  if constexpr (VEC) {
    if (prefetch && t < (DOT ? 2 : 1)) {
      const int64_t start = int64_t(c) * G * Lel;
      int64_t bytes = (n - start < G * Lel ? n - start : G * Lel) * static_cast<int64_t>(sizeof(T));
      bytes &= ~int64_t(15);
      TFB_CHECK(bytes <= 0 || (reinterpret_cast<uintptr_t>((t ? y : x) + start) & 15u) == 0);
      if (bytes > 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"((t ? y : x) + start),
                     "r"(static_cast<unsigned>(bytes))
                     : "memory");
    }
  }
  // programmatic dependent of the previous kernel (no memory access before it retired),
  // and itself lets the next kernel of the stream become resident early
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // ---- loads of every chain first (one round trip), then the recurrences ----
  VT a[G], b[G];
  bool full[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int64_t start = (int64_t(c) * G + g) * Lel;
    full[g] = VEC && g < gsz && start + Lel <= n;
    if (full[g]) {
      TFB_CHECK((reinterpret_cast<uintptr_t>(x + start) & 15u) == 0 && start + Lel <= n);
      a[g] = ld_stream(reinterpret_cast<const VT*>(x + start) + t);
      if constexpr (DOT) b[g] = ld_stream(reinterpret_cast<const VT*>(y + start) + t);
    }
  }
  Pair<A> st[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    st[g] = zero_pair<A>();
    const int64_t start = (int64_t(c) * G + g) * Lel;
    if (full[g]) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        if constexpr (DOT) accumulate<M, T, true>(st[g], vget(a[g], j), vget(b[g], j));
        else accumulate<M, T, false>(st[g], vget(a[g], j), T(0));
      }
    } else if (g < gsz) {  // partial / misaligned leaf: leaf_chain's scalar path
      const int64_t base = start + int64_t(t) * V;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int64_t i = base + j;
        if (i < n) accumulate<M, T, DOT>(st[g], x[i], DOT ? y[i] : T(0));
      }
    }
  }

  // ---- the G leaf trees (block_tree's exact merge order), interleaved ----
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      Pair<A> o = shfl_down_pair(st[g], off);
      if (!HasErr<M>::value) o.e = A(0);
      if ((lane & (2 * off - 1)) == 0) st[g] = merge<M, A>(st[g], o);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) red[g * kWarps + warp] = st[g];
  }
  __syncthreads();
  if (warp == 0) {
    // lane = g*8 + w: warp w's pair of leaf g; levels 1, 2, 4 finish each leaf tree
    Pair<A> v = red[lane];
#pragma unroll
    for (int off = 1; off < kWarps; off <<= 1) {
      Pair<A> o = shfl_down_pair(v, off);
      if (!HasErr<M>::value) o.e = A(0);
      if ((lane & (2 * off - 1)) == 0) v = merge<M, A>(v, o);
    }
    // leaves past P are the tree's (+0, +0) padding
    const int64_t leaf = int64_t(c) * G + (lane >> 3);
    if ((lane & 7) == 0 && leaf >= P) v = zero_pair<A>();
    // aligned subtree over this CTA's gsz leaves (lanes 0, 8, 16, 24)
    for (int off = kWarps; off < kWarps * gsz; off <<= 1) {
      Pair<A> o = shfl_down_pair(v, off);
      if (!HasErr<M>::value) o.e = A(0);
      if ((lane & (2 * off - 1)) == 0) v = merge<M, A>(v, o);
    }
    if (lane == 0) {
      if (C == 1) {
        *out = v;
      } else {
        Pair<A>* dst = cluster.map_shared_rank(slots, 0);
        dst[c] = v;
      }
    }
  }
  if (C == 1) return;
  cluster.sync();  // release/acquire at cluster scope: CTA 0 sees every slot
  if (c == 0 && warp == 0) {
    Pair<A> v = lane < C ? slots[lane] : zero_pair<A>();
    for (int off = 1; off < C; off <<= 1) {
      Pair<A> o = shfl_down_pair(v, off);
      if (!HasErr<M>::value) o.e = A(0);
      if ((lane & (2 * off - 1)) == 0) v = merge<M, A>(v, o);
    }
    if (lane == 0) *out = v;
  }
}

}  // namespace tfb
