// reduce.cu — sm_100a twofold reduction kernels and their C-ABI launchers.
//
// Reduction tree (the GPU's non-sequential flavor; DESIGN.md §3 states it and
// oracle/twofold_oracle.c:tfo_emulate restates it bit-for-bit):
//   leaf      L = 2^leaf_log2 contiguous elements, L = 256 * V * R
//             (V = 16 B / sizeof(T) elements per vector, R vectors per thread)
//   thread t  runs the reference's sequential recurrence over the leaf's
//             elements start + (k*256 + t)*V + j, k = 0..R-1, j = 0..V-1
//             (coalesced 16-byte loads; elements past n are skipped)
//   leaf pair balanced contiguous binary tree over the 256 thread states
//             (warp shuffles, then one shared-memory level)
//   row pair  balanced contiguous binary tree over the row's leaf pairs,
//             padded with (+0,+0) to a power of two (merge order by leaf
//             index, never by arrival order), built by one of three tails:
//             the CTA that retires the row's last leaf (atomic ticket; the
//             TMA loader), a programmatic-dependent tree kernel (the LDG
//             loader's default), or — inputs of <= 64 one-vector leaves — one
//             thread-block cluster merging through DSMEM (small.cuh)
// The partition depends only on (dtype, n, leaf_log2), so results are
// bit-identical across reruns, grid sizes, tails, loaders and SM counts.
// Loaders: 128-bit LDG streaming (here) or the warp-specialised bulk-copy
// pipeline (tma.cuh), chosen per size from the measured loader_table.inc.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "eft.cuh"
#include "twofold_b200.h"
#include "status.h"

namespace tfb {

constexpr int kThreads = 256;  // chains per leaf (the tree geometry) and default CTA size
constexpr int kWarps = kThreads / 32;

// Tuning builds only (-DTFB_TRACE, scripts/trace_cfg2.py): per-CTA %globaltimer stamps
// of the leaves / tree kernels into a caller-provided buffer (tf_trace_buffer), 8 slots
// per CTA; the tree kernel takes the record after the last CTA slot.
#ifdef TFB_TRACE
__device__ unsigned long long* tfb_trace_ptr = nullptr;
__device__ __forceinline__ unsigned long long trace_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_mark(unsigned rec, int slot) {
  if (threadIdx.x == 0 && tfb_trace_ptr) tfb_trace_ptr[rec * 8ull + slot] = trace_now();
}
#define TFB_TR(rec, slot) trace_mark(rec, slot)
#else
#define TFB_TR(rec, slot)
#endif

template <typename T> struct Vec;
template <> struct Vec<float> { using type = float4; static constexpr int V = 4; };
template <> struct Vec<double> { using type = double2; static constexpr int V = 2; };

// Streaming 128-bit loads: read-only path, no L1 allocation (each byte is
// read exactly once).
#ifndef TFB_LD_HINT
#define TFB_LD_HINT ".L1::no_allocate.L2::256B"  // tuning builds may override (scripts/build_ld_variants.sh)
#endif
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm("ld.global.nc" TFB_LD_HINT ".v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 r;
  asm("ld.global.nc" TFB_LD_HINT ".v2.f64 {%0,%1}, [%2];"
      : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ float vget(const float4& v, int j) {
  return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
}
__device__ __forceinline__ double vget(const double2& v, int j) { return j == 0 ? v.x : v.y; }

template <typename A>
__device__ __forceinline__ Pair<A> ld_pair_cg(const Pair<A>* p) {
  Pair<A> r;
  r.s = __ldcg(&p->s);
  r.e = __ldcg(&p->e);
  return r;
}

// Retire ticket: publish this CTA's unit pair (written by the same thread just
// before) and count it.  TFB_RETIRE_ACQREL=1: one acq_rel RMW at gpu scope;
// 0: the classic __threadfence + atomicAdd.  The last CTA then runs
// acquire_fence() before any thread reads the other CTAs' pairs.
#ifndef TFB_RETIRE_ACQREL
#define TFB_RETIRE_ACQREL 0  // both forms compile to MEMBAR.ALL.GPU + ATOM + CCTL.IVALL on sm_100a
#endif
// `count` unit pairs of one row are retired at once (the TMA loader: a CTA
// stores the pairs of all its leaves of the row with plain stores and takes ONE
// ticket when it leaves the row, no fence round trip per leaf); the CTA whose
// ticket completes the row's count builds the row tree.
__device__ __forceinline__ unsigned retire_ticket(unsigned* counter, unsigned count = 1u) {
#if TFB_RETIRE_ACQREL
  unsigned prev;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(prev) : "l"(counter), "r"(count) : "memory");
  return prev;
#else
  __threadfence();
  return atomicAdd(counter, count);
#endif
}
__device__ __forceinline__ void acquire_fence() {
#if TFB_RETIRE_ACQREL
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
#else
  __threadfence();
#endif
}

template <int M> struct HasErr {
  static constexpr bool value = (M == kFast || M == kRigorous || M == kKahan || M == kFastTP || M == kRigorousTP);
};

// Balanced contiguous binary tree over the first `width` (power of two,
// 1..256) threads' states; result valid in thread 0.  Level `off` merges
// thread t (t % 2off == 0) with thread t + off as the right operand.
// CTA-level barrier for the first NT threads: __syncthreads when the whole CTA
// takes part (BAR == 0), else named barrier BAR (warp-specialised kernels whose
// producer warp must not join).
template <int BAR, int NT>
__device__ __forceinline__ void group_sync() {
  if constexpr (BAR == 0) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NT) : "memory");
}

template <int M, typename A, int BAR = 0, int NT = kThreads>
__device__ __forceinline__ Pair<A> block_tree(Pair<A> st, Pair<A>* smem, int width) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wl = width < 32 ? width : 32;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    if (off >= wl) break;
    Pair<A> o;
    o.s = __shfl_down_sync(0xffffffffu, st.s, off);
    if constexpr (HasErr<M>::value) o.e = __shfl_down_sync(0xffffffffu, st.e, off);
    else o.e = A(0);
    if ((lane & (2 * off - 1)) == 0) st = merge<M, A>(st, o);
  }
  if (width > 32) {
    if (lane == 0) smem[warp] = st;
    group_sync<BAR, NT>();
    if (warp == 0) {
      const int nw = width >> 5;
      st = lane < nw ? smem[lane] : zero_pair<A>();
#pragma unroll
      for (int off = 1; off < kWarps; off <<= 1) {
        if (off >= nw) break;
        Pair<A> o;
        o.s = __shfl_down_sync(0xffffffffu, st.s, off);
        if constexpr (HasErr<M>::value) o.e = __shfl_down_sync(0xffffffffu, st.e, off);
        else o.e = A(0);
        if ((lane & (2 * off - 1)) == 0) st = merge<M, A>(st, o);
      }
    }
    group_sync<BAR, NT>();
  }
  return st;
}

// Balanced tree over P pairs (padded with (+0,+0) to P2 = pow2ceil(P)) by one
// CTA.  If P2 >= 256, thread t first folds leaves [t*g, (t+1)*g), g = P2/256,
// with a binary-counter stack (the same balanced shape, sequentially), then
// the 256-thread tree finishes; otherwise threads < P2 hold one pair each.
template <int M, typename A, int NT = kThreads, int BAR = 0>
__device__ Pair<A> tree_over(const Pair<A>* parts, int64_t P, Pair<A>* smem) {
  int64_t P2 = 1;
  while (P2 < P) P2 <<= 1;
  const int t = threadIdx.x;
  if (P2 >= NT) {
    const int64_t g = P2 / NT;
    const int64_t base = static_cast<int64_t>(t) * g;
    Pair<A> stack[32];
    for (int64_t i0 = 0; i0 < g; i0 += 8) {
      Pair<A> buf[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t idx = base + i0 + q;
        buf[q] = (i0 + q < g && idx < P) ? ld_pair_cg(parts + idx) : zero_pair<A>();
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t i = i0 + q;
        if (i < g) {
          Pair<A> cur = buf[q];
          int b = 0;
          for (; (i >> b) & 1; ++b) cur = merge<M, A>(stack[b], cur);
          stack[b] = cur;
        }
      }
    }
    int lg = 0;
    while ((int64_t(1) << lg) < g) ++lg;
    return block_tree<M, A, BAR, NT>(stack[lg], smem, NT);
  }
  Pair<A> cur = t < P ? ld_pair_cg(parts + t) : zero_pair<A>();
  return block_tree<M, A, BAR, NT>(cur, smem, static_cast<int>(P2));
}

}  // namespace tfb
#include "peer.cuh"
namespace tfb {

template <typename T, bool DOT, int U>
__device__ __forceinline__ void load_batch(const typename Vec<T>::type* xv, const typename Vec<T>::type* yv,
                                           int k, typename Vec<T>::type (&a)[U],
                                           typename Vec<T>::type (&b)[U]) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    a[u] = ld_stream(xv + static_cast<int64_t>(k + u) * kThreads);
    if constexpr (DOT) b[u] = ld_stream(yv + static_cast<int64_t>(k + u) * kThreads);
  }
}

template <int M, typename T, bool DOT, int U>
__device__ __forceinline__ void consume_batch(Pair<typename Acc<M, T>::type>& st,
                                              const typename Vec<T>::type (&a)[U],
                                              const typename Vec<T>::type (&b)[U]) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
#pragma unroll
    for (int j = 0; j < Vec<T>::V; ++j) {
      if constexpr (DOT) accumulate<M, T, true>(st, vget(a[u], j), vget(b[u], j));
      else accumulate<M, T, false>(st, vget(a[u], j), T(0));
    }
  }
}

// Misaligned binary32 operands (both MS elements past a 16-byte boundary): chain t's
// vector starts MS elements into aligned vector t and ends in aligned vector
// t + 1 — loaded by the next lane (warp shuffle) or, for lane 31, by itself.
// Every aligned vector read lies in a 16-byte block holding an element of the
// leaf, i.e. inside the caller's allocation.
template <typename T> __device__ __forceinline__ T shfl_down1(T v) { return __shfl_down_sync(0xffffffffu, v, 1); }
// Element j of chain t's vector: components MS.. of its own aligned vector, then
// components 0..MS-1 of the next one (nx).
template <int MS, typename T>
__device__ __forceinline__ T shifted_get(const typename Vec<T>::type& own, const T (&nx)[MS], int j) {
  constexpr int V = Vec<T>::V;
  return MS + j < V ? vget(own, MS + j) : nx[MS + j - V];
}
// nx = components 0..MS-1 of the next aligned vector: lane + 1's, or (lane 31)
// the elements it loaded itself together with its own batch (`edge_vals`).
template <int MS, typename T>
__device__ __forceinline__ void next_comps(const typename Vec<T>::type& own, const T (&edge_vals)[MS], bool edge,
                                           T (&nx)[MS]) {
#pragma unroll
  for (int q = 0; q < MS; ++q) {
    const T v = shfl_down1(vget(own, q));
    nx[q] = edge ? edge_vals[q] : v;
  }
}

// One thread's sequential recurrence over its elements of the leaf at
// `start` of a row of n elements.  VEC: 16-byte aligned row, full leaf.
// MS > 0 (with VEC false): both operands MS elements past a 16-byte boundary,
// full leaf: aligned vector loads + one lane shuffle (same elements, same order).
template <int M, typename T, bool DOT, bool VEC, int U, int MS = 0>
__device__ __forceinline__ Pair<typename Acc<M, T>::type> leaf_chain(
    const T* __restrict__ x, const T* __restrict__ y, int64_t start, int64_t n, int R, int t) {
  using A = typename Acc<M, T>::type;
  using VT = typename Vec<T>::type;
  constexpr int V = Vec<T>::V;
  Pair<A> st = zero_pair<A>();
  const int64_t L = static_cast<int64_t>(R) * kThreads * V;
  TFB_CHECK(t >= 0 && t < kThreads && start >= 0);
  if constexpr (!VEC && MS > 0) {
    if (start + L <= n) {
    TFB_CHECK((reinterpret_cast<uintptr_t>(x + start - MS) & 15u) == 0);
    const VT* xa = reinterpret_cast<const VT*>(x + start - MS) + t;
    const VT* ya = DOT ? reinterpret_cast<const VT*>(y + start - MS) + t : nullptr;
    const bool edge = (threadIdx.x & 31) == 31;
    constexpr int US = (sizeof(T) == 4 && DOT && MS >= 2 && U > 2) ? U / 2 : U;  // f32 dots: registers
    int k = 0;
    for (; k < R; k += US) {
      const int nu = R - k < US ? R - k : US;
      VT a[US], b[US];
      T ea[US][MS], eb[US][MS];
#pragma unroll
      for (int u = 0; u < US; ++u) {
        if (u < nu) {
          a[u] = ld_stream(xa + static_cast<int64_t>(k + u) * kThreads);
          if constexpr (DOT) b[u] = ld_stream(ya + static_cast<int64_t>(k + u) * kThreads);
          if (edge) {  // lane 31: its last MS elements lie in the next warp's first vector
            const int64_t e = start + (static_cast<int64_t>(k + u) * kThreads + t) * V + (V - MS);
#pragma unroll
            for (int q = 0; q < MS; ++q) {
              ea[u][q] = __ldg(x + e + q);  // measured faster than a no-allocate load here
              if constexpr (DOT) eb[u][q] = __ldg(y + e + q);
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < US; ++u) {
        if (u < nu) {
          T an[MS], bn[MS];
          next_comps<MS, T>(a[u], ea[u], edge, an);
          if constexpr (DOT) next_comps<MS, T>(b[u], eb[u], edge, bn);
#pragma unroll
          for (int j = 0; j < V; ++j) {
            if constexpr (DOT)
              accumulate<M, T, true>(st, shifted_get<MS, T>(a[u], an, j), shifted_get<MS, T>(b[u], bn, j));
            else accumulate<M, T, false>(st, shifted_get<MS, T>(a[u], an, j), T(0));
          }
        }
      }
    }
    return st;
    }
  }
  if (VEC && start + L <= n) {
    TFB_CHECK((reinterpret_cast<uintptr_t>(x + start) & 15u) == 0);
    const VT* xv = reinterpret_cast<const VT*>(x + start) + t;
    const VT* yv = DOT ? reinterpret_cast<const VT*>(y + start) + t : nullptr;
    // Software pipeline: batch k+U is in flight while batch k is consumed, so
    // each thread keeps 2U vectors per operand outstanding.  Elements are
    // consumed in exactly the same order as without the pipeline.
    int k = 0;
#if TFB_PIPELINE
    if (R >= U) {
      VT a0[U], b0[U], a1[U], b1[U];
      load_batch<T, DOT, U>(xv, yv, 0, a0, b0);
      for (; k + 2 * U <= R; k += 2 * U) {
        load_batch<T, DOT, U>(xv, yv, k + U, a1, b1);
        consume_batch<M, T, DOT, U>(st, a0, b0);
        if (k + 2 * U < R) load_batch<T, DOT, U>(xv, yv, k + 2 * U, a0, b0);
        consume_batch<M, T, DOT, U>(st, a1, b1);
      }
      if (k + U <= R) {  // R == U (odd number of batches only happens for R == U)
        consume_batch<M, T, DOT, U>(st, a0, b0);
        k += U;
      }
    }
#else
    for (; k + U <= R; k += U) {
      VT a[U], b[U];
      load_batch<T, DOT, U>(xv, yv, k, a, b);
      consume_batch<M, T, DOT, U>(st, a, b);
    }
#endif
    for (; k < R; ++k) {
      VT a = ld_stream(xv + static_cast<int64_t>(k) * kThreads);
      VT b;
      if constexpr (DOT) b = ld_stream(yv + static_cast<int64_t>(k) * kThreads);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        if constexpr (DOT) accumulate<M, T, true>(st, vget(a, j), vget(b, j));
        else accumulate<M, T, false>(st, vget(a, j), T(0));
      }
    }
  } else if (!VEC && start + L <= n) {
    // full leaf, operands not 16-byte aligned: element loads, but U vectors' worth
    // per operand in flight before the recurrence consumes them (same order)
    constexpr int UE = U > 2 ? U / 2 : U;
    int k = 0;
    for (; k + UE <= R; k += UE) {
      T a[UE][V], b[UE][V];
#pragma unroll
      for (int u = 0; u < UE; ++u)
#pragma unroll
        for (int j = 0; j < V; ++j) {
          const int64_t i = start + (static_cast<int64_t>(k + u) * kThreads + t) * V + j;
          a[u][j] = __ldg(x + i);
          if constexpr (DOT) b[u][j] = __ldg(y + i);
        }
#pragma unroll
      for (int u = 0; u < UE; ++u)
#pragma unroll
        for (int j = 0; j < V; ++j) accumulate<M, T, DOT>(st, a[u][j], DOT ? b[u][j] : T(0));
    }
    for (; k < R; ++k) {
      const int64_t base = start + (static_cast<int64_t>(k) * kThreads + t) * V;
#pragma unroll
      for (int j = 0; j < V; ++j) accumulate<M, T, DOT>(st, x[base + j], DOT ? y[base + j] : T(0));
    }
  } else {
    // a row's partial last leaf: the k-rows that lie entirely inside the row one
    // 16-byte vector at a time (aligned rows), then bounds-checked elements
    int k = 0;
    if constexpr (VEC) {
      const int kfull = static_cast<int>((n - start) / (int64_t(kThreads) * V));
      const VT* xv = reinterpret_cast<const VT*>(x + start) + t;
      const VT* yv = DOT ? reinterpret_cast<const VT*>(y + start) + t : nullptr;
#pragma unroll 1
      for (; k < kfull; ++k) {
        VT a = ld_stream(xv + static_cast<int64_t>(k) * kThreads);
        VT b;
        if constexpr (DOT) b = ld_stream(yv + static_cast<int64_t>(k) * kThreads);
#pragma unroll
        for (int j = 0; j < V; ++j) {
          if constexpr (DOT) accumulate<M, T, true>(st, vget(a, j), vget(b, j));
          else accumulate<M, T, false>(st, vget(a, j), T(0));
        }
      }
    }
#pragma unroll 1
    for (; k < R; ++k) {
      const int64_t base = start + (static_cast<int64_t>(k) * kThreads + t) * V;
      if (base >= n) break;  // later k only go further right
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int64_t i = base + j;
        if (i < n) {
          accumulate<M, T, DOT>(st, x[i], DOT ? y[i] : T(0));
        }
      }
    }
  }
  return st;
}

#ifndef TFB_PIPELINE
#define TFB_PIPELINE 0  // measured: no gain, costs occupancy (profiles/r01_variants.md)
#endif
#ifndef TFB_UNROLL_F32
#define TFB_UNROLL_F32 4
#endif
#ifndef TFB_UNROLL_F64
#define TFB_UNROLL_F64 2
#endif
template <typename T> struct Unroll;
template <> struct Unroll<float> { static constexpr int value = TFB_UNROLL_F32; };
template <> struct Unroll<double> { static constexpr int value = TFB_UNROLL_F64; };

// Grid reduction over rows x cols.  A leaf's 256 chains may be split over
// S = 256/NT CTAs: unit u = (row r, leaf l, part s), u = (r*P + l)*S + s, and CTA
// part s runs chains [s*NT, (s+1)*NT).  Its block tree is exactly the leaf
// tree's subtree over those chains, and the row tree over the P*S unit pairs is
// the same balanced tree (zero pairs merge to zero pairs), so the result does
// not depend on S — S only balances the grid over the SMs.
// mode 0: write unit pairs to partials[u] only.  mode 1: fused — the CTA that
// retires a row's last unit builds the row tree into out[r].
// TFB_LDG_MINB (tuning builds only): min resident CTAs per SM the 256-thread
// LDG kernel is compiled for.  Unset = plain __launch_bounds__(NT): an explicit
// minimum of 1 makes ptxas spend up to 104 registers (3 CTAs/SM instead of 5).
#ifdef TFB_LDG_MINB
#define TFB_LDG_BOUNDS(NT, UF) __launch_bounds__(NT, (NT) == kThreads && (UF) == 1 ? TFB_LDG_MINB : 1)
#else
#define TFB_LDG_BOUNDS(NT, UF) __launch_bounds__(NT)
#endif
// Preamble of leaves_kernel, before the grid dependency resolves: ask the L2 for the head
// of this CTA's first leaf (bulk prefetch — a hint that moves no data into the SM, and the
// L2 is the point of coherence, so a predecessor still writing the operands is
// unaffected).  When the call is queued behind another kernel, HBM streams the head while
// that kernel's tail retires (launch_leaves_nt picks the size; 0 = off).  Not inlined: its
// address arithmetic must not add to the streaming loop's register budget.
template <typename T, bool DOT>
__device__ __noinline__ void prefetch_first_leaf(const T* x, const T* y, int64_t ldx, int64_t ldy, int64_t cols,
                                                 int leaf_log2, int64_t per_row, int64_t units, int pf_kb) {
  if (pf_kb <= 0 || static_cast<int64_t>(blockIdx.x) >= units) return;
  const int64_t r = blockIdx.x / per_row;
  const int64_t start = (blockIdx.x - r * per_row) << leaf_log2;
  int64_t bytes = cols - start < (int64_t(1) << leaf_log2) ? cols - start : (int64_t(1) << leaf_log2);
  bytes *= static_cast<int64_t>(sizeof(T));
  if (bytes > (static_cast<int64_t>(pf_kb) << 10)) bytes = static_cast<int64_t>(pf_kb) << 10;
  bytes &= ~int64_t(15);
  const int op = threadIdx.x & 1;
  const int64_t off = static_cast<int64_t>(threadIdx.x >> 1) * 4096;
  if (off < bytes && (DOT || op == 0)) {
    const char* p = reinterpret_cast<const char*>((op ? y + r * ldy : x + r * ldx) + start) + off;
    const unsigned sz = static_cast<unsigned>(bytes - off < 4096 ? bytes - off : 4096);
    // inside the row's leaf, 16-byte aligned and sized (the bulk prefetch's contract)
    TFB_CHECK((reinterpret_cast<uintptr_t>(p) & 15u) == 0 && sz > 0 && (sz & 15u) == 0 &&
              start + (off + sz) / static_cast<int64_t>(sizeof(T)) <= cols);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(sz) : "memory");
  }
}

// leaves_kernel flags: bit 0 fused tail (retire ticket); bits 8.. KiB per operand of the
// CTA's first leaf to prefetch into L2 before the dependency wait
constexpr int kLeavesFused = 1;
constexpr int kLeavesPrefetchShift = 8;
template <int M, typename T, bool DOT, bool VEC, int NT, int UF = 1, int MS = 0>
__global__ void TFB_LDG_BOUNDS(NT, UF) leaves_kernel(
    const T* __restrict__ x, const T* __restrict__ y, int64_t ldx, int64_t ldy,
    int64_t rows, int64_t cols, int leaf_log2, int64_t P,
    Pair<typename Acc<M, T>::type>* __restrict__ partials, unsigned* __restrict__ counters,
    Pair<typename Acc<M, T>::type>* __restrict__ out, int flags, int64_t part_cap) {
  using A = typename Acc<M, T>::type;
  constexpr int V = Vec<T>::V;
  constexpr int S = kThreads / NT;
  __shared__ Pair<A> smem[kWarps];
  __shared__ int s_last;
  const int R = (1 << leaf_log2) / (kThreads * V);
  const int64_t per_row = P * S;
  const int64_t units = rows * per_row;
  const int fused = flags & kLeavesFused;
  TFB_TR(blockIdx.x, 0);
#ifdef TFB_TRACE
  if (threadIdx.x == 0 && tfb_trace_ptr) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    tfb_trace_ptr[blockIdx.x * 8ull + 4] = sm;
  }
#endif
  if constexpr (VEC && S == 1)
    prefetch_first_leaf<T, DOT>(x, y, ldx, ldy, cols, leaf_log2, per_row, units, flags >> kLeavesPrefetchShift);
  // Launched as a programmatic dependent of the previous kernel in the stream
  // (launch_leaves_nt): resident early, but no memory access before that grid has
  // completed and flushed — so any predecessor, ours or the caller's, is safe.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  TFB_TR(blockIdx.x, 1);
  // partials-only mode may feed a programmatic-dependent tree kernel: let it be
  // scheduled now (it waits on griddepcontrol.wait for this grid's completion)
  if (!fused) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t r = u / per_row;
    const int64_t rem = u - r * per_row;
    const int64_t l = rem / S;
    const int part = static_cast<int>(rem - l * S);
    const T* xr = x + r * ldx;
    const T* yr = DOT ? y + r * ldy : nullptr;
    Pair<A> st = leaf_chain<M, T, DOT, VEC, Unroll<T>::value * UF, MS>(
        xr, yr, l << leaf_log2, cols, R, part * NT + static_cast<int>(threadIdx.x));
    TFB_TR(blockIdx.x, 2);
    st = block_tree<M, A>(st, smem, NT);
    if (!fused) {
      TFB_CHECK(u < part_cap);
      if (threadIdx.x == 0) partials[u] = st;
      TFB_TR(blockIdx.x, 3);
      continue;
    }
    if (per_row == 1) {
      if (threadIdx.x == 0) out[r] = st;
      continue;
    }
    if (threadIdx.x == 0) {
      TFB_CHECK(u < part_cap && counters != nullptr);
      partials[u] = st;
      s_last = (retire_ticket(&counters[r]) == static_cast<unsigned>(per_row - 1));
    }
    __syncthreads();
    if (s_last) {
      acquire_fence();
      Pair<A> root = tree_over<M, A, NT>(partials + r * per_row, per_row, smem);
      if (threadIdx.x == 0) {
        out[r] = root;
        counters[r] = 0u;  // leave the workspace reusable
      }
    }
    __syncthreads();
  }
}

template <int M, typename A>
__global__ void __launch_bounds__(kThreads) tree_kernel(const Pair<A>* __restrict__ pairs,
                                                        int64_t count, Pair<A>* __restrict__ out) {
  __shared__ Pair<A> smem[kWarps];
  Pair<A> root = count > 0 ? tree_over<M, A>(pairs, count, smem) : zero_pair<A>();
  if (threadIdx.x == 0) out[0] = root;
}

// Row trees over unit pairs written by a partials-only leaves launch; launched
// as a programmatic dependent (PDL) of it: resident early, waits for the
// primary grid's completion (and memory flush) in griddepcontrol.wait.
template <int M, typename A>
__global__ void __launch_bounds__(kThreads) rows_tree_kernel(const Pair<A>* __restrict__ partials, int64_t rows,
                                                             int64_t per_row, Pair<A>* __restrict__ out,
                                                             int64_t part_cap, const PeerCtx* __restrict__ peer,
                                                             uint32_t epoch) {
  __shared__ Pair<A> smem[kWarps];
  TFB_TR(4096, 0);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  TFB_TR(4096, 1);
  // the next kernel of the stream (e.g. the next call's leaves) may become resident now;
  // it waits for this grid's completion before touching memory
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  TFB_CHECK(rows * per_row <= part_cap);
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    Pair<A> root = tree_over<M, A>(partials + r * per_row, per_row, smem);
    finish_root<M, A>(root, out + r, peer, epoch, smem);
    __syncthreads();
  }
  TFB_TR(4096, 2);
}

// Sequential flavor: the reference recurrence, one thread, left to right.
template <int M, typename T, bool DOT>
__global__ void seq_kernel(const T* __restrict__ x, const T* __restrict__ y, int64_t n,
                           Pair<typename Acc<M, T>::type>* __restrict__ out) {
  using A = typename Acc<M, T>::type;
  Pair<A> st = zero_pair<A>();
  int64_t i = 0;
  for (; i + 8 <= n; i += 8) {
    T a[8], b[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      a[q] = x[i + q];
      if constexpr (DOT) b[q] = y[i + q];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      accumulate<M, T, DOT>(st, a[q], DOT ? b[q] : T(0));
    }
  }
  for (; i < n; ++i) {
    accumulate<M, T, DOT>(st, x[i], DOT ? y[i] : T(0));
  }
  out[0] = st;
}

// Lane flavor (kernels.py:257-541): lane j takes elements i*k + j of the
// blocked prefix, lanes merge left to right, the tail n % k continues on the
// merged state.
template <int M, typename T, bool DOT>
__global__ void lanes_kernel(const T* __restrict__ x, const T* __restrict__ y, int64_t n, int k,
                             Pair<typename Acc<M, T>::type>* __restrict__ out) {
  using A = typename Acc<M, T>::type;
  __shared__ Pair<A> lane_state[16];
  const int j = threadIdx.x;
  const int64_t nb = n - n % k;
  Pair<A> st = zero_pair<A>();
  for (int64_t i = 0; i < nb; i += k) {
    accumulate<M, T, DOT>(st, x[i + j], DOT ? y[i + j] : T(0));
  }
  lane_state[j] = st;
  __syncthreads();
  if (j != 0) return;
  Pair<A> s;
  if constexpr (M == kDirect || M == kWide) {
    s = zero_pair<A>();  // s = 0; s = s + acc[j] for all j   (kernels.py:267-269)
    for (int q = 0; q < k; ++q) s.s = Ar<A>::add(s.s, lane_state[q].s);
  } else {
    s = lane_state[0];
    for (int q = 1; q < k; ++q) s = merge<M, A>(s, lane_state[q]);
  }
  for (int64_t i = nb; i < n; ++i) {
    accumulate<M, T, DOT>(s, x[i], DOT ? y[i] : T(0));
  }
  out[0] = s;
}

// "noread" compute roof (the paper's p-functions; bench.py
// run_noread_baseline :281-307): the same per-thread recurrence as the grid
// kernel, fed from registers instead of memory, iters*8 addends per thread.
// The operands are runtime values and every op is an IEEE intrinsic, so the
// compiler cannot shorten the chain; the final states are stored to keep it live.
template <int M, typename T, bool DOT>
__global__ void __launch_bounds__(kThreads) noread_kernel(const T* __restrict__ seed8, int64_t iters,
                                                          Pair<typename Acc<M, T>::type>* __restrict__ out) {
  using A = typename Acc<M, T>::type;
  T a[8], b[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    a[j] = seed8[j] * static_cast<T>(1 + ((threadIdx.x + j) & 7));
    b[j] = seed8[(j + 3) & 7];
  }
  Pair<A> st = zero_pair<A>();
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) accumulate<M, T, DOT>(st, a[j], DOT ? b[j] : T(0));
  }
  out[blockIdx.x * int64_t(blockDim.x) + threadIdx.x] = st;
}

}  // namespace tfb
#include "tma.cuh"
#include "small.cuh"
#include "rows.cuh"
#include "seqpipe.cuh"
#include "seqsplit.cuh"
namespace tfb {

// ---------------------------------------------------------------------------
// Host side.

struct DevInfo { int sms = 0; };

static int device_sms() {
  static std::mutex mu;
  static std::unordered_map<int, int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cache[dev] = sms;
  return sms;
}

static int occupancy_of(const void* fn, int threads = kThreads) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(fn);
  if (it != cache.end()) return it->second;
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, threads, 0) != cudaSuccess ||
      blocks < 1)
    blocks = 1;
  cache[fn] = blocks;
  return blocks;
}

static inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int ceil_log2_i64(int64_t n) {
  int l = 0;
  while ((int64_t(1) << l) < n) ++l;
  return l;
}

int floor_leaf_log2(int dtype) {  // smallest leaf: one 16-byte vector per thread
  return dtype == TF_F32 ? 10 : 9;
}

// Auto leaf: about 2^-11 of the operand bytes (~2048 leaves), at least one
// vector per thread, at most 2^16 elements.  `total` = rows * cols.
// Measured optimum on B200 for every BASELINE config (profiles/r01_leaf_sweep.md).
int auto_leaf_log2(int dtype, int64_t total) {
  int l = ceil_log2_i64(total > 0 ? total : 1) + (dtype == TF_F32 ? 2 : 3) - 11;
  const int lo = floor_leaf_log2(dtype);
  if (l < lo) l = lo;
  if (l > 16) l = 16;
  return l;
}

// Leaf split S = 256/NT for the fused kernel (grid balance for small unit
// counts).  Result-neutral (see leaves_kernel); TFB_SPLIT=1|2|4 or
// tf_set_leaf_split() override it.
constexpr int kMaxSplit = 4;
static int g_split_override = -1;

// Description of the calling thread's last grid-reduction launch (tf_last_launch).
static thread_local char g_last_launch[192] = {0};
static const char* method_tag(int M) {
  static const char* tags[] = {"direct", "wide", "twofold-fast", "twofold-rigorous", "kahan",
                               "twofold-fast+TP", "twofold-rigorous+TP"};
  return M >= 0 && M < 7 ? tags[M] : "?";
}  // -1: read TFB_SPLIT once; 0: auto; 1|2|4: forced

static int choose_split(int64_t units, int fused) {
  if (!fused) return 1;  // leaves-only mode promises one pair per leaf
  if (g_split_override < 0) {
    const char* e = getenv("TFB_SPLIT");
    g_split_override = e ? atoi(e) : 0;
  }
  const int env = g_split_override;
  if (env == 1 || env == 2 || env == 4) return env;
  // measured (profiles/r01_summary.md): with correct scratch the split only
  // adds unit pairs to the final tree — no grid size benefits, so default off
  (void)units;
  return 1;
}

// Loader for aligned inputs: 0 = auto, 1 = 128-bit LDG streaming
// (leaves_kernel), 2 = bulk-copy/TMA pipeline (leaves_tma_kernel, 4 stages x
// 16 KiB per operand), 3 = TMA with 8 stages x 8 KiB, 4/5 = experimental dot
// stage shapes (3 x 32 KiB, 6 x 16 KiB).  Results are identical.  Auto
// (measured, profiles/r01_summary.md): TMA for >= 512 MiB dots (cfg5 +1.1 %,
// cfg4 +2.5 %) and >= 4 GiB twofold sums, LDG otherwise (Kahan sums and
// mid/small sizes favour LDG's higher CTA occupancy).  Env TFB_LOADER or
// tf_set_loader() override.
// Measured loader table (scripts/tune_loaders.py writes loader_table.inc):
// best loader per (f64, dot, method class, floor(log2(bytes)) in [20, 33]).
// Method classes: 0 direct/wide, 1 twofold-fast(+TP), 2 twofold-rigorous(+TP), 3 kahan.
#include "loader_table.inc"

static int auto_loader(int M, bool f64, bool dot, int64_t bytes) {
  const int mclass = (M == kFast || M == kFastTP) ? 1 : (M == kRigorous || M == kRigorousTP) ? 2 : M == kKahan ? 3 : 0;
  int b = 0;
  while ((int64_t(2) << b) <= bytes && b < 62) ++b;  // floor(log2(bytes))
  if (b < kLoaderTableMinLog2) return 1;
  if (b > kLoaderTableMaxLog2) b = kLoaderTableMaxLog2;
  return kLoaderTable[f64 ? 1 : 0][dot ? 1 : 0][mclass][b - kLoaderTableMinLog2];
}

static int g_loader = -1;
static int loader_choice() {
  if (g_loader < 0) {
    const char* e = getenv("TFB_LOADER");
    g_loader = e ? atoi(e) : 0;
  }
  return g_loader;
}

// Tail of the fused reduction: 0 = auto, 1 = last-CTA retire ticket (one
// launch), 2 = partials-only launch + programmatic-dependent tree kernel.
// Identical results; env TFB_TAIL or tf_set_tail() choose.
static int g_tail = -1;
static int tail_choice() {
  if (g_tail < 0) {
    const char* e = getenv("TFB_TAIL");
    g_tail = e ? atoi(e) : 0;
  }
  return g_tail;
}

// L2 prefetch preamble of the LDG leaves kernel (result-neutral): KiB per operand of each
// CTA's first leaf requested before the dependency wait.  -1 = automatic, 0 = off; env
// TFB_PF_KB or tf_set_prefetch() choose.  Automatic (scripts/prefetch_sweep.py,
// profiles/r02_prefetch_preamble.txt): a total budget shared by the grid's CTAs and
// operands — more than the L2 can hold ahead of the demand stream costs re-reads.
static int g_prefetch_kb = -2;
static int prefetch_choice() {
  if (g_prefetch_kb == -2) {
    const char* e = getenv("TFB_PF_KB");
    g_prefetch_kb = e ? atoi(e) : -1;
    if (g_prefetch_kb < -1) g_prefetch_kb = -1;
    if (g_prefetch_kb > 512) g_prefetch_kb = 512;
  }
  return g_prefetch_kb;
}
// Automatic size (measured, profiles/r02_prefetch_preamble.txt): inputs up to 8 MiB are
// requested whole (the requests land before the dependency resolves); above, the grid
// shares a budget of 0.3 x the input, at most 32 MiB — requests the L2 cannot complete
// ahead of the demand stream compete with it (cfg2: 32 KiB per operand per CTA 22.0 us,
// 64 KiB 25.1 us, off 24.1 us).
static int prefetch_kb_for(unsigned grid, int operands, int64_t input_bytes) {
  const int c = prefetch_choice();
  if (c >= 0) return c;
  int64_t budget = input_bytes;
  if (input_bytes > (int64_t(8) << 20)) {
    budget = input_bytes / 10 * 3;
    if (budget < (int64_t(8) << 20)) budget = int64_t(8) << 20;
    if (budget > (int64_t(32) << 20)) budget = int64_t(32) << 20;
  }
  int64_t kb = (budget / (int64_t(grid) * operands) + 1023) >> 10;
  kb = (kb + 3) & ~int64_t(3);  // whole 4 KiB pieces, at least one
  return static_cast<int>(kb > 512 ? 512 : kb);
}

template <int M, typename A>
static int launch_rows_tree_pdl(const void* partials, int64_t rows, int64_t per_row, void* out,
                                cudaStream_t stream, int64_t part_cap, const PeerCtx* peer, uint32_t epoch) {
  cudaLaunchConfig_t cfg = {};
  const int64_t sms = device_sms();
  cfg.gridDim = dim3(static_cast<unsigned>(rows < sms * 4 ? rows : sms * 4));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, rows_tree_kernel<M, A>, static_cast<const Pair<A>*>(partials), rows, per_row,
                         static_cast<Pair<A>*>(out), part_cap, peer, epoch) != cudaSuccess)
    return record_cuda_error();
  return check_launch();
}

template <int M, typename T, bool DOT, int NS, int SR, int MINB = 1>
static int launch_leaves_tma(const T* px, const T* py, int64_t ldx, int64_t ldy, int64_t rows, int64_t cols,
                             int leaf_log2, int64_t P, void* partials, void* counters, void* out,
                             cudaStream_t stream, const PeerCtx* peer, uint32_t epoch) {
  using A = typename Acc<M, T>::type;
  auto kern = &leaves_tma_kernel<M, T, DOT, NS, SR, MINB>;
  const size_t smem = TmaSmem<T, DOT, NS, SR>::kBytes;
  static std::mutex mu;
  static std::unordered_map<int, int> occ;  // per device
  int dev = 0;
  cudaGetDevice(&dev);
  int blocks = 0;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = occ.find(dev);
    if (it == occ.end()) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
          cudaSuccess)
        return record_cuda_error();
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, kTmaThreads, smem) != cudaSuccess ||
          blocks < 1)
        blocks = 1;
      occ[dev] = blocks;
    } else {
      blocks = it->second;
    }
  }
  const int64_t units = rows * P;
  const int64_t slots = static_cast<int64_t>(device_sms()) * blocks;
  const unsigned grid = static_cast<unsigned>(units < slots ? units : slots);
  snprintf(g_last_launch, sizeof(g_last_launch),
           "leaves_tma_kernel<%s,%s,%s,NS=%d,SR=%d> grid=%u block=%d smem=%zu units=%lld leaf_log2=%d",
           method_tag(M), sizeof(T) == 4 ? "f32" : "f64", DOT ? "dot" : "sum", NS, SR, grid, kTmaThreads, smem,
           static_cast<long long>(units), leaf_log2);
  // programmatic dependent of the previous kernel + L2 prefetch preamble, like the LDG
  // leaves kernel (launch_leaves_nt); the fused peer combine keeps the plain launch
  static const bool chain_env = !getenv("TFB_PDL_CHAIN") || atoi(getenv("TFB_PDL_CHAIN")) != 0;
  static const bool tma_chain = !getenv("TFB_TMA_CHAIN") || atoi(getenv("TFB_TMA_CHAIN")) != 0;
  // (one-CTA-per-SM rings only: with the 3 / 4 CTA small rings it measured mixed, profiles/r02_tma_chain.txt)
  const bool chain = chain_env && tma_chain && peer == nullptr && MINB == 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTmaThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = chain ? 1 : 0;
  const int chain_pf_kb =
      chain ? prefetch_kb_for(grid, DOT ? 2 : 1, rows * cols * int64_t(sizeof(T)) * (DOT ? 2 : 1)) : -1;
  if (cudaLaunchKernelEx(&cfg, kern, px, py, ldx, ldy, rows, cols, leaf_log2, P, static_cast<Pair<A>*>(partials),
                         static_cast<unsigned*>(counters), static_cast<Pair<A>*>(out), peer, epoch,
                         chain_pf_kb) != cudaSuccess)
    return record_cuda_error();
  return check_launch();
}

// One cluster of max(1, P2/4) CTAs (small.cuh).  Cluster sizes above 8 are
// opted into once per kernel and device.
template <int M, typename T, bool DOT, bool VEC>
static int launch_small(const T* px, const T* py, int64_t n, int64_t P, void* out, cudaStream_t stream) {
  using A = typename Acc<M, T>::type;
  auto kern = &small_cluster_kernel<M, T, DOT, VEC>;
  int64_t P2 = 1;
  while (P2 < P) P2 <<= 1;
  const int C = static_cast<int>(P2 < kSmallLeaves ? 1 : P2 / kSmallLeaves);
  if (C > 8) {
    static std::mutex mu;
    static std::unordered_map<int, bool> ok;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    if (!ok.count(dev)) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
        return record_cuda_error();
      ok[dev] = true;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(C));
  cfg.blockDim = dim3(kThreads);
  cfg.stream = stream;
  static const bool chain = !getenv("TFB_PDL_CHAIN") || atoi(getenv("TFB_PDL_CHAIN")) != 0;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(C);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see launch_leaves_nt
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = chain ? 2 : 1;
  snprintf(g_last_launch, sizeof(g_last_launch),
           "small_cluster_kernel<%s,%s,%s,%s> grid=%d cluster=%d block=%d leaves=%lld", method_tag(M),
           sizeof(T) == 4 ? "f32" : "f64", DOT ? "dot" : "sum", VEC ? "ldg128" : "scalar", C, C, kThreads,
           static_cast<long long>(P));
  if (cudaLaunchKernelEx(&cfg, kern, px, py, n, P, P2, static_cast<Pair<A>*>(out),
                         chain && prefetch_choice() != 0 ? 1 : 0) != cudaSuccess)
    return record_cuda_error();
  return check_launch();
}

// Rows family, one leaf per row: 0 = auto, 1 = always the CTA-per-leaf
// kernels, 2 = always the short-row kernel.  Identical results; env TFB_ROWS or
// tf_set_rows_kernel() choose.  Auto (measured, scripts/rows_shapes.py): lane
// groups for 16-byte aligned rows of <= 16 KiB per operand (5.6-6.3 TB/s from
// 16 to 4096 f32 columns, where a CTA per row reaches 0.07-5.8), misaligned
// binary32 rows of <= 16 KiB and misaligned binary64 rows of < 700 elements; a
// CTA per row above (LDG 6.3-6.5 TB/s
// from 16 to 128 KiB rows; the TMA pipeline from 256 KiB rows, cfg4).
constexpr int64_t kShortRowMaxBytes = int64_t(16) << 10;
// misaligned pitches: lane groups up to 1024 columns, a CTA per row (shifted-vector /
// batched element loads) above (profiles/r02_rows_misaligned.txt: f32 1001 columns 3.5 vs
// 3.4 TB/s, 4099: 3.3 vs 6.0; f64 1001: 4.6 vs 4.5, 4099: 4.7 vs 5.7)
constexpr int64_t kShortRowMaxMisCols = 1024;
constexpr int64_t kTmaRowMinBytes = int64_t(256) << 10;
static int g_rows_kernel = -1;
static int rows_kernel_choice() {
  if (g_rows_kernel < 0) {
    const char* e = getenv("TFB_ROWS");
    g_rows_kernel = e ? atoi(e) : 0;
  }
  return g_rows_kernel;
}

// The short-row kernels as programmatic dependents of the previous kernel in the stream
// (wait before any memory access, L2 prefetch of each warp's first rows before the wait);
// TFB_PDL_CHAIN=0 / TFB_ROWS_CHAIN=0 launch them plainly.  The kernels take the flag last.
template <typename Kern, typename... Args>
static int launch_rows_chained(Kern kern, unsigned grid, int block, cudaStream_t stream, int64_t input_bytes,
                               int operands, Args... args) {
  static const bool chain = (!getenv("TFB_PDL_CHAIN") || atoi(getenv("TFB_PDL_CHAIN")) != 0) &&
                            (!getenv("TFB_ROWS_CHAIN") || atoi(getenv("TFB_ROWS_CHAIN")) != 0);
  // bytes per warp and operand: the leaves kernels' budget (whole input up to 8 MiB, else
  // 0.3 x input, at most 32 MiB) shared by the grid's warps
  // measured (profiles/r02_rows_chain.txt): small calls gain 15-20 % (1000 x 64 f32 dot 2.74 -> 2.28 us,
  // 4096 x 256: 3.67 -> 3.00), 32-64 MiB calls lose 2-6 %, large ones are level: chained up to 8 MiB
  const bool use = chain && input_bytes <= (int64_t(8) << 20);
  int pf = -1;
  if (use) {
    const int kb = prefetch_kb_for(grid, operands, input_bytes);  // KiB per CTA and operand
    const int64_t per_warp = (static_cast<int64_t>(kb) << 10) / (block / 32);
    pf = static_cast<int>(per_warp > 65536 ? 65536 : per_warp);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = use ? 1 : 0;
  if (cudaLaunchKernelEx(&cfg, kern, args..., pf) != cudaSuccess) return record_cuda_error();
  return check_launch();
}

template <int M, typename T, bool DOT, int VEC>
static int launch_rows_short(const T* px, const T* py, int64_t ldx, int64_t ldy, int64_t rows, int64_t cols,
                             int leaf_log2, void* out, cudaStream_t stream) {
  using A = typename Acc<M, T>::type;
  constexpr int V = Vec<T>::V;
  auto kern = &rows_short_kernel<M, T, DOT, VEC>;
  const int g_log2 = rows_short_glog2(cols, V);
  const int64_t K = (cols + int64_t(kThreads) * V - 1) / (int64_t(kThreads) * V);
  TFB_CHECK(K <= (int64_t(1) << leaf_log2) / (int64_t(kThreads) * V));
  constexpr int kBlock = TFB_RS_BLOCK;
  const int64_t rows_per_cta = int64_t(kBlock / 32) * (32 >> g_log2);
  const int64_t want = (rows + rows_per_cta - 1) / rows_per_cta;
  const int64_t slots =
      static_cast<int64_t>(device_sms()) * occupancy_of(reinterpret_cast<const void*>(kern), kBlock);
  const unsigned grid = static_cast<unsigned>(want < slots ? want : slots);
  snprintf(g_last_launch, sizeof(g_last_launch),
           "rows_short_kernel<%s,%s,%s,%s> grid=%u block=%d rows=%lld cols=%lld lanes/row=%d leaf_log2=%d",
           method_tag(M), sizeof(T) == 4 ? "f32" : "f64", DOT ? "dot" : "sum",
           VEC == 2 ? "ldg256" : VEC == 1 ? "ldg128" : "scalar", grid, kBlock, static_cast<long long>(rows),
           static_cast<long long>(cols), 1 << g_log2, leaf_log2);
  return launch_rows_chained(kern, grid, kBlock, stream, rows * cols * int64_t(sizeof(T)) * (DOT ? 2 : 1), DOT ? 2 : 1,
                             px, py, ldx, ldy, rows, cols, static_cast<int>(K), g_log2, static_cast<Pair<A>*>(out));
}

// Misaligned one-leaf rows whose x / y share the 32-byte class sequence: class-uniform
// warps (rows.cuh rows_cls_kernel).  TFB_ROWS_CLS=0 disables it (A/B runs).
static int rows_cls_enabled() {
  static const int v = getenv("TFB_ROWS_CLS") ? atoi(getenv("TFB_ROWS_CLS")) : 1;
  return v;
}

template <int M, typename T, bool DOT>
static int launch_rows_cls(const T* px, const T* py, int64_t ldx, int64_t ldy, int64_t rows, int64_t cols,
                           int leaf_log2, void* out, cudaStream_t stream) {
  using A = typename Acc<M, T>::type;
  constexpr int V = Vec<T>::V;
  auto kern = &rows_cls_kernel<M, T, DOT>;
  const int g_log2 = rows_short_glog2(cols, V);
  const int64_t K = (cols + int64_t(kThreads) * V - 1) / (int64_t(kThreads) * V);
  TFB_CHECK(K <= (int64_t(1) << leaf_log2) / (int64_t(kThreads) * V));
  const int64_t pitch = (ldx * int64_t(sizeof(T))) % 32;
  int period = 1;
  while ((pitch * period) % 32) period <<= 1;  // rows until the 32-byte offset repeats
  constexpr int kBlock = TFB_RS_BLOCK;
  const int64_t rows_per_cta = int64_t(kBlock / 32) * (32 >> g_log2);
  const int64_t want = (rows + rows_per_cta - 1) / rows_per_cta + period;  // + a partial super-block
  const int64_t slots =
      static_cast<int64_t>(device_sms()) * occupancy_of(reinterpret_cast<const void*>(kern), kBlock);
  const unsigned grid = static_cast<unsigned>(want < slots ? want : slots);
  snprintf(g_last_launch, sizeof(g_last_launch),
           "rows_cls_kernel<%s,%s,%s,win32> grid=%u block=%d rows=%lld cols=%lld lanes/row=%d period=%d leaf_log2=%d",
           method_tag(M), sizeof(T) == 4 ? "f32" : "f64", DOT ? "dot" : "sum", grid, kBlock,
           static_cast<long long>(rows), static_cast<long long>(cols), 1 << g_log2, period, leaf_log2);
  return launch_rows_chained(kern, grid, kBlock, stream, rows * cols * int64_t(sizeof(T)) * (DOT ? 2 : 1), DOT ? 2 : 1,
                             px, py, ldx, ldy, rows, cols, static_cast<int>(K), g_log2, period,
                             static_cast<Pair<A>*>(out));
}

template <int M, typename T, bool DOT, bool VEC, int NT, int UF = 1, int MS = 0>
static int launch_leaves_nt(const T* px, const T* py, int64_t ldx, int64_t ldy, int64_t rows, int64_t cols,
                            int leaf_log2, int64_t P, void* partials, void* counters, void* out, int fused,
                            cudaStream_t stream, int64_t part_cap = INT64_MAX) {
  using A = typename Acc<M, T>::type;
  const void* fn = reinterpret_cast<const void*>(&leaves_kernel<M, T, DOT, VEC, NT, UF, MS>);
  const int64_t units = rows * P * (kThreads / NT);
  const int64_t slots = static_cast<int64_t>(device_sms()) * occupancy_of(fn, NT);
  const int64_t grid64 = units < slots ? units : slots;
  const unsigned grid = static_cast<unsigned>(grid64 > 0 ? grid64 : 1);
  snprintf(g_last_launch, sizeof(g_last_launch),
           "leaves_kernel<%s,%s,%s,%s,NT=%d,U=%d> grid=%u block=%d units=%lld leaf_log2=%d", method_tag(M),
           sizeof(T) == 4 ? "f32" : "f64", DOT ? "dot" : "sum",
           VEC ? "ldg128" : (MS ? (MS == 1 ? "ldg128-shift1" : MS == 2 ? "ldg128-shift2" : "ldg128-shift3") : "scalar"),
           NT, Unroll<T>::value * UF, grid, NT, static_cast<long long>(units), leaf_log2);
  // programmatic dependent of the previous kernel (the kernel waits before any memory
  // access): a preceding tree kernel's trigger lets these CTAs become resident before it
  // retires, hiding the launch gap between back-to-back calls.  TFB_PDL_CHAIN=0 disables.
  static const bool chain = !getenv("TFB_PDL_CHAIN") || atoi(getenv("TFB_PDL_CHAIN")) != 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = chain ? 1 : 0;
  const int flags = (fused ? kLeavesFused : 0) |
                    ((chain && VEC && NT == kThreads
                          ? prefetch_kb_for(grid, DOT ? 2 : 1, rows * cols * int64_t(sizeof(T)) * (DOT ? 2 : 1))
                          : 0)
                     << kLeavesPrefetchShift);
  if (cudaLaunchKernelEx(&cfg, leaves_kernel<M, T, DOT, VEC, NT, UF, MS>, px, py, ldx, ldy, rows, cols, leaf_log2, P,
                         static_cast<Pair<A>*>(partials), static_cast<unsigned*>(counters),
                         static_cast<Pair<A>*>(out), flags, part_cap) != cudaSuccess)
    return record_cuda_error();
  return check_launch();
}

// Scalar-path (not 16-byte aligned) 256-thread launch: operands that share their
// offset modulo 16 bytes (1-D, or rows whose pitch is a multiple of 16 bytes)
// take the shifted-vector loads (leaf_chain, MS > 0), the rest element loads.
template <int M, typename T, bool DOT>
static int launch_leaves_unaligned(const T* px, const T* py, int64_t ldx, int64_t ldy, int64_t rows, int64_t cols,
                                   int leaf_log2, int64_t P, void* partials, void* counters, void* out, int fused,
                                   cudaStream_t stream, int64_t part_cap) {
  const uintptr_t mx = reinterpret_cast<uintptr_t>(px) & 15u;
  const bool pitch_ok = rows == 1 || ((ldx * int64_t(sizeof(T))) % 16 == 0 &&
                                      (!DOT || (ldy * int64_t(sizeof(T))) % 16 == 0));
  const bool same = !DOT || (reinterpret_cast<uintptr_t>(py) & 15u) == mx;
  // binary32 only: the binary64 variant needs 70 registers (3 CTAs/SM) and measured no
  // faster than element loads (f64 dot 2^27 at offset 1: 338 vs 339-455 us)
  // (measured against the batched element loads below: f32 2^24 dot 23.0-25.9 vs 28.1-28.8 us)
  const int ms = (sizeof(T) == 4 && pitch_ok && same && mx % sizeof(T) == 0) ? static_cast<int>(mx / sizeof(T)) : 0;
#define TFB_UNAL(MSV)                                                                                       \
  launch_leaves_nt<M, T, DOT, false, 256, 1, MSV>(px, py, ldx, ldy, rows, cols, leaf_log2, P, partials, \
                                                   counters, out, fused, stream, part_cap)
  if constexpr (sizeof(T) == 4) {
    if (ms == 1) return TFB_UNAL(1);
    if (ms == 2) return TFB_UNAL(2);
    if (ms == 3) return TFB_UNAL(3);
  }
  return TFB_UNAL(0);
#undef TFB_UNAL
}

template <int M, typename T, bool DOT>
static int launch_leaves(const void* x, const void* y, int64_t ldx, int64_t ldy, int64_t rows,
                         int64_t cols, int leaf_log2, void* partials, void* counters, void* out,
                         int fused, cudaStream_t stream, int64_t partial_capacity = -1,
                         int64_t counter_capacity = -1, const PeerCtx* peer = nullptr, uint32_t epoch = 0) {
  const int64_t P = (cols + (int64_t(1) << leaf_log2) - 1) >> leaf_log2;
  const int64_t units = rows * P;
  if (units == 0) {  // empty shard: still take part in the peer combine with (+0, +0)
    if (peer && fused)
      return launch_rows_tree_pdl<M, typename Acc<M, T>::type>(nullptr, 1, 0, out, stream, 0, peer, epoch);
    return TF_OK;
  }
  const bool vec = aligned16(x) && ((ldx * int64_t(sizeof(T))) % 16 == 0 || rows == 1) &&
                   (!DOT || (aligned16(y) && ((ldy * int64_t(sizeof(T))) % 16 == 0 || rows == 1)));
  auto px = static_cast<const T*>(x);
  auto py = static_cast<const T*>(y);
  // Small 1-D inputs (one-vector leaves, <= 64 of them): a single cluster
  // launch, no scratch, no tail kernel (small.cuh).  Auto tail only.
  if (fused && !peer && rows == 1 && P <= kSmallMaxLeaves && tail_choice() == 0 &&
      (int64_t(1) << leaf_log2) == int64_t(kThreads) * Vec<T>::V)
    return vec ? launch_small<M, T, DOT, true>(px, py, cols, P, out, stream)
               : launch_small<M, T, DOT, false>(px, py, cols, P, out, stream);
  // Many rows of at most one leaf each: a group of lanes per row (rows.cuh).
  if (fused && !peer && rows > 1 && P == 1) {
    const int rk = rows_kernel_choice();
    // aligned rows up to 16 KiB per operand, misaligned pitches up to 1024 columns (lane
    // blocks with aligned loads + selects); a CTA per row above
    if (rk == 2 || (rk == 0 && (vec ? cols * int64_t(sizeof(T)) <= kShortRowMaxBytes : cols <= kShortRowMaxMisCols))) {
      auto a32 = [](const void* p, int64_t ld) {
        return (reinterpret_cast<uintptr_t>(p) & 31u) == 0 && (ld * int64_t(sizeof(T))) % 32 == 0;
      };
      if (vec && a32(x, ldx) && (!DOT || a32(y, ldy)))
        return launch_rows_short<M, T, DOT, 2>(px, py, ldx, ldy, rows, cols, leaf_log2, out, stream);
      // misaligned, x and y on the same 32-byte class sequence: class-uniform warps
      const bool same_cls = !DOT || (((reinterpret_cast<uintptr_t>(x) - reinterpret_cast<uintptr_t>(y)) & 31u) == 0 &&
                                     ((ldx - ldy) * int64_t(sizeof(T))) % 32 == 0);
      if (!vec && same_cls && rows_cls_enabled() && rk == 0 && rows_short_glog2(cols, Vec<T>::V) > 0)
        return launch_rows_cls<M, T, DOT>(px, py, ldx, ldy, rows, cols, leaf_log2, out, stream);
      return vec ? launch_rows_short<M, T, DOT, 1>(px, py, ldx, ldy, rows, cols, leaf_log2, out, stream)
                 : launch_rows_short<M, T, DOT, 0>(px, py, ldx, ldy, rows, cols, leaf_log2, out, stream);
    }
  }
  // partial-pair capacity the kernels may write: callers of the leaves-only mode
  // (tf_reduce_leaves) promise ceil(n/L) pairs
  const int64_t cap = fused ? (partial_capacity < 0 ? 0 : partial_capacity) : units;
  int S = choose_split(units, fused);
  // never exceed the scratch the caller provided (fused mode): S unit pairs per leaf
  // need rows*P*S partials, and any S*P > 1 needs the retire counters
  if (fused) {
    while (S > 1 && (partial_capacity < units * S || !partials || !counters || counter_capacity < rows)) S /= 2;
  }

#define TFB_NT(NT)                                                                                     \
  (vec ? launch_leaves_nt<M, T, DOT, true, NT>(px, py, ldx, ldy, rows, cols, leaf_log2, P, partials,   \
                                               counters, out, fused, stream, cap)                     \
       : launch_leaves_nt<M, T, DOT, false, NT>(px, py, ldx, ldy, rows, cols, leaf_log2, P, partials,  \
                                                counters, out, fused, stream, cap))
  int loader = loader_choice();
  if (loader == 0) {
    const int64_t bytes = rows * cols * static_cast<int64_t>(sizeof(T)) * (DOT ? 2 : 1);
    // the table is measured on 1-D arrays.  Rows: below kTmaRowMinBytes per row the
    // TMA rings never fill (1.8-2.0 TB/s at 16-64 KiB rows): LDG; long rows stream
    // like 1-D arrays, and large row-wise dots take the TMA pipeline (cfg4: 295 vs 303 us)
    const bool long_rows = cols * int64_t(sizeof(T)) >= kTmaRowMinBytes;
    if (rows > 1 && !long_rows) loader = 1;
    else if (rows > 1 && DOT && bytes >= (int64_t(512) << 20)) loader = 2;
    else loader = auto_loader(M, sizeof(T) == 8, DOT, bytes);
  }
  if (vec && fused && S == 1) {
    switch (loader) {
      case 2:
        return launch_leaves_tma<M, T, DOT, 4, 4>(px, py, ldx, ldy, rows, cols, leaf_log2, P, partials, counters,
                                                  out, stream, peer, epoch);
      case 3:
        return launch_leaves_tma<M, T, DOT, 8, 2>(px, py, ldx, ldy, rows, cols, leaf_log2, P, partials, counters,
                                                  out, stream, peer, epoch);
      case 6:  // small rings, 4 CTAs per SM
        return launch_leaves_tma<M, T, DOT, 4, 1, 4>(px, py, ldx, ldy, rows, cols, leaf_log2, P, partials,
                                                     counters, out, stream, peer, epoch);
      case 7:  // small rings, 3 CTAs per SM
        return launch_leaves_tma<M, T, DOT, 4, 2, 3>(px, py, ldx, ldy, rows, cols, leaf_log2, P, partials,
                                                     counters, out, stream, peer, epoch);
      default:
        break;
    }
  }
  const bool deep = vec && S == 1 && loader == 8;  // LDG with twice the loads in flight per thread
  // LDG loader.  Tail: auto/2 = partials-only launch + PDL tree kernel (measured
  // -0.5..-0.8 us on small inputs), 1 = single launch with last-CTA ticket.
  const int tail = tail_choice();
  // The peer combine lives in the PDL tree kernel for the LDG loader (keeping it
  // out of leaves_kernel keeps that kernel at 48 registers / 5 CTAs per SM).
  if (peer && !(partials && partial_capacity >= units * S)) return TF_EWORKSPACE;
  if (fused && (peer || (tail != 1 && units * S > rows)) && partials && partial_capacity >= units * S) {
    int rc;
    if (S == 4) rc = (vec ? launch_leaves_nt<M, T, DOT, true, 64>(px, py, ldx, ldy, rows, cols, leaf_log2, P,
                                                                   partials, nullptr, nullptr, 0, stream, partial_capacity)
                          : launch_leaves_nt<M, T, DOT, false, 64>(px, py, ldx, ldy, rows, cols, leaf_log2, P,
                                                                    partials, nullptr, nullptr, 0, stream, partial_capacity));
    else if (S == 2) rc = (vec ? launch_leaves_nt<M, T, DOT, true, 128>(px, py, ldx, ldy, rows, cols, leaf_log2,
                                                                         P, partials, nullptr, nullptr, 0, stream, partial_capacity)
                               : launch_leaves_nt<M, T, DOT, false, 128>(px, py, ldx, ldy, rows, cols, leaf_log2,
                                                                          P, partials, nullptr, nullptr, 0,
                                                                          stream, partial_capacity));
    else if (deep) rc = launch_leaves_nt<M, T, DOT, true, 256, 2>(px, py, ldx, ldy, rows, cols, leaf_log2, P,
                                                                  partials, nullptr, nullptr, 0, stream,
                                                                  partial_capacity);
    else rc = (vec ? launch_leaves_nt<M, T, DOT, true, 256>(px, py, ldx, ldy, rows, cols, leaf_log2, P, partials,
                                                             nullptr, nullptr, 0, stream, partial_capacity)
                   : launch_leaves_unaligned<M, T, DOT>(px, py, ldx, ldy, rows, cols, leaf_log2, P, partials,
                                                         nullptr, nullptr, 0, stream, partial_capacity));
    if (rc) return rc;
    return launch_rows_tree_pdl<M, typename Acc<M, T>::type>(partials, rows, P * S, out, stream, partial_capacity,
                                                             peer, epoch);
  }
  if (S == 4) return TFB_NT(64);
  if (S == 2) return TFB_NT(128);
  if (deep)
    return launch_leaves_nt<M, T, DOT, true, 256, 2>(px, py, ldx, ldy, rows, cols, leaf_log2, P, partials, counters,
                                                     out, fused, stream, cap);
  if (!vec)
    return launch_leaves_unaligned<M, T, DOT>(px, py, ldx, ldy, rows, cols, leaf_log2, P, partials, counters, out,
                                              fused, stream, cap);
  return TFB_NT(256);
#undef TFB_NT
}

// Sequential flavors: inputs of at least a few chunks whose operands share
// their offset modulo 16 bytes stream through the bulk-copy ring (seqpipe.cuh);
// the rest use the plain one-thread / k-thread kernels.  Same element order.
template <int M, typename T, bool DOT>
static int launch_seq_pipe(const void* x, const void* y, int64_t n, int k, void* out, cudaStream_t s) {
  using A = typename Acc<M, T>::type;
  constexpr int64_t CE = kSeqChunkBytes / sizeof(T);
  const uintptr_t mx = reinterpret_cast<uintptr_t>(x) & 15u;
  if (n < 4 * CE || (DOT && (reinterpret_cast<uintptr_t>(y) & 15u) != mx)) return -1;
  const int64_t head = static_cast<int64_t>((16u - mx) & 15u) / static_cast<int64_t>(sizeof(T));
  const int64_t nchunks = (n - head) / CE;
  auto kern = &seq_pipe_kernel<M, T, DOT>;
  const size_t smem = SeqSmem<T, DOT>::kBytes;
  static std::mutex mu;
  static std::unordered_map<int, bool> ok;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    if (!ok.count(dev)) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
          cudaSuccess)
        return record_cuda_error();
      ok[dev] = true;
    }
  }
  kern<<<1, kSeqThreads, smem, s>>>(static_cast<const T*>(x), static_cast<const T*>(y), n, k, head, nchunks,
                                     static_cast<Pair<A>*>(out));
  return check_launch();
}

// seq flavor with the s / e chains decoupled (seqsplit.cuh): direct, wide, fast and
// rigorous, no TwoProduct; same preconditions as the bulk-copy ring.  TFB_SEQ_SPLIT=0
// keeps seq_pipe_kernel (A/B runs).
template <int M, typename T, bool DOT>
static int launch_seq_split(const void* x, const void* y, int64_t n, void* out, cudaStream_t s) {
  using A = typename Acc<M, T>::type;
  static const bool on = !getenv("TFB_SEQ_SPLIT") || atoi(getenv("TFB_SEQ_SPLIT")) != 0;
  if constexpr (M == kKahan || is_tp<M>()) {
    return -1;
  } else {
    constexpr int64_t CE = SplitSmem<M, T, DOT>::CE;
    const uintptr_t mx = reinterpret_cast<uintptr_t>(x) & 15u;
    if (!on || n < 4 * CE || (DOT && (reinterpret_cast<uintptr_t>(y) & 15u) != mx)) return -1;
    const int64_t head = static_cast<int64_t>((16u - mx) & 15u) / static_cast<int64_t>(sizeof(T));
    const int64_t nchunks = (n - head) / CE;
    auto kern = &seq_split_kernel<M, T, DOT>;
    const size_t smem = SplitSmem<M, T, DOT>::kBytes;
    static std::mutex mu;
    static std::unordered_map<int, bool> ok;
    {
      int dev = 0;
      cudaGetDevice(&dev);
      std::lock_guard<std::mutex> g(mu);
      if (!ok.count(dev)) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
            cudaSuccess)
          return record_cuda_error();
        ok[dev] = true;
      }
    }
    kern<<<1, kSplitThreads, smem, s>>>(static_cast<const T*>(x), static_cast<const T*>(y), n, head, nchunks,
                                         static_cast<Pair<A>*>(out));
    return check_launch();
  }
}

template <int M, typename T, bool DOT>
static int launch_seq(const void* x, const void* y, int64_t n, void* out, cudaStream_t s) {
  using A = typename Acc<M, T>::type;
  const int rs = launch_seq_split<M, T, DOT>(x, y, n, out, s);
  if (rs >= 0) return rs;
  const int rc = launch_seq_pipe<M, T, DOT>(x, y, n, 1, out, s);
  if (rc >= 0) return rc;
  seq_kernel<M, T, DOT><<<1, 1, 0, s>>>(static_cast<const T*>(x), static_cast<const T*>(y), n,
                                        static_cast<Pair<A>*>(out));
  return check_launch();
}

template <int M, typename T, bool DOT>
static int launch_lanes(const void* x, const void* y, int64_t n, int k, void* out, cudaStream_t s) {
  using A = typename Acc<M, T>::type;
  const int rc = launch_seq_pipe<M, T, DOT>(x, y, n, k, out, s);
  if (rc >= 0) return rc;
  lanes_kernel<M, T, DOT><<<1, k, 0, s>>>(static_cast<const T*>(x), static_cast<const T*>(y), n, k,
                                          static_cast<Pair<A>*>(out));
  return check_launch();
}

template <int M, typename T, bool DOT>
static int launch_noread(const void* seed8, int64_t iters, int64_t blocks, void* out, cudaStream_t s) {
  using A = typename Acc<M, T>::type;
  noread_kernel<M, T, DOT><<<static_cast<unsigned>(blocks), kThreads, 0, s>>>(
      static_cast<const T*>(seed8), iters, static_cast<Pair<A>*>(out));
  return check_launch();
}

template <int M, typename A>
static int launch_tree(const void* pairs, int64_t count, void* out, cudaStream_t s) {
  tree_kernel<M, A><<<1, kThreads, 0, s>>>(static_cast<const Pair<A>*>(pairs), count,
                                           static_cast<Pair<A>*>(out));
  return check_launch();
}

// Method x dtype x {sum, dot} dispatch.  WIDE exists for f32 data only
// (kernels.py:600-601).
#define TFB_DISPATCH(method, dtype, dot, CALL)                                   \
  do {                                                                           \
    if ((dtype) != TF_F32 && (dtype) != TF_F64) return TF_EINVAL_DTYPE;          \
    if ((method) == TF_WIDE && (dtype) != TF_F32) return TF_EINVAL_DTYPE;        \
    switch (method) {                                                            \
      case TF_DIRECT:                                                            \
        if ((dtype) == TF_F32) { if (dot) return CALL(kDirect, float, true);     \
                                 else return CALL(kDirect, float, false); }      \
        else { if (dot) return CALL(kDirect, double, true);                      \
               else return CALL(kDirect, double, false); }                       \
      case TF_WIDE:                                                              \
        if (dot) return CALL(kWide, float, true);                                \
        else return CALL(kWide, float, false);                                   \
      case TF_TWOFOLD_FAST:                                                      \
        if ((dtype) == TF_F32) { if (dot) return CALL(kFast, float, true);       \
                                 else return CALL(kFast, float, false); }        \
        else { if (dot) return CALL(kFast, double, true);                        \
               else return CALL(kFast, double, false); }                         \
      case TF_TWOFOLD_RIGOROUS:                                                  \
        if ((dtype) == TF_F32) { if (dot) return CALL(kRigorous, float, true);   \
                                 else return CALL(kRigorous, float, false); }    \
        else { if (dot) return CALL(kRigorous, double, true);                    \
               else return CALL(kRigorous, double, false); }                     \
      case TF_KAHAN:                                                             \
        if ((dtype) == TF_F32) { if (dot) return CALL(kKahan, float, true);      \
                                 else return CALL(kKahan, float, false); }       \
        else { if (dot) return CALL(kKahan, double, true);                       \
               else return CALL(kKahan, double, false); }                        \
      case kFastTP:                                                              \
        if (!(dot)) return TF_EINVAL_ARG;                                        \
        if ((dtype) == TF_F32) return CALL(kFastTP, float, true);                \
        else return CALL(kFastTP, double, true);                                 \
      case kRigorousTP:                                                          \
        if (!(dot)) return TF_EINVAL_ARG;                                        \
        if ((dtype) == TF_F32) return CALL(kRigorousTP, float, true);            \
        else return CALL(kRigorousTP, double, true);                             \
      default:                                                                   \
        return TF_EINVAL_METHOD;                                                 \
    }                                                                            \
  } while (0)

static size_t pair_bytes(int method, int dtype) {
  return ((method & ~TF_TRACK_PRODUCT) == TF_WIDE || dtype == TF_F64) ? 16u : 8u;
}

// Public method id (+ TF_TRACK_PRODUCT flag) -> internal Method id.
static int internal_method(int method) {
  const int base = method & ~TF_TRACK_PRODUCT;
  if (!(method & TF_TRACK_PRODUCT)) return base;
  if (base == TF_TWOFOLD_FAST) return kFastTP;
  if (base == TF_TWOFOLD_RIGOROUS) return kRigorousTP;
  return -1;
}

static int validate(int method, int dtype) {
  const int base = method & ~TF_TRACK_PRODUCT;
  if (base < TF_DIRECT || base > TF_KAHAN) return TF_EINVAL_METHOD;
  if (dtype != TF_F32 && dtype != TF_F64) return TF_EINVAL_DTYPE;
  if (base == TF_WIDE && dtype != TF_F32) return TF_EINVAL_DTYPE;
  if (internal_method(method) < 0) return TF_EINVAL_ARG;  // TwoProduct needs a twofold method
  return TF_OK;
}

static int resolve_leaf(int dtype, int64_t total, int leaf_log2, int* out) {
  if (leaf_log2 == 0) {
    *out = auto_leaf_log2(dtype, total);
    return TF_OK;
  }
  if (leaf_log2 < floor_leaf_log2(dtype) || leaf_log2 > 24) return TF_EINVAL_ARG;
  *out = leaf_log2;
  return TF_OK;
}

}  // namespace tfb

using namespace tfb;

extern "C" {

const char* tf_last_launch(void) { return g_last_launch; }

int tf_set_tail(int tail) {
  if (tail < 0 || tail > 2) return TF_EINVAL_ARG;
  g_tail = tail;
  return TF_OK;
}

int tf_set_prefetch(int kib) {
  if (kib < -1 || kib > 512) return TF_EINVAL_ARG;
  g_prefetch_kb = kib;
  return TF_OK;
}

int tf_set_loader(int loader) {
  if (loader < 0 || loader > 8 || loader == 4 || loader == 5) return TF_EINVAL_ARG;
  g_loader = loader;
  return TF_OK;
}

int tf_set_rows_kernel(int kind) {
  if (kind < 0 || kind > 2) return TF_EINVAL_ARG;
  g_rows_kernel = kind;
  return TF_OK;
}

int tf_set_leaf_split(int split) {
  if (split != 0 && split != 1 && split != 2 && split != 4) return TF_EINVAL_ARG;
  g_split_override = split;
  return TF_OK;
}

int tf_leaf_log2(int dtype, int64_t n) {
  if (dtype != TF_F32 && dtype != TF_F64) return -TF_EINVAL_DTYPE;
  return auto_leaf_log2(dtype, n);
}

int tf_workspace_size(int method, int dtype, int64_t rows, int64_t cols, int leaf_log2,
                      size_t* partials_bytes, int64_t* counters, int64_t* leaves) {
  int rc = validate(method, dtype);
  if (rc) return rc;
  if (rows < 0 || cols < 0) return TF_EINVAL_SHAPE;
  int lg;
  if ((rc = resolve_leaf(dtype, rows * cols, leaf_log2, &lg))) return rc;
  const int64_t P = (cols + (int64_t(1) << lg) - 1) >> lg;
  // sized for the largest leaf split (kMaxSplit unit pairs per leaf).  Many rows of one
  // leaf each need no scratch at all (every row pair is stored straight into out).
  const bool none = rows > 1 && P <= 1;
  if (partials_bytes)
    *partials_bytes = none ? 0 : static_cast<size_t>(rows * P * kMaxSplit) * pair_bytes(method, dtype);
  if (counters) *counters = none ? 0 : rows;
  if (leaves) *leaves = P;
  return TF_OK;
}

}  // extern "C"

static int reduce_rows_impl(int method, int dtype, const void* x, const void* y, int64_t rows, int64_t cols,
                            int64_t ldx, int64_t ldy, int leaf_log2, void* out_pairs, void* partials,
                            size_t partials_bytes, void* counters, int64_t counters_len, void* stream,
                            const PeerCtx* peer, uint32_t epoch) {
  int rc = validate(method, dtype);
  if (rc) return rc;
  if (rows < 0 || cols < 0) return TF_EINVAL_SHAPE;
  if (rows > 1 && (ldx < cols || (y && ldy < cols))) return TF_EINVAL_SHAPE;
  if (peer && rows != 1) return TF_EINVAL_ARG;  // the peer combine merges one row across ranks
  if (rows == 0) return TF_OK;
  if (!out_pairs || (cols > 0 && !x)) return TF_EINVAL_ARG;
  int lg;
  if ((rc = resolve_leaf(dtype, rows * cols, leaf_log2, &lg))) return rc;
  auto s = static_cast<cudaStream_t>(stream);
  if (cols == 0 && !peer) {  // every row is empty: (+0, +0)
    if (cudaMemsetAsync(out_pairs, 0, static_cast<size_t>(rows) * pair_bytes(method, dtype), s) !=
        cudaSuccess)
      return record_cuda_error();
    return TF_OK;
  }
  int64_t P = (cols + (int64_t(1) << lg) - 1) >> lg;
  const size_t min_need = static_cast<size_t>(rows * P) * pair_bytes(method, dtype);
  if (P > 1 && (!partials || partials_bytes < min_need || !counters || counters_len < rows))
    return TF_EWORKSPACE;
  const int64_t capacity = partials ? static_cast<int64_t>(partials_bytes / pair_bytes(method, dtype)) : 0;
  void* parts = partials;
  const bool dot = y != nullptr;
#define TFB_CALL_LEAVES(M, T, DOT) \
  launch_leaves<M, T, DOT>(x, y, ldx, ldy, rows, cols, lg, parts, counters, out_pairs, 1, s, capacity, \
                           counters ? counters_len : 0, peer, epoch)
  TFB_DISPATCH(internal_method(method), dtype, dot, TFB_CALL_LEAVES);
#undef TFB_CALL_LEAVES
}

extern "C" {

int tf_reduce_rows(int method, int dtype, const void* x, const void* y, int64_t rows, int64_t cols,
                   int64_t ldx, int64_t ldy, int leaf_log2, void* out_pairs, void* partials,
                   size_t partials_bytes, void* counters, int64_t counters_len, void* stream) {
  return reduce_rows_impl(method, dtype, x, y, rows, cols, ldx, ldy, leaf_log2, out_pairs, partials,
                          partials_bytes, counters, counters_len, stream, nullptr, 0);
}

int tf_reduce(int method, int dtype, const void* x, const void* y, int64_t n, int leaf_log2,
              void* out_pair, void* partials, size_t partials_bytes, void* counters,
              int64_t counters_len, void* stream) {
  if (n < 0) return TF_EINVAL_SHAPE;
  return tf_reduce_rows(method, dtype, x, y, 1, n, n, n, leaf_log2, out_pair, partials,
                        partials_bytes, counters, counters_len, stream);
}

int tf_reduce_peer(int method, int dtype, const void* x, const void* y, int64_t n, int leaf_log2,
                   void* out_pair, void* partials, size_t partials_bytes, void* counters,
                   int64_t counters_len, const void* peer_ctx, uint32_t epoch, void* stream) {
  if (n < 0) return TF_EINVAL_SHAPE;
  if (!peer_ctx || epoch == 0) return TF_EINVAL_ARG;
  return reduce_rows_impl(method, dtype, x, y, 1, n, n, n, leaf_log2, out_pair, partials, partials_bytes,
                          counters, counters_len, stream, static_cast<const PeerCtx*>(peer_ctx), epoch);
}

int tf_peer_ctx_size(void) { return static_cast<int>(sizeof(PeerCtx)); }

int tf_reduce_leaves(int method, int dtype, const void* x, const void* y, int64_t n, int leaf_log2,
                     void* partials_out, void* stream) {
  int rc = validate(method, dtype);
  if (rc) return rc;
  if (n < 0) return TF_EINVAL_SHAPE;
  if (n == 0) return TF_OK;
  if (!x || !partials_out) return TF_EINVAL_ARG;
  int lg;
  if ((rc = resolve_leaf(dtype, n, leaf_log2, &lg))) return rc;
  auto s = static_cast<cudaStream_t>(stream);
  const bool dot = y != nullptr;
#define TFB_CALL_PARTS(M, T, DOT) \
  launch_leaves<M, T, DOT>(x, y, n, n, 1, n, lg, partials_out, nullptr, nullptr, 0, s)
  TFB_DISPATCH(internal_method(method), dtype, dot, TFB_CALL_PARTS);
#undef TFB_CALL_PARTS
}

int tf_merge_tree(int method, int dtype, const void* pairs, int64_t count, void* out_pair,
                  void* stream) {
  int rc = validate(method, dtype);
  if (rc) return rc;
  if (count < 0) return TF_EINVAL_SHAPE;
  if (!out_pair || (count > 0 && !pairs)) return TF_EINVAL_ARG;
  auto s = static_cast<cudaStream_t>(stream);
  switch (method & ~TF_TRACK_PRODUCT) {  // TwoProduct pairs merge like their base method
    case TF_DIRECT:
      return dtype == TF_F32 ? launch_tree<kDirect, float>(pairs, count, out_pair, s)
                             : launch_tree<kDirect, double>(pairs, count, out_pair, s);
    case TF_WIDE:
      return launch_tree<kWide, double>(pairs, count, out_pair, s);
    case TF_TWOFOLD_FAST:
      return dtype == TF_F32 ? launch_tree<kFast, float>(pairs, count, out_pair, s)
                             : launch_tree<kFast, double>(pairs, count, out_pair, s);
    case TF_TWOFOLD_RIGOROUS:
      return dtype == TF_F32 ? launch_tree<kRigorous, float>(pairs, count, out_pair, s)
                             : launch_tree<kRigorous, double>(pairs, count, out_pair, s);
    default:
      return dtype == TF_F32 ? launch_tree<kKahan, float>(pairs, count, out_pair, s)
                             : launch_tree<kKahan, double>(pairs, count, out_pair, s);
  }
}

int tf_noread(int method, int dtype, int dot, const void* seed8, int64_t iters, int64_t blocks,
              void* out_pairs, void* stream) {
  int rc = validate(method, dtype);
  if (rc) return rc;
  if (iters < 0 || blocks < 1 || !seed8 || !out_pairs) return TF_EINVAL_ARG;
  auto s = static_cast<cudaStream_t>(stream);
#define TFB_CALL_NOREAD(M, T, DOT) launch_noread<M, T, DOT>(seed8, iters, blocks, out_pairs, s)
  TFB_DISPATCH(internal_method(method), dtype, dot != 0, TFB_CALL_NOREAD);
#undef TFB_CALL_NOREAD
}

int tf_reduce_seq(int method, int dtype, const void* x, const void* y, int64_t n, void* out_pair,
                  void* stream) {
  int rc = validate(method, dtype);
  if (rc) return rc;
  if (n < 0) return TF_EINVAL_SHAPE;
  if (!out_pair || (n > 0 && !x)) return TF_EINVAL_ARG;
  auto s = static_cast<cudaStream_t>(stream);
  const bool dot = y != nullptr;
#define TFB_CALL_SEQ(M, T, DOT) launch_seq<M, T, DOT>(x, y, n, out_pair, s)
  TFB_DISPATCH(internal_method(method), dtype, dot, TFB_CALL_SEQ);
#undef TFB_CALL_SEQ
}

int tf_reduce_lanes(int method, int dtype, const void* x, const void* y, int64_t n, int lanes,
                    void* out_pair, void* stream) {
  int rc = validate(method, dtype);
  if (rc) return rc;
  if (n < 0) return TF_EINVAL_SHAPE;
  if (lanes < 2 || lanes > 16 || (lanes & (lanes - 1))) return TF_EINVAL_ARG;
  if (!out_pair || (n > 0 && !x)) return TF_EINVAL_ARG;
  auto s = static_cast<cudaStream_t>(stream);
  const bool dot = y != nullptr;
#define TFB_CALL_LANES(M, T, DOT) launch_lanes<M, T, DOT>(x, y, n, lanes, out_pair, s)
  TFB_DISPATCH(internal_method(method), dtype, dot, TFB_CALL_LANES);
#undef TFB_CALL_LANES
}

}  // extern "C"

#ifdef TFB_TRACE
// Tuning builds only: where the kernels' %globaltimer stamps go (device pointer, >= 8 * 4104 u64; null = off).
extern "C" int tf_trace_buffer(void* dev_u64) {
  unsigned long long* p = static_cast<unsigned long long*>(dev_u64);
  return cudaMemcpyToSymbol(tfb::tfb_trace_ptr, &p, sizeof(p)) == cudaSuccess ? TF_OK : TF_ECUDA;
}
#endif
