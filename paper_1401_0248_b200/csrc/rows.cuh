// rows.cuh — short-row kernel of the rows family (tf_reduce_rows): rows that
// fit in one leaf (cols <= L = 2^leaf_log2), reduced by a group of G lanes
// instead of a 256-thread CTA.  Included by reduce.cu after the shared helpers.
//
// Same chains and the same balanced tree as leaves_kernel, so each row is
// bit-identical to the CTA-per-leaf path (and to the 1-D reduction of the row):
//   * chain t (0..255) runs the recurrence over the row's elements
//     (k*256 + t)*V + j, k = 0..K-1, j = 0..V-1 (elements >= cols skipped);
//   * lane j of the row's group owns chains 8j..8j+7, i.e. for every k one
//     contiguous block of 8 vectors (128 bytes per operand);
//   * the tree: 3 levels inside the lane (its aligned 8-chain subtree), log2(G)
//     shuffle levels across the group, then the levels above 8G chains merge
//     with the all-zero right subtrees, whose tree is exactly (+0, +0).  Those
//     merges are executed, not skipped (they normalise -0 exactly as the full
//     tree does).
// G = pow2ceil(lanes holding data) <= 32; a warp reduces 32/G rows at a time,
// so a 16-element row costs one lane, not a CTA.

namespace tfb {

#ifndef TFB_RS_MINB
#define TFB_RS_MINB 0  // tuning builds: min resident CTAs per SM (0 = unconstrained, measured best)
#endif
#ifndef TFB_RS_PARTS
#define TFB_RS_PARTS 0  // batches the lane's 8 vectors per k are loaded in (0 = f32: 2, f64: 1; measured)
#endif
#ifndef TFB_RS_SELECT64
#define TFB_RS_SELECT64 1  // the misaligned select path for binary64 too (measured, profiles/r01_summary.md)
#endif
#ifndef TFB_RS_BLOCK
#define TFB_RS_BLOCK 256  // threads per CTA (any multiple of 32 up to 256)
#endif
#if TFB_RS_MINB > 0
#define TFB_RS_BOUNDS __launch_bounds__(kThreads, TFB_RS_MINB)
#else
#define TFB_RS_BOUNDS __launch_bounds__(kThreads)
#endif

// 32-byte streaming loads (LDG.E...256): lane blocks are 128 bytes apart, so a
// 16-byte load would use half of every 32-byte sector it touches (and, with no
// L1 allocation, fetch each sector twice); 32 bytes per lane use all of it.
__device__ __forceinline__ void ld_stream32(const float4* p, float4& a, float4& b) {
  asm("ld.global.nc.L1::no_allocate.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
      : "l"(p));
}
__device__ __forceinline__ void ld_stream32(const double2* p, double2& a, double2& b) {
  asm("ld.global.nc.L1::no_allocate.L2::256B.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
      : "l"(p));
}

// Misaligned lane blocks: 16-byte __ldg vectors (binary32) or 32-byte windows
// (binary64); measured per dtype (profiles/r02_rows_misaligned.txt: 32-byte windows
// +20-30 % for binary64, -25 % for binary32 whose selects then dominate).
// TFB_RS_MISLD overrides for tuning builds: 0 = 16-byte, 2 = 32-byte windows.
#ifndef TFB_RS_MISLD
#define TFB_RS_MISLD (-1)
#endif
template <typename T>
__host__ __device__ constexpr int mis_ld_kind() {
  return TFB_RS_MISLD >= 0 ? TFB_RS_MISLD : (sizeof(T) == 8 ? 2 : 0);
}

// Five 16-byte vectors of the row starting at the aligned vector holding element p[0]
// (misaligned by m elements): three 32-byte loads (LDG.E.256, whole sectors) at the
// 32-byte boundary below, then the 16-byte half is chosen per row.  Only 32-byte
// blocks holding one of the `rem` row elements from p are read.
template <typename T>
__device__ __forceinline__ void window32(const T* p, int m, int64_t rem, typename Vec<T>::type (&out)[5]) {
  using VT = typename Vec<T>::type;
  constexpr int V = Vec<T>::V;
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const int mv = (a & 16u) ? 1 : 0;  // p's 16-byte vector is the upper half of its 32-byte block
  const VT* base = reinterpret_cast<const VT*>(a & ~uintptr_t(31));
  VT c[6];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int64_t first = int64_t(2 * i) * V - (mv * V + m);  // element index (from p) of the block's start
    if (first < rem && (i < 2 || mv * V + m > 0)) {
      ld_stream32(base + 2 * i, c[2 * i], c[2 * i + 1]);
    } else {
      c[2 * i] = VT{};
      c[2 * i + 1] = VT{};
    }
  }
#pragma unroll
  for (int w = 0; w < 5; ++w) out[w] = mv ? c[w + 1] : c[w];
}

// Cross-call preamble of the short-row kernels (launched as programmatic dependents, like
// leaves_kernel): lane 0 of every warp asks the L2 for the contiguous span of the warp's
// first rows [p, p + bytes) — trimmed to whole 16-byte units inside the span, a hint only —
// then the CTA waits for the previous grid before any memory access.
__device__ __forceinline__ void prefetch_span(const void* p, int64_t bytes, int cap) {
  const uintptr_t a = (reinterpret_cast<uintptr_t>(p) + 15u) & ~uintptr_t(15);
  int64_t n = bytes - static_cast<int64_t>(a - reinterpret_cast<uintptr_t>(p));
  if (n > cap) n = cap;
  n &= ~int64_t(15);
  if (n > 0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<const void*>(a)),
                 "r"(static_cast<unsigned>(n))
                 : "memory");
}

// One 16-byte vector through a chain (elements in order).
template <int M, typename T, bool DOT>
__device__ __forceinline__ void chain_vec(Pair<typename Acc<M, T>::type>& st, const typename Vec<T>::type& a,
                                          const typename Vec<T>::type& b) {
#pragma unroll
  for (int q = 0; q < Vec<T>::V; ++q) {
    if constexpr (DOT) accumulate<M, T, true>(st, vget(a, q), vget(b, q));
    else accumulate<M, T, false>(st, vget(a, q), T(0));
  }
}

// flat[m + i] of a run of elements read m (runtime, < V) before the wanted start;
// i is a compile-time index after unrolling, so flat stays in registers.
template <typename T, int N>
__device__ __forceinline__ T pick_at(const T (&flat)[N], int m, int i) {
  if constexpr (Vec<T>::V == 2) {
    return m ? flat[i + 1] : flat[i];
  } else {
    return m == 0 ? flat[i] : m == 1 ? flat[i + 1] : m == 2 ? flat[i + 2] : flat[i + 3];
  }
}

// VEC: 0 = element loads (misaligned rows), 1 = 16-byte loads (16-byte aligned
// rows), 2 = 32-byte loads (32-byte aligned rows).  Same elements, same order.
template <int M, typename T, bool DOT, int VEC>
__global__ void TFB_RS_BOUNDS rows_short_kernel(
    const T* __restrict__ x, const T* __restrict__ y, int64_t ldx, int64_t ldy, int64_t rows, int64_t cols,
    int K, int g_log2, Pair<typename Acc<M, T>::type>* __restrict__ out, int chain) {  // chain: -1 plain launch, else bytes per warp and operand to prefetch
  using A = typename Acc<M, T>::type;
  using VT = typename Vec<T>::type;
  constexpr int V = Vec<T>::V;
  constexpr int kChains = 8;  // chains per lane
  const int lane = threadIdx.x & 31;
  const int G = 1 << g_log2;
  const int j = lane & (G - 1);  // lane within the row's group
  const int64_t groups = 32 >> g_log2;
  const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  if (chain >= 0) {
    const int64_t rf = warp * groups;
    if (chain > 0 && lane == 0 && rf < rows) {
      const int64_t nr = rows - rf < groups ? rows - rf : groups;  // the warp's first rows: one contiguous span
      prefetch_span(x + rf * ldx, ((nr - 1) * ldx + cols) * static_cast<int64_t>(sizeof(T)), chain);
      if constexpr (DOT) prefetch_span(y + rf * ldy, ((nr - 1) * ldy + cols) * static_cast<int64_t>(sizeof(T)), chain);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  // the loop bound is warp-uniform: every lane reaches every shuffle
  for (int64_t r0 = warp * groups; r0 < rows; r0 += nwarps * groups) {
    const int64_t r = r0 + (lane >> g_log2);
    Pair<A> ch[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) ch[c] = zero_pair<A>();
    if (r < rows) {
      const T* xr = x + r * ldx;
      const T* yr = DOT ? y + r * ldy : nullptr;
      for (int k = 0; k < K; ++k) {
        const int64_t e0 = (int64_t(k) * kThreads + kChains * j) * V;  // this lane's block of 8 vectors
        if (e0 >= cols) break;
        const int64_t rem = cols - e0;  // > 0
        if (VEC != 0 && rem >= kChains * V) {
          TFB_CHECK((reinterpret_cast<uintptr_t>(xr + e0) & (VEC == 2 ? 31u : 15u)) == 0);
          const VT* xv = reinterpret_cast<const VT*>(xr + e0);
          const VT* yv = DOT ? reinterpret_cast<const VT*>(yr + e0) : nullptr;
          constexpr int kParts = TFB_RS_PARTS > 0 ? TFB_RS_PARTS : (sizeof(T) == 8 ? 1 : 2);
          constexpr int kPer = kChains / kParts;
#pragma unroll
          for (int h = 0; h < kParts; ++h) {  // batches of vectors: loads first, then the chains
            VT a[kPer], b[kPer];
            if constexpr (VEC == 2) {
#pragma unroll
              for (int c = 0; c < kPer; c += 2) {
                ld_stream32(xv + kPer * h + c, a[c], a[c + 1]);
                if constexpr (DOT) ld_stream32(yv + kPer * h + c, b[c], b[c + 1]);
              }
            } else {
#pragma unroll
              for (int c = 0; c < kPer; ++c) {
                a[c] = ld_stream(xv + kPer * h + c);
                if constexpr (DOT) b[c] = ld_stream(yv + kPer * h + c);
              }
            }
#pragma unroll
            for (int c = 0; c < kPer; ++c) chain_vec<M, T, DOT>(ch[kPer * h + c], a[c], b[c]);
          }
        } else if (VEC != 0) {
          // partial block (the row's end): whole vectors where they fit, then the
          // elements of the last partial vector — each chain still in element order
          const VT* xv = reinterpret_cast<const VT*>(xr + e0);
          const VT* yv = DOT ? reinterpret_cast<const VT*>(yr + e0) : nullptr;
#pragma unroll
          for (int c = 0; c < kChains; c += 2) {
            const int64_t o = int64_t(c) * V;
            if (o >= rem) break;
            VT a0, a1, b0, b1;
            if (VEC == 2 && o + 2 * V <= rem) {
              ld_stream32(xv + c, a0, a1);
              if constexpr (DOT) ld_stream32(yv + c, b0, b1);
              chain_vec<M, T, DOT>(ch[c], a0, b0);
              chain_vec<M, T, DOT>(ch[c + 1], a1, b1);
              continue;
            }
#pragma unroll
            for (int cc = c; cc < c + 2; ++cc) {
              const int64_t oo = int64_t(cc) * V;
              if (oo + V <= rem) {
                a0 = ld_stream(xv + cc);
                if constexpr (DOT) b0 = ld_stream(yv + cc);
                chain_vec<M, T, DOT>(ch[cc], a0, b0);
              } else {
#pragma unroll
                for (int q = 0; q < V; ++q)
                  if (oo + q < rem) accumulate<M, T, DOT>(ch[cc], xr[e0 + oo + q], DOT ? yr[e0 + oo + q] : T(0));
              }
            }
          }
        } else if ((sizeof(T) == 4 || TFB_RS_SELECT64) && (rem >= kChains * V || g_log2 > 0)) {
          // misaligned binary32 row (pitch not a multiple of 16 bytes): aligned 16-byte
          // loads around the block (only vectors holding a row element: every address
          // read lies in a 16-byte block of the row), each element picked at the row's
          // offset m by selects (per operand; not local memory), two halves of 4
          // vectors; a partial last block is masked element-wise (rows of one lane — at most
          // 8V elements — measured faster with element loads).  binary64: +54-72 % at 63-255
          // columns, -17 % at 17 (its registers), kept.
          const int mx = static_cast<int>((reinterpret_cast<uintptr_t>(xr + e0) & 15u) / sizeof(T));
          const int my = DOT ? static_cast<int>((reinterpret_cast<uintptr_t>(yr + e0) & 15u) / sizeof(T)) : 0;
          const VT* xa = reinterpret_cast<const VT*>(xr + e0 - mx);
          const VT* ya = DOT ? reinterpret_cast<const VT*>(yr + e0 - my) : nullptr;
          const bool whole = rem >= kChains * V;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (!whole && int64_t(4 * h) * V >= rem) break;
            VT a[5], b[5];
            if constexpr (mis_ld_kind<T>() == 2) {
              window32<T>(xr + e0 + int64_t(4 * h) * V, mx, rem - int64_t(4 * h) * V, a);
              if constexpr (DOT) window32<T>(yr + e0 + int64_t(4 * h) * V, my, rem - int64_t(4 * h) * V, b);
            } else {
#pragma unroll
              for (int w = 0; w < 5; ++w) {
                const int64_t fx = int64_t(4 * h + w) * V - mx;  // first element of the vector
                a[w] = (w < 4 || mx) && fx < rem ? __ldg(xa + 4 * h + w) : VT{};
                if constexpr (DOT) {
                  const int64_t fy = int64_t(4 * h + w) * V - my;
                  b[w] = (w < 4 || my) && fy < rem ? __ldg(ya + 4 * h + w) : VT{};
                }
              }
            }
            T fa[5 * V], fb[5 * V];
#pragma unroll
            for (int w = 0; w < 5; ++w)
#pragma unroll
              for (int q = 0; q < V; ++q) {
                fa[w * V + q] = vget(a[w], q);
                if constexpr (DOT) fb[w * V + q] = vget(b[w], q);
              }
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
              for (int q = 0; q < V; ++q) {
                if (!whole && int64_t(4 * h + c) * V + q >= rem) continue;
                const T xv = pick_at(fa, mx, c * V + q);
                if constexpr (DOT) accumulate<M, T, true>(ch[4 * h + c], xv, pick_at(fb, my, c * V + q));
                else accumulate<M, T, false>(ch[4 * h + c], xv, T(0));
              }
          }
        } else {
#pragma unroll
          for (int c = 0; c < kChains; ++c)
#pragma unroll
            for (int q = 0; q < V; ++q) {
              const int64_t i = e0 + c * V + q;
              if (i < cols) accumulate<M, T, DOT>(ch[c], xr[i], DOT ? yr[i] : T(0));
            }
        }
      }
    }
    // the lane's aligned 8-chain subtree
#pragma unroll
    for (int w = 1; w < kChains; w <<= 1)
#pragma unroll
      for (int c = 0; c < kChains; c += 2 * w) ch[c] = merge<M, A>(ch[c], ch[c + w]);
    Pair<A> st = ch[0];
    // across the group's lanes (balanced, left operand = lower lane)
    for (int off = 1; off < G; off <<= 1) {
      Pair<A> o;
      o.s = __shfl_down_sync(0xffffffffu, st.s, off, G);
      if constexpr (HasErr<M>::value) o.e = __shfl_down_sync(0xffffffffu, st.e, off, G);
      else o.e = A(0);
      if ((j & (2 * off - 1)) == 0) st = merge<M, A>(st, o);
    }
    if (j == 0 && r < rows) {
      // levels 3 + g_log2 .. 7 of the 256-chain tree: right subtrees are all zero
      for (int lv = 3 + g_log2; lv < 8; ++lv) st = merge<M, A>(st, zero_pair<A>());
      out[r] = st;
    }
  }
}

// Misaligned pitches, class-uniform warps (rows_cls_kernel).  Row r's lane blocks
// all sit at the same offset MOFF (elements) past a 32-byte boundary — the row
// start's offset, since blocks are 128 bytes apart — and that offset repeats
// with period p = 32 / gcd(ld * sizeof T, 32) rows.  Warps are therefore given
// rows of ONE residue class mod p (rows q, q + p, q + 2p, ... of a super-block),
// so MOFF is warp-uniform and a compile-time constant after one switch: each
// lane block is read with five 32-byte loads (LDG.E.256, whole sectors; the
// window shared by the two halves loaded once) and its elements are picked by
// compile-time register indices — no per-element selects.  Used when x and y
// share the class sequence (same base offset and pitch mod 32 bytes, e.g. two
// views of the same shape); the chains, their order and the tree are exactly
// rows_short_kernel's, so the bits are too.
#ifndef TFB_CLS_ALL
#define TFB_CLS_ALL 0  // tuning builds: 1 = load the block's five windows before any chain step
#endif
template <int M, typename T, bool DOT, int MOFF>
__device__ __forceinline__ void cls_rows_chains(Pair<typename Acc<M, T>::type> (&ch)[8], const T* xr, const T* yr,
                                                int64_t cols, int K, int j) {
  using VT = typename Vec<T>::type;
  constexpr int V = Vec<T>::V;
  constexpr int W = 32 / sizeof(T);  // elements per 32-byte window
  constexpr int kChains = 8;
  for (int k = 0; k < K; ++k) {
    const int64_t e0 = (int64_t(k) * kThreads + kChains * j) * V;  // the lane's block: elements [e0, e0 + 8V)
    if (e0 >= cols) break;
    const int64_t rem = cols - e0;
    const VT* base = reinterpret_cast<const VT*>(xr + e0 - MOFF);  // 32-byte aligned
    const VT* ybase = DOT ? reinterpret_cast<const VT*>(yr + e0 - MOFF) : nullptr;
    const bool whole = rem >= kChains * V;
#if TFB_CLS_ALL
    // all five windows first (more loads in flight), then both halves
    VT za[10], zb[10];
#pragma unroll
    for (int wi = 0; wi < 5; ++wi) {
      const int64_t first = int64_t(wi) * W - MOFF;
      if ((wi < 4 || MOFF > 0) && first < rem) {
        ld_stream32(base + 2 * wi, za[2 * wi], za[2 * wi + 1]);
        if constexpr (DOT) ld_stream32(ybase + 2 * wi, zb[2 * wi], zb[2 * wi + 1]);
      } else {
        za[2 * wi] = za[2 * wi + 1] = VT{};
        if constexpr (DOT) zb[2 * wi] = zb[2 * wi + 1] = VT{};
      }
    }
    T ga[5 * W], gb[5 * W];
#pragma unroll
    for (int v = 0; v < 10; ++v)
#pragma unroll
      for (int q = 0; q < V; ++q) {
        ga[v * V + q] = vget(za[v], q);
        if constexpr (DOT) gb[v * V + q] = vget(zb[v], q);
      }
#pragma unroll
    for (int c = 0; c < kChains; ++c)
#pragma unroll
      for (int q = 0; q < V; ++q) {
        if (!whole && int64_t(c) * V + q >= rem) continue;
        if constexpr (DOT) accumulate<M, T, true>(ch[c], ga[MOFF + c * V + q], gb[MOFF + c * V + q]);
        else accumulate<M, T, false>(ch[c], ga[MOFF + c * V + q], T(0));
      }
    (void)j;
    continue;
#endif
    VT wa[6], wb[6];  // windows 2..4 of the previous half are reused: 0,1,2 | 2,3,4
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!whole && int64_t(4 * h) * V >= rem) break;
#pragma unroll
      for (int w = (h == 0 ? 0 : 1); w < 3; ++w) {  // window index within the half: 2h + w
        const int wi = 2 * h + w;
        const int64_t first = int64_t(wi) * W - MOFF;  // block-relative element of the window's start
        const bool need = (wi < 4 || MOFF > 0) && first < rem;
        if (need) {
          ld_stream32(base + 2 * wi, wa[2 * w], wa[2 * w + 1]);
          if constexpr (DOT) ld_stream32(ybase + 2 * wi, wb[2 * w], wb[2 * w + 1]);
        } else {
          wa[2 * w] = wa[2 * w + 1] = VT{};
          if constexpr (DOT) wb[2 * w] = wb[2 * w + 1] = VT{};
        }
      }
      T fa[3 * W], fb[3 * W];
#pragma unroll
      for (int v = 0; v < 6; ++v)
#pragma unroll
        for (int q = 0; q < V; ++q) {
          fa[v * V + q] = vget(wa[v], q);
          if constexpr (DOT) fb[v * V + q] = vget(wb[v], q);
        }
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int q = 0; q < V; ++q) {
          if (!whole && int64_t(4 * h + c) * V + q >= rem) continue;
          if constexpr (DOT) accumulate<M, T, true>(ch[4 * h + c], fa[MOFF + c * V + q], fb[MOFF + c * V + q]);
          else accumulate<M, T, false>(ch[4 * h + c], fa[MOFF + c * V + q], T(0));
        }
      // window 2 of this half is window 0 of the next
      wa[0] = wa[4];
      wa[1] = wa[5];
      if constexpr (DOT) {
        wb[0] = wb[4];
        wb[1] = wb[5];
      }
    }
  }
}

template <int M, typename T, bool DOT>
__global__ void TFB_RS_BOUNDS rows_cls_kernel(
    const T* __restrict__ x, const T* __restrict__ y, int64_t ldx, int64_t ldy, int64_t rows, int64_t cols,
    int K, int g_log2, int period, Pair<typename Acc<M, T>::type>* __restrict__ out, int chain) {
  using A = typename Acc<M, T>::type;
  constexpr int kChains = 8;
  constexpr int W = 32 / sizeof(T);
  const int lane = threadIdx.x & 31;
  const int G = 1 << g_log2;
  const int j = lane & (G - 1);
  const int64_t groups = 32 >> g_log2;
  const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  if (chain >= 0) {
    // the warp's first rows are `period` apart: one request per row, by the row group's first lane
    const int64_t rf = (warp / period) * period * groups + warp % period + int64_t(period) * (lane >> g_log2);
    if (chain > 0 && j == 0 && rf < rows) {
      const int cap = chain / static_cast<int>(groups) > 16 ? chain / static_cast<int>(groups) : 16;
      prefetch_span(x + rf * ldx, cols * static_cast<int64_t>(sizeof(T)), cap);
      if constexpr (DOT) prefetch_span(y + rf * ldy, cols * static_cast<int64_t>(sizeof(T)), cap);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  // slot s = (super-block s / p, class s % p); the warp's rows: q + p*i of the block
  for (int64_t s = warp;; s += nwarps) {  // warp-uniform
    const int64_t sb = s / period, q = s % period;
    const int64_t rfirst = sb * period * groups + q;
    if (sb * period * groups >= rows) break;
    const int64_t r = rfirst + int64_t(period) * (lane >> g_log2);
    const int moff = static_cast<int>((reinterpret_cast<uintptr_t>(x + rfirst * ldx) & 31u) / sizeof(T));
    Pair<A> ch[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) ch[c] = zero_pair<A>();
    if (r < rows) {
      const T* xr = x + r * ldx;
      const T* yr = DOT ? y + r * ldy : nullptr;
      // the warp's rows share one 32-byte offset class (x and y alike): the premise of
      // the compile-time picks (debug builds assert it)
      TFB_CHECK(static_cast<int>((reinterpret_cast<uintptr_t>(xr) & 31u) / sizeof(T)) == moff);
      TFB_CHECK(!DOT || static_cast<int>((reinterpret_cast<uintptr_t>(yr) & 31u) / sizeof(T)) == moff);
      switch (moff) {  // warp-uniform
#define TFB_CLS_CASE(O) \
  case O:               \
    if constexpr (O < W) cls_rows_chains<M, T, DOT, O>(ch, xr, yr, cols, K, j); \
    break;
        TFB_CLS_CASE(0) TFB_CLS_CASE(1) TFB_CLS_CASE(2) TFB_CLS_CASE(3)
        TFB_CLS_CASE(4) TFB_CLS_CASE(5) TFB_CLS_CASE(6) TFB_CLS_CASE(7)
#undef TFB_CLS_CASE
        default: break;
      }
    }
#pragma unroll
    for (int w = 1; w < kChains; w <<= 1)
#pragma unroll
      for (int c = 0; c < kChains; c += 2 * w) ch[c] = merge<M, A>(ch[c], ch[c + w]);
    Pair<A> st = ch[0];
    for (int off = 1; off < G; off <<= 1) {
      Pair<A> o;
      o.s = __shfl_down_sync(0xffffffffu, st.s, off, G);
      if constexpr (HasErr<M>::value) o.e = __shfl_down_sync(0xffffffffu, st.e, off, G);
      else o.e = A(0);
      if ((j & (2 * off - 1)) == 0) st = merge<M, A>(st, o);
    }
    if (j == 0 && r < rows) {
      for (int lv = 3 + g_log2; lv < 8; ++lv) st = merge<M, A>(st, zero_pair<A>());
      out[r] = st;
    }
  }
}

// Lanes per row: pow2ceil(ceil(chains holding data / 8)), chains = min(256, ceil(cols / V)).
inline int rows_short_glog2(int64_t cols, int V) {
  int64_t chains = (cols + V - 1) / V;
  if (chains > kThreads) chains = kThreads;
  const int64_t lanes = (chains + 7) / 8;
  int g = 0;
  while ((int64_t(1) << g) < lanes) ++g;
  return g;
}

}  // namespace tfb
