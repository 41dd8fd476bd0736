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

template <int M, typename T, bool DOT, bool VEC>
__global__ void __launch_bounds__(kThreads) rows_short_kernel(
    const T* __restrict__ x, const T* __restrict__ y, int64_t ldx, int64_t ldy, int64_t rows, int64_t cols,
    int K, int g_log2, Pair<typename Acc<M, T>::type>* __restrict__ out) {
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
        if (VEC && e0 + kChains * V <= cols) {
          TFB_CHECK((reinterpret_cast<uintptr_t>(xr + e0) & 15u) == 0);
          const VT* xv = reinterpret_cast<const VT*>(xr + e0);
          const VT* yv = DOT ? reinterpret_cast<const VT*>(yr + e0) : nullptr;
#pragma unroll
          for (int h = 0; h < 2; ++h) {  // two halves of 4 vectors: loads first, then the chains
            VT a[4], b[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              a[c] = ld_stream(xv + 4 * h + c);
              if constexpr (DOT) b[c] = ld_stream(yv + 4 * h + c);
            }
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
              for (int q = 0; q < V; ++q) {
                if constexpr (DOT) accumulate<M, T, true>(ch[4 * h + c], vget(a[c], q), vget(b[c], q));
                else accumulate<M, T, false>(ch[4 * h + c], vget(a[c], q), T(0));
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
