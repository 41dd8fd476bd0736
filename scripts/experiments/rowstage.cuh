// rowstage.cuh — short rows staged through shared memory (cp.async ring per warp).
// Included by reduce.cu after rows.cuh.
//
// rows_short_kernel is latency-bound: a lane's loads of the next rows are not
// issued before the current rows' chains and tree are done, and its register
// budget leaves three CTAs per SM.  Here every warp keeps a ring of kRsStages row
// groups in flight with cp.async (16-byte chunks, coalesced per row: lane j of a
// row's group copies chunks j, j + G, ...), and the lanes then read their lane
// blocks from shared memory.  Same chains (lane j of the group owns chains
// 8j..8j+7), same order, same tree as rows_short_kernel — bit-identical.
// Layout: a lane block (8 chunks = 128 bytes) is stored at a pitch of 144 bytes,
// so the eight lanes of a quarter-warp hit eight different 16-byte bank groups
// both when the copies land and when LDS.128 reads them back.
// Scope: 16-byte aligned rows (base and pitch) that fit one leaf; a row of several
// k-rows (256 chunks each) takes a whole warp, one k-row per ring stage.

namespace tfb {

#ifndef TFB_RS_STAGES
#define TFB_RS_STAGES 3
#endif
#ifndef TFB_RS_THREADS
#define TFB_RS_THREADS 256
#endif
constexpr int kRsStages = TFB_RS_STAGES;
constexpr int kRsPitch = 144;                      // bytes per lane block in shared memory
// bytes per warp, stage and operand: 32 lane blocks + one extra chunk per row of the warp
__host__ __device__ constexpr int rs_warp_stage(int g_log2) { return 32 * kRsPitch + (32 >> g_log2) * 16; }
constexpr int kRsThreads = TFB_RS_THREADS;

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, int src_bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gsrc), "r"(src_bytes) : "memory");
}

template <typename T>
__device__ __forceinline__ typename Vec<T>::type lds_vec(const unsigned char* p);
template <>
__device__ __forceinline__ float4 lds_vec<float>(const unsigned char* p) {
  return *reinterpret_cast<const float4*>(p);
}
template <>
__device__ __forceinline__ double2 lds_vec<double>(const unsigned char* p) {
  return *reinterpret_cast<const double2*>(p);
}

// Element i of a run read from `m` elements before the wanted start (m < V, uniform per
// row): one select level per bit of m, the picks themselves are compile-time indices.
template <typename T, int N>
__device__ __forceinline__ void shift_run(const T (&f)[N + Vec<T>::V], int m, T (&out)[N]) {
  if constexpr (Vec<T>::V == 2) {
#pragma unroll
    for (int i = 0; i < N; ++i) out[i] = m ? f[i + 1] : f[i];
  } else {
    T t[N + 2];
#pragma unroll
    for (int i = 0; i < N + 2; ++i) t[i] = (m & 1) ? f[i + 1] : f[i];
#pragma unroll
    for (int i = 0; i < N; ++i) out[i] = (m & 2) ? t[i + 2] : t[i];
  }
}

// MULTI: rows of several k-rows (G = 32, one row per warp iteration, a ring stage per
// k-row, the chain states carried from k-row to k-row); otherwise K = 1.
// MIS: rows that are not 16-byte aligned (any base, any pitch, x and y independently):
// the ring receives the aligned 16-byte chunks around each k-row (every chunk read holds
// an element of the row), a lane reads the nine chunks around its block and shifts the
// run by the row's offset.
template <int M, typename T, bool DOT, bool MULTI, bool MIS>
__global__ void __launch_bounds__(kRsThreads) rows_stage_kernel(
    const T* __restrict__ x, const T* __restrict__ y, int64_t ldx, int64_t ldy, int64_t rows, int64_t cols,
    int g_log2, Pair<typename Acc<M, T>::type>* __restrict__ out) {
  using A = typename Acc<M, T>::type;
  using VT = typename Vec<T>::type;
  constexpr int V = Vec<T>::V;
  constexpr int kChains = 8;
  constexpr int kOps = DOT ? 2 : 1;
  constexpr int kRowChunk = kThreads * 16;  // bytes of a k-row
  extern __shared__ __align__(128) unsigned char rs_smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int G = MULTI ? 32 : (1 << g_log2);
  const int glog = MULTI ? 5 : g_log2;
  const int j = lane & (G - 1);
  const int grp = lane >> glog;
  const int groups = 32 >> glog;
  const int row_pitch = G * kRsPitch + 16;  // a row's lane blocks + the chunk after the last one (MIS)
  const int kRsWarpStage = rs_warp_stage(glog);
  const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  unsigned char* wbase = rs_smem + static_cast<size_t>(wib) * kRsStages * kOps * kRsWarpStage;
  const int64_t row_bytes = cols * static_cast<int64_t>(sizeof(T));
  const int K = MULTI ? static_cast<int>((row_bytes + kRowChunk - 1) / kRowChunk) : 1;
  // only the last k-row can end in a partial lane block: then every lane runs the
  // predicated chain steps (a warp-uniform choice; a per-lane one would diverge)
  const bool ragged = (cols % (kChains * V)) != 0;
  const int64_t my_iters = [&] {  // row groups of this warp (warp-uniform)
    const int64_t total = (rows + groups - 1) / groups;
    return warp < total ? (total - warp + nwarps - 1) / nwarps : 0;
  }();
  const int64_t row_step = nwarps * groups;

  // one operand's chunks of k-row k of a row starting at g (bytes) into the row's region sb
  auto copy_op = [&](unsigned char* sb, const unsigned char* g, int k) {
    const unsigned char* seg = g + int64_t(k) * kRowChunk;
    const int64_t left_row = row_bytes - int64_t(k) * kRowChunk;  // bytes of the row from this k-row on
    const int64_t seg_bytes = left_row >= kRowChunk ? kRowChunk : left_row;
    if constexpr (MIS) {
      const int mb = static_cast<int>(reinterpret_cast<uintptr_t>(seg) & 15u);
      const int nq = static_cast<int>((mb + seg_bytes + 15) >> 4);  // <= 257
      const unsigned char* base = seg - mb;
      for (int q = j; q < nq; q += G) cp_async16(sb + (q >> 3) * kRsPitch + (q & 7) * 16, base + int64_t(q) * 16, 16);
    } else {
      const int nq = static_cast<int>((seg_bytes + 15) >> 4);
      for (int q = j; q < nq; q += G) {
        const int64_t left = seg_bytes - int64_t(q) * 16;
        const int nb = left < 16 ? static_cast<int>(left) : 16;  // the row's last chunk may be partial: zero-filled
        cp_async16(sb + (q >> 3) * kRsPitch + (q & 7) * 16, seg + int64_t(q) * 16, nb);
      }
    }
  };
  // copies of k-row k of row r (this lane's row of the group) into `stage`; always one commit group
  auto issue = [&](int64_t r, int k, int stage) {
    if (r < rows) {
      unsigned char* sb = wbase + static_cast<size_t>(stage) * kOps * kRsWarpStage + grp * row_pitch;
      copy_op(sb, reinterpret_cast<const unsigned char*>(x + r * ldx), k);
      if constexpr (DOT) copy_op(sb + kRsWarpStage, reinterpret_cast<const unsigned char*>(y + r * ldy), k);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  // producer cursor (row, k-row, stage) runs kRsStages - 1 units ahead of the consumer's
  int64_t pr = warp * groups + grp, pit = 0;
  int pk = 0, pstage = 0;
  auto produce = [&]() {
    if (pit < my_iters) {
      issue(pr, pk, pstage);
      if (++pk == K) {
        pk = 0;
        ++pit;
        pr += row_step;
      }
    } else {
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    if (++pstage == kRsStages) pstage = 0;
  };
#pragma unroll
  for (int s = 0; s < kRsStages - 1; ++s) produce();

  int cstage = 0;
  int64_t r = warp * groups + grp;
  for (int64_t it = 0; it < my_iters; ++it, r += row_step) {
    Pair<A> ch[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) ch[c] = zero_pair<A>();
    // the row's offsets past a 16-byte boundary (elements); every k-row starts at the same one
    const int mx = MIS && r < rows ? static_cast<int>((reinterpret_cast<uintptr_t>(x + r * ldx) & 15u) / sizeof(T)) : 0;
    const int my = MIS && DOT && r < rows ? static_cast<int>((reinterpret_cast<uintptr_t>(y + r * ldy) & 15u) / sizeof(T)) : 0;
    for (int k = 0; k < K; ++k) {
      produce();
      asm volatile("cp.async.wait_group %0;" ::"n"(kRsStages - 1) : "memory");
      __syncwarp();
      const int64_t e0 = (int64_t(k) * kThreads + kChains * j) * V;  // this lane's block: elements [e0, e0 + 8V)
      if (r < rows && e0 < cols) {
        const unsigned char* sb = wbase + static_cast<size_t>(cstage) * kOps * kRsWarpStage + grp * row_pitch + j * kRsPitch;
        T ea[kChains * V], eb[kChains * V];
        if constexpr (MIS) {
          T fa[(kChains + 1) * V], fb[(kChains + 1) * V];
#pragma unroll
          for (int c = 0; c <= kChains; ++c) {
            const VT va = lds_vec<T>(sb + (c < kChains ? 16 * c : kRsPitch));
#pragma unroll
            for (int q = 0; q < V; ++q) fa[c * V + q] = vget(va, q);
            if constexpr (DOT) {
              const VT vb = lds_vec<T>(sb + kRsWarpStage + (c < kChains ? 16 * c : kRsPitch));
#pragma unroll
              for (int q = 0; q < V; ++q) fb[c * V + q] = vget(vb, q);
            }
          }
          shift_run<T, kChains * V>(fa, mx, ea);
          if constexpr (DOT) shift_run<T, kChains * V>(fb, my, eb);
        } else {
#pragma unroll
          for (int c = 0; c < kChains; ++c) {
            const VT va = lds_vec<T>(sb + 16 * c);
#pragma unroll
            for (int q = 0; q < V; ++q) ea[c * V + q] = vget(va, q);
            if constexpr (DOT) {
              const VT vb = lds_vec<T>(sb + kRsWarpStage + 16 * c);
#pragma unroll
              for (int q = 0; q < V; ++q) eb[c * V + q] = vget(vb, q);
            }
          }
        }
        if (!ragged || k + 1 < K) {
#pragma unroll
          for (int c = 0; c < kChains; ++c)
#pragma unroll
            for (int q = 0; q < V; ++q) {
              if constexpr (DOT) accumulate<M, T, true>(ch[c], ea[c * V + q], eb[c * V + q]);
              else accumulate<M, T, false>(ch[c], ea[c * V + q], T(0));
            }
        } else {
          const int rem = cols - e0 < kChains * V ? static_cast<int>(cols - e0) : kChains * V;
#pragma unroll
          for (int c = 0; c < kChains; ++c)
#pragma unroll
            for (int q = 0; q < V; ++q)
              if (c * V + q < rem) {
                if constexpr (DOT) accumulate<M, T, true>(ch[c], ea[c * V + q], eb[c * V + q]);
                else accumulate<M, T, false>(ch[c], ea[c * V + q], T(0));
              }
        }
      }
      __syncwarp();  // the stage may be refilled by the next unit's copies
      if (++cstage == kRsStages) cstage = 0;
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
      for (int lv = 3 + glog; lv < 8; ++lv) st = merge<M, A>(st, zero_pair<A>());
      out[r] = st;
    }
  }
}

}  // namespace tfb
