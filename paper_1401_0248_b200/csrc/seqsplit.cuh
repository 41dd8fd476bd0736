// seqsplit.cuh — the seq flavor (kernels.py:127-170, :186-230) with its two
// dependency chains decoupled.  Included by reduce.cu after seqpipe.cuh.
//
// The reference's sequential twofold recurrence carries two running values:
//   s_i = fl(s_{i-1} + y_i)                         (every method)
//   fast:      c_i = fl(fl(s_i - s_{i-1}) - y_i),   e_i = fl(e_{i-1} - c_i)
//   rigorous:  yt = fl(s_i - s_{i-1}), dy = fl(y_i - yt),
//              ds = fl(s_{i-1} - fl(s_i - yt)),    e_i = fl(e_{i-1} + fl(ds + dy))
// Only s and e are loop-carried; c_i / (ds + dy) depend on s_{i-1}, s_i, y_i
// alone, and the dot addends y_i = fl(a_i b_i) on nothing.  One thread running
// all of it is issue-bound (~9 instructions per element).  Here:
//   * a producer lane streams the input into a ring of shared-memory stages
//     (cp.async.bulk, as seqpipe.cuh);
//   * helper warps form the addends (dots) and, once the s-chain has filled a
//     stage's s_i, the per-element corrections c_i / d_i, in parallel;
//   * the s-chain lane runs s_i = s_{i-1} + y_i alone (one FP add per element on
//     the critical path, loads and stores off it);
//   * the e-chain lane runs e_i = e_{i-1} -/+ c_i in element order.
// Every value is produced by the same IEEE operation on the same operands as in
// the reference, and s and e are accumulated in the reference's order, so the
// pair is bit-identical to seq_pipe_kernel / the reference seq flavor (tested).
// Stages hand over through mbarriers: full (TMA) -> y ready (dots) -> s ready ->
// c ready -> empty.  The unaligned head and the tail after the last whole stage
// run the full recurrence on the combined state.  Direct and wide have no e
// chain; Kahan (a four-add loop-carried chain) and TwoProduct dots keep
// seq_pipe_kernel.

namespace tfb {

constexpr int kSplitStages = 4;
constexpr int kSplitChunkBytes = 8192;  // per operand per stage
constexpr int kSplitWarps = 12;         // 0: s-chain, 1: e-chain, 5: producer, 2,3,6,7,10,11: helpers
constexpr int kSplitThreads = kSplitWarps * 32;
constexpr int kSplitHelperWarps = 6;
constexpr int kSplitHelpers = kSplitHelperWarps * 32;

__device__ __forceinline__ int split_helper_index(int warp) {
  // helpers sit on the schedulers (warp % 4) the two chain lanes do not use
  switch (warp) {
    case 2: return 0;
    case 3: return 1;
    case 6: return 2;
    case 7: return 3;
    case 10: return 4;
    case 11: return 5;
    default: return -1;
  }
}

// mbarrier wait that backs off (the producer / helpers must not steal issue slots
// from the two chain lanes while they wait)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  for (;;) {
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(200);
  }
}

// acc = acc OP src[i] for i = 0..count-1 in order (OP: +, or - when SUB), storing
// every running value to dst when STORE.  Blocks of 8 16-byte vectors, double
// buffered in registers (the next block's shared-memory loads are in flight while
// this block's adds run; no register copies), so only the FP add's latency is on
// the chain.  count is a multiple of 2 * 8 vectors (the stage size).
template <bool SUB, bool STORE, typename A, int B = 8>
__device__ __forceinline__ void chain_block(A& acc, const typename Vec<A>::type (&in)[B], A* __restrict__ dst) {
  using VA = typename Vec<A>::type;
  constexpr int W = Vec<A>::V;
  VA* dv = reinterpret_cast<VA*>(dst);
#pragma unroll
  for (int p = 0; p < B; ++p) {
    A r[W];
#pragma unroll
    for (int q = 0; q < W; ++q) {
      acc = SUB ? Ar<A>::sub(acc, vget(in[p], q)) : Ar<A>::add(acc, vget(in[p], q));
      r[q] = acc;
    }
    if constexpr (STORE) {
      if constexpr (W == 4) dv[p] = make_float4(r[0], r[1], r[2], r[3]);
      else dv[p] = make_double2(r[0], r[1]);
    }
  }
}

template <bool SUB, bool STORE, typename A>
__device__ __forceinline__ A run_chain(A acc, const A* __restrict__ src, A* __restrict__ dst, int count) {
  using VA = typename Vec<A>::type;
  constexpr int W = Vec<A>::V;
  constexpr int B = 8;
  const VA* sv = reinterpret_cast<const VA*>(src);
  const int nb = count / (W * B);
  VA a[B], b[B];
#pragma unroll
  for (int p = 0; p < B; ++p) a[p] = sv[p];
  for (int k = 0; k < nb; k += 2) {
#pragma unroll
    for (int p = 0; p < B; ++p) b[p] = sv[(k + 1) * B + p];
    chain_block<SUB, STORE, A, B>(acc, a, dst + k * B * W);
    if (k + 2 < nb) {
#pragma unroll
      for (int p = 0; p < B; ++p) a[p] = sv[(k + 2) * B + p];
    }
    chain_block<SUB, STORE, A, B>(acc, b, dst + (k + 1) * B * W);
  }
  return acc;
}

template <int M, typename T, bool DOT>
struct SplitSmem {
  using A = typename Acc<M, T>::type;
  static constexpr int CE = kSplitChunkBytes / static_cast<int>(sizeof(T));
  static constexpr size_t kIn = size_t(kSplitChunkBytes) * (DOT ? 2 : 1);  // x (+ y)
  static constexpr size_t kY = (DOT || sizeof(A) != sizeof(T)) ? sizeof(A) * CE : 0;  // addends
  static constexpr bool kErr = (Base<M>::value == kFast || Base<M>::value == kRigorous);
  static constexpr size_t kS = kErr ? sizeof(A) * CE : 0;  // s_i, for the corrections
  static constexpr size_t kC = kErr ? sizeof(A) * CE : 0;  // c_i / d_i
  static constexpr size_t kStage = kIn + kY + kS + kC;
  static constexpr size_t kBytes = kSplitStages * kStage + 5 * kSplitStages * 8 + 64;
};

template <int M, typename T, bool DOT>
__global__ void __launch_bounds__(kSplitThreads) seq_split_kernel(const T* __restrict__ x, const T* __restrict__ y,
                                                                  int64_t n, int64_t head, int64_t nchunks,
                                                                  Pair<typename Acc<M, T>::type>* __restrict__ out) {
  using A = typename Acc<M, T>::type;
  using SM = SplitSmem<M, T, DOT>;
  constexpr int CE = SM::CE;
  constexpr bool kErr = (Base<M>::value == kFast || Base<M>::value == kRigorous);
  constexpr bool kYbuf = SM::kY > 0;
  extern __shared__ __align__(128) unsigned char split_smem[];
  auto stage_base = [&](int slot) { return split_smem + size_t(slot) * SM::kStage; };
  uint64_t* bars = reinterpret_cast<uint64_t*>(split_smem + kSplitStages * SM::kStage);
  uint64_t* full = bars;
  uint64_t* yrdy = bars + kSplitStages;
  uint64_t* srdy = bars + 2 * kSplitStages;
  uint64_t* crdy = bars + 3 * kSplitStages;
  uint64_t* empty = bars + 4 * kSplitStages;
  __shared__ A s_before[kSplitStages];  // s entering each stage (s_{i-1} of its first element)
  __shared__ Pair<A> hand;              // head state in; chunk-end s out
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSplitStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&yrdy[i], kSplitHelpers);
      mbar_init(&srdy[i], 1);
      mbar_init(&crdy[i], kSplitHelpers);
      mbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the unaligned head, full recurrence, one thread (a few elements)
    Pair<A> st = zero_pair<A>();
    for (int64_t e = 0; e < head && e < n; ++e) accumulate<M, T, DOT>(st, x[e], DOT ? y[e] : T(0));
    hand = st;
  }
  __syncthreads();

  auto xs = [&](int slot) { return reinterpret_cast<T*>(stage_base(slot)); };
  auto ys = [&](int slot) { return reinterpret_cast<T*>(stage_base(slot) + kSplitChunkBytes); };
  auto yb = [&](int slot) { return reinterpret_cast<A*>(stage_base(slot) + SM::kIn); };
  auto sb = [&](int slot) { return reinterpret_cast<A*>(stage_base(slot) + SM::kIn + SM::kY); };
  auto cb = [&](int slot) { return reinterpret_cast<A*>(stage_base(slot) + SM::kIn + SM::kY + SM::kS); };

  if (warp == 5) {  // ---------------- producer (scheduler 1, sleeping waits) ----------------
    if (lane != 0) return;
    for (int64_t c = 0; c < nchunks; ++c) {
      const int slot = static_cast<int>(c % kSplitStages);
      const uint32_t phase = static_cast<uint32_t>((c / kSplitStages) & 1);
      mbar_wait_sleep(&empty[slot], phase ^ 1u);
      mbar_arrive_expect_tx(&full[slot], kSplitChunkBytes * (DOT ? 2u : 1u));
      bulk_g2s(xs(slot), x + head + c * CE, kSplitChunkBytes, &full[slot]);
      if constexpr (DOT) bulk_g2s(ys(slot), y + head + c * CE, kSplitChunkBytes, &full[slot]);
    }
    return;
  }

  const int h = split_helper_index(warp);
  if (h >= 0) {  // ---------------- helpers ----------------
    // iteration c: the addends of stage c (so the s-chain finds them ready when it
    // arrives there), then the corrections of stage c-1 (whose s_i it just wrote)
    const int t = h * 32 + lane;
    for (int64_t c = 0; c <= nchunks; ++c) {
      if (kYbuf && c < nchunks) {  // addends: fl(a*b) in the data type (widened exactly for wide)
        const int slot = static_cast<int>(c % kSplitStages);
        mbar_wait_sleep(&full[slot], static_cast<uint32_t>((c / kSplitStages) & 1));
        const T* cx = xs(slot);
        const T* cy = ys(slot);
        A* cyb = yb(slot);
        for (int i = t; i < CE; i += kSplitHelpers) cyb[i] = addend<M, T, DOT>(cx[i], DOT ? cy[i] : T(0));
        mbar_arrive(&yrdy[slot]);
      }
      if (kErr && c >= 1) {  // per-element corrections of stage c-1
        const int64_t cp = c - 1;
        const int slot = static_cast<int>(cp % kSplitStages);
        mbar_wait_sleep(&srdy[slot], static_cast<uint32_t>((cp / kSplitStages) & 1));
        const A* cs = sb(slot);
        const A* cya = kYbuf ? yb(slot) : nullptr;
        const T* cx = xs(slot);
        A* cc = cb(slot);
        const A s0 = s_before[slot];
        for (int i = t; i < CE; i += kSplitHelpers) {
          const A sp = i == 0 ? s0 : cs[i - 1];
          const A sn = cs[i];
          const A yy = kYbuf ? cya[i] : static_cast<A>(cx[i]);
          using R = Ar<A>;
          if constexpr (Base<M>::value == kFast) {
            cc[i] = R::sub(R::sub(sn, sp), yy);  // c = (t - s) - y      (kernels.py:151)
          } else {
            const A yt = R::sub(sn, sp);         // yt = t - s           (kernels.py:164-167)
            const A dy = R::sub(yy, yt);
            const A ds = R::sub(sp, R::sub(sn, yt));
            cc[i] = R::add(ds, dy);
          }
        }
        mbar_arrive(&crdy[slot]);
      }
    }
    return;
  }
  if (warp > 1) return;  // idle warps (4, 8, 9)

  if (warp == 0 && lane == 0) {  // ---------------- s-chain ----------------
    using R = Ar<A>;
    A s = hand.s;
    for (int64_t c = 0; c < nchunks; ++c) {
      const int slot = static_cast<int>(c % kSplitStages);
      const uint32_t phase = static_cast<uint32_t>((c / kSplitStages) & 1);
      if constexpr (kYbuf) mbar_wait(&yrdy[slot], phase);
      else mbar_wait(&full[slot], phase);
      s_before[slot] = s;
      const A* src = kYbuf ? yb(slot) : reinterpret_cast<const A*>(xs(slot));  // !kYbuf: A == T
      s = run_chain<false, kErr>(s, src, sb(slot), CE);
      mbar_arrive(&srdy[slot]);
    }
    hand.s = s;  // read by the e-chain lane after its last stage (ordered by the barrier below)
  } else if (warp == 1 && lane == 0) {  // ---------------- e-chain ----------------
    using R = Ar<A>;
    A e = hand.e;
    for (int64_t c = 0; c < nchunks; ++c) {
      const int slot = static_cast<int>(c % kSplitStages);
      const uint32_t phase = static_cast<uint32_t>((c / kSplitStages) & 1);
      if constexpr (kErr) {
        mbar_wait(&crdy[slot], phase);
        // fast: e = e - c (kernels.py:152); rigorous: e = e + (ds + dy) (:168)
        e = run_chain<Base<M>::value == kFast, false>(e, cb(slot), static_cast<A*>(nullptr), CE);
      } else {
        mbar_wait(&srdy[slot], phase);  // direct / wide: nothing to accumulate, just free the stage
      }
      mbar_arrive(&empty[slot]);
    }
    hand.e = e;
  }
  // both chains done: the tail after the last whole stage, full recurrence, one thread
  asm volatile("bar.sync 1, 64;" ::: "memory");  // warps 0 and 1 only
  if (threadIdx.x == 0) {
    Pair<A> st{hand.s, hand.e};
    for (int64_t e = head + nchunks * CE; e < n; ++e) accumulate<M, T, DOT>(st, x[e], DOT ? y[e] : T(0));
    out[0] = st;
  }
}

}  // namespace tfb
