// eft.cuh — device error-free transforms, per-element recurrences and pair
// merges for the five methods of arXiv 1401.0248.
//
// Every operation is an explicit round-to-nearest intrinsic (__fadd_rn,
// __dsub_rn, ...): ptxas never contracts an intrinsic pair into FFMA/DFMA,
// never reassociates, and the library is also built with -fmad=false
// -ftz=false as a second guard (tests/test_sass.py greps the SASS).
//
// Reference formulas (pkg/src/twofold):
//   fast_two_sum  eft.py:39-42        two_sum  eft.py:51-56
//   direct step   kernels.py:131      wide step kernels.py:139, :198-199
//   tf step       kernels.py:149-153  tr step   kernels.py:163-169
//   kahan step    kernels.py:179-182  dot addend y = fl(a*b) kernels.py:209, :239
//   twofold merge kernels.py:310-317  kahan merge kernels.py:379-390
//   direct merge  kernels.py:267-269
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// Debug builds (-DTFB_DEBUG=1, scripts/build_debug.sh) assert every global
// access range and scratch capacity on the device (compute-sanitizer is not
// available on the GPU pool; this is the substitute).
#ifndef TFB_DEBUG
#define TFB_DEBUG 0
#endif
#if TFB_DEBUG
#include <cassert>
#define TFB_CHECK(cond) assert(cond)
#else
#define TFB_CHECK(cond) ((void)0)
#endif

namespace tfb {

enum Method : int {
  kDirect = 0, kWide = 1, kFast = 2, kRigorous = 3, kKahan = 4,
  // opt-in TwoProduct dots (not in the reference, which
  // rounds every product, kernels.py:23-26): the product's exact round-off
  // fma(a, b, -fl(a*b)) is added to the error channel.
  kFastTP = 5, kRigorousTP = 6
};

// The summation recurrence a method uses (TP variants sum like their base).
template <int M> struct Base { static constexpr int value = M; };
template <> struct Base<kFastTP> { static constexpr int value = kFast; };
template <> struct Base<kRigorousTP> { static constexpr int value = kRigorous; };
template <int M> __host__ __device__ constexpr bool is_tp() { return M == kFastTP || M == kRigorousTP; }

template <typename T> struct Ar;
#if TFB_PLAIN_OPS
// NEGATIVE CONTROL ONLY (canary.cu built into libtfb_canary_unsafe.so): plain
// operators the compiler is free to contract into FMAs under --use_fast_math.
// The product library never defines TFB_PLAIN_OPS (tests/test_sass.py).
template <> struct Ar<float> {
  static __device__ __forceinline__ float add(float a, float b) { return a + b; }
  static __device__ __forceinline__ float sub(float a, float b) { return a - b; }
  static __device__ __forceinline__ float mul(float a, float b) { return a * b; }
  static __device__ __forceinline__ float fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
};
template <> struct Ar<double> {
  static __device__ __forceinline__ double add(double a, double b) { return a + b; }
  static __device__ __forceinline__ double sub(double a, double b) { return a - b; }
  static __device__ __forceinline__ double mul(double a, double b) { return a * b; }
  static __device__ __forceinline__ double fma(double a, double b, double c) { return __fma_rn(a, b, c); }
};
#else
template <> struct Ar<float> {
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
};
template <> struct Ar<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double fma(double a, double b, double c) { return __fma_rn(a, b, c); }
};
#endif

// (value, error) state.  For KAHAN, `e` holds the pending correction c.
template <typename A> struct Pair { A s, e; };

// Accumulator type: the data type, except WIDE (binary32 data, binary64 sum).
template <int M, typename T> struct Acc { using type = T; };
template <> struct Acc<kWide, float> { using type = double; };

// The addend the recurrence sees: x, or the product rounded in the DATA type
// (kernels.py:198 for wide, :209 otherwise), then widened exactly for WIDE.
template <int M, typename T, bool DOT>
__device__ __forceinline__ typename Acc<M, T>::type addend(T a, T b) {
  using A = typename Acc<M, T>::type;
  if constexpr (DOT) return static_cast<A>(Ar<T>::mul(a, b));
  else return static_cast<A>(a);
}

// One element of the sequential recurrence.
template <int M0, typename A>
__device__ __forceinline__ void step(Pair<A>& st, A y) {
  using R = Ar<A>;
  constexpr int M = Base<M0>::value;
  if constexpr (M == kDirect || M == kWide) {
    st.s = R::add(st.s, y);
  } else if constexpr (M == kFast) {
    A t = R::add(st.s, y);
    A c = R::sub(R::sub(t, st.s), y);
    st.e = R::sub(st.e, c);
    st.s = t;
  } else if constexpr (M == kRigorous) {
    A t = R::add(st.s, y);
    A yt = R::sub(t, st.s);
    A dy = R::sub(y, yt);
    A ds = R::sub(st.s, R::sub(t, yt));
    st.e = R::add(st.e, R::add(ds, dy));
    st.s = t;
  } else {  // kKahan: y' = y - c; t = s + y'; c = (t - s) - y'; s = t
    A yy = R::sub(y, st.e);
    A t = R::add(st.s, yy);
    st.e = R::sub(R::sub(t, st.s), yy);
    st.s = t;
  }
}

// Merge right state R into left state L (order matters for the error fold).
template <int M0, typename A>
__device__ __forceinline__ Pair<A> merge(Pair<A> L, Pair<A> Rt) {
  using R = Ar<A>;
  constexpr int M = Base<M0>::value;
  if constexpr (M == kDirect || M == kWide) {
    L.s = R::add(L.s, Rt.s);
  } else if constexpr (M == kFast || M == kRigorous) {
    // two_sum(L.s, Rt.s) with the round-off and Rt.e folded into L.e:
    // e = (e + ((s - sv) + (v - bv))) + e_j      (kernels.py:313-317)
    A x = R::add(L.s, Rt.s);
    A bv = R::sub(x, L.s);
    A sv = R::sub(x, bv);
    L.e = R::add(R::add(L.e, R::add(R::sub(L.s, sv), R::sub(Rt.s, bv))), Rt.e);
    L.s = x;
  } else {  // kKahan: feed the lane sum, then its negated pending correction
    step<kKahan, A>(L, Rt.s);
    step<kKahan, A>(L, -Rt.e);
  }
  return L;
}

template <typename A>
__device__ __forceinline__ Pair<A> zero_pair() { return Pair<A>{A(0), A(0)}; }

// One element: the addend through the recurrence; for TP dots also the
// product's exact round-off r = fma(a, b, -p) into the error channel.
template <int M, typename T, bool DOT>
__device__ __forceinline__ void accumulate(Pair<typename Acc<M, T>::type>& st, T a, T b) {
  using A = typename Acc<M, T>::type;
  if constexpr (DOT && is_tp<M>()) {
    const T p = Ar<T>::mul(a, b);
    const T r = Ar<T>::fma(a, b, -p);
    step<M, A>(st, p);
    st.e = Ar<A>::add(st.e, r);
  } else {
    step<M, A>(st, addend<M, T, DOT>(a, b));
  }
}

// Dekker FAST-TWO-SUM (eft.py:39-42) and Knuth TWO-SUM (eft.py:51-56).
template <typename T>
__device__ __forceinline__ void fast_two_sum(T a, T b, T& x, T& y) {
  x = Ar<T>::add(a, b);
  T bv = Ar<T>::sub(x, a);
  y = Ar<T>::sub(b, bv);
}
template <typename T>
__device__ __forceinline__ void two_sum(T a, T b, T& x, T& y) {
  x = Ar<T>::add(a, b);
  T bv = Ar<T>::sub(x, a);
  T av = Ar<T>::sub(x, bv);
  T br = Ar<T>::sub(b, bv);
  T ar = Ar<T>::sub(a, av);
  y = Ar<T>::add(ar, br);
}

}  // namespace tfb
