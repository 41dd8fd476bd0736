// hostleaf.cpp — the host-buffer engine's CPU leaf reducer (hybrid host path).
//
// When the operands live in host memory, every byte the GPU reduces must first
// cross PCIe (~55 GB/s on this pool), while the host cores read the same DRAM
// directly.  tf_host_reduce therefore lets its worker threads reduce some of
// the FULL leaves themselves and upload only their 8/16-byte leaf pairs; the
// GPU reduces the rest and merges all pairs with tf_merge_tree.  For that to
// leave the result bit-identical, a host leaf must be exactly the device leaf
// (reduce.cu): chain t of the leaf's 256 runs the reference
// recurrence (kernels.py:149-153 / :163-169 / :179-182 / :131 / :139, the
// product rounded in the data type, kernels.py:198, :209) over elements
// (k*256 + t)*V + j, k = 0..R-1, j = 0..V-1 (V = 16 B / sizeof T), then a
// balanced contiguous tree over the 256 chain states with the reference lane
// merge (kernels.py:310-317, :379-390; plain add for direct / wide).
//
// Vectorisation: eight chains per vector, the leaf's k-rows streamed in order
// (each 4 KiB row per operand read once), the 256 chain states in L1.  The
// chain-j addends of eight chains are gathered from the interleaved row by
// register shuffles.  Arithmetic is element-wise IEEE binary32/binary64 with
// round-to-nearest: built with -ffp-contract=off (no FMA contraction),
// without fast-math, and the workers clear FTZ/DAZ (subnormals in contract,
// like the device build's -ftz=false).  Compiled twice (AVX-512 and the
// x86-64 baseline) and dispatched at run time; same results either way.
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <type_traits>
#include <vector>

#ifndef TFB_HL_SUFFIX
#define TFB_HL_SUFFIX base
#endif
#define TFB_HL_CAT2(a, b) a##_##b
#define TFB_HL_CAT(a, b) TFB_HL_CAT2(a, b)
#define TFB_HL_NAME(f) TFB_HL_CAT(f, TFB_HL_SUFFIX)

namespace {

enum { kDirect = 0, kWide = 1, kFast = 2, kRigorous = 3, kKahan = 4 };
constexpr int kChains = 256;

typedef double v8d __attribute__((vector_size(64)));
typedef float v8f __attribute__((vector_size(32)));
typedef float v16f __attribute__((vector_size(64)));

template <typename A>
struct P {
  A s, e;
};

// One element of the sequential recurrence (eft.cuh step<M>), element-wise.
template <int M, typename A>
inline void step(P<A>& st, A y) {
  if constexpr (M == kDirect || M == kWide) {
    st.s = st.s + y;
  } else if constexpr (M == kFast) {
    A t = st.s + y;
    A c = (t - st.s) - y;
    st.e = st.e - c;
    st.s = t;
  } else if constexpr (M == kRigorous) {
    A t = st.s + y;
    A yt = t - st.s;
    A dy = y - yt;
    A ds = st.s - (t - yt);
    st.e = st.e + (ds + dy);
    st.s = t;
  } else {  // Kahan: y' = y - c; t = s + y'; c = (t - s) - y'; s = t
    A yy = y - st.e;
    A t = st.s + yy;
    st.e = (t - st.s) - yy;
    st.s = t;
  }
}

// Merge right into left (eft.cuh merge<M>).
template <int M, typename A>
inline P<A> merge(P<A> L, P<A> R) {
  if constexpr (M == kDirect || M == kWide) {
    L.s = L.s + R.s;
  } else if constexpr (M == kFast || M == kRigorous) {
    A x = L.s + R.s;
    A bv = x - L.s;
    A sv = x - bv;
    L.e = (L.e + ((L.s - sv) + (R.s - bv))) + R.e;
    L.s = x;
  } else {
    step<kKahan, A>(L, R.s);
    step<kKahan, A>(L, -R.e);
  }
  return L;
}

template <typename V>
inline V loadv(const void* p) {
  V v;
  std::memcpy(&v, p, sizeof(V));
  return v;
}

// Balanced contiguous tree over cnt (a power of two) states / pairs, in place:
// level by level, (2i, 2i+1) with the left operand first — the device trees'
// order (block_tree over the 256 chains, tree_over over a row's leaves).
template <int M, typename A>
inline P<A> tree_pow2(P<A>* a, int64_t cnt) {
  for (int64_t w = cnt; w > 1; w >>= 1)
    for (int64_t i = 0; i < w / 2; ++i) a[i] = merge<M, A>(a[2 * i], a[2 * i + 1]);
  return a[0];
}

// The addend of one element in the accumulator type: the product rounded in the
// data type (kernels.py:198, :209), widened exactly for wide.
template <typename S, typename T, bool DOT>
inline S addend_scalar(T a, T b) {
  if constexpr (DOT) {
    const T p = a * b;
    return static_cast<S>(p);
  } else {
    return static_cast<S>(a);
  }
}

// binary64 leaf of n <= L elements: V = 2, a k-row is 512 elements; chains
// 8g..8g+7 are the 16 consecutive elements at 16g, their j = 0 / 1 addends the even
// / odd ones.  Full k-rows run vectorised; a partial last k-row (a partial leaf)
// continues every chain in order on its scalar state, elements past n skipped.
template <int M, bool DOT>
void leaf_f64(const double* x, const double* y, int64_t n, double* out) {
  alignas(64) P<v8d> st[kChains / 8];
  for (auto& p : st) p = P<v8d>{v8d{}, v8d{}};
  const int64_t kfull = n / 512;
  for (int64_t k = 0; k < kfull; ++k) {
    const double* xk = x + k * 512;
    const double* yk = DOT ? y + k * 512 : nullptr;
    for (int g = 0; g < kChains / 8; ++g) {
      const v8d x0 = loadv<v8d>(xk + 16 * g), x1 = loadv<v8d>(xk + 16 * g + 8);
      v8d e = __builtin_shufflevector(x0, x1, 0, 2, 4, 6, 8, 10, 12, 14);
      v8d o = __builtin_shufflevector(x0, x1, 1, 3, 5, 7, 9, 11, 13, 15);
      if constexpr (DOT) {
        const v8d y0 = loadv<v8d>(yk + 16 * g), y1 = loadv<v8d>(yk + 16 * g + 8);
        e = e * __builtin_shufflevector(y0, y1, 0, 2, 4, 6, 8, 10, 12, 14);
        o = o * __builtin_shufflevector(y0, y1, 1, 3, 5, 7, 9, 11, 13, 15);
      }
      step<M, v8d>(st[g], e);
      step<M, v8d>(st[g], o);
    }
  }
  P<double> s[kChains];
  for (int t = 0; t < kChains; ++t) s[t] = P<double>{st[t / 8].s[t % 8], st[t / 8].e[t % 8]};
  if (kfull * 512 < n)
    for (int t = 0; t < kChains; ++t)
      for (int j = 0; j < 2; ++j) {
        const int64_t i = (kfull * 256 + t) * 2 + j;
        if (i < n) step<M, double>(s[t], addend_scalar<double, double, DOT>(x[i], DOT ? y[i] : 0.0));
      }
  const P<double> r = tree_pow2<M, double>(s, kChains);
  out[0] = r.s;
  out[1] = r.e;
}

// binary32 leaf of n <= L elements: V = 4, a k-row is 1024 elements; chains
// 8g..8g+7 are the 32 consecutive elements at 32g, chain c's j-th addend at 4c + j.
// WIDE widens the binary32 addend (product rounded in binary32) exactly to binary64
// chains.  A partial last k-row continues on the scalar states, as binary64.
template <int M, bool DOT>
void leaf_f32(const float* x, const float* y, int64_t n, double* out) {
  using A = typename std::conditional<M == kWide, v8d, v8f>::type;
  using S = typename std::conditional<M == kWide, double, float>::type;
  alignas(64) P<A> st[kChains / 8];
  for (auto& p : st) p = P<A>{A{}, A{}};
  const int64_t kfull = n / 1024;
  for (int64_t k = 0; k < kfull; ++k) {
    const float* xk = x + k * 1024;
    const float* yk = DOT ? y + k * 1024 : nullptr;
    for (int g = 0; g < kChains / 8; ++g) {
      const v16f x0 = loadv<v16f>(xk + 32 * g), x1 = loadv<v16f>(xk + 32 * g + 16);
      v16f y0{}, y1{};
      if constexpr (DOT) {
        y0 = loadv<v16f>(yk + 32 * g);
        y1 = loadv<v16f>(yk + 32 * g + 16);
      }
#define TFB_HL_J(J)                                                                                            \
  {                                                                                                            \
    v8f a = __builtin_shufflevector(x0, x1, J, 4 + J, 8 + J, 12 + J, 16 + J, 20 + J, 24 + J, 28 + J);          \
    if constexpr (DOT) a = a * __builtin_shufflevector(y0, y1, J, 4 + J, 8 + J, 12 + J, 16 + J, 20 + J, 24 + J, \
                                                       28 + J);                                                \
    if constexpr (M == kWide) step<M, A>(st[g], __builtin_convertvector(a, v8d));                              \
    else step<M, A>(st[g], a);                                                                                 \
  }
      TFB_HL_J(0)
      TFB_HL_J(1)
      TFB_HL_J(2)
      TFB_HL_J(3)
#undef TFB_HL_J
    }
  }
  P<S> s[kChains];
  for (int t = 0; t < kChains; ++t) s[t] = P<S>{st[t / 8].s[t % 8], st[t / 8].e[t % 8]};
  if (kfull * 1024 < n)
    for (int t = 0; t < kChains; ++t)
      for (int j = 0; j < 4; ++j) {
        const int64_t i = (kfull * 256 + t) * 4 + j;
        if (i < n) step<M, S>(s[t], addend_scalar<S, float, DOT>(x[i], DOT ? y[i] : 0.0f));
      }
  const P<S> r = tree_pow2<M, S>(s, kChains);
  out[0] = r.s;
  out[1] = r.e;
}

template <int M, bool DOT>
void leaves(int dtype, const void* x, const void* y, int lg, int64_t lo, int64_t hi, void* pairs) {
  const int64_t L = int64_t(1) << lg;
  double o[2];
  for (int64_t l = lo; l < hi; ++l) {
    if (dtype == 1) {
      if constexpr (M != kWide) {
        leaf_f64<M, DOT>(static_cast<const double*>(x) + l * L, DOT ? static_cast<const double*>(y) + l * L : nullptr,
                         L, o);
        static_cast<double*>(pairs)[2 * (l - lo)] = o[0];
        static_cast<double*>(pairs)[2 * (l - lo) + 1] = o[1];
      }
    } else {
      leaf_f32<M, DOT>(static_cast<const float*>(x) + l * L, DOT ? static_cast<const float*>(y) + l * L : nullptr,
                       L, o);
      if constexpr (M == kWide) {
        static_cast<double*>(pairs)[2 * (l - lo)] = o[0];
        static_cast<double*>(pairs)[2 * (l - lo) + 1] = o[1];
      } else {
        static_cast<float*>(pairs)[2 * (l - lo)] = static_cast<float>(o[0]);
        static_cast<float*>(pairs)[2 * (l - lo) + 1] = static_cast<float>(o[1]);
      }
    }
  }
}

// Row pairs of rows [lo, hi) of a (rows, cols) matrix with leading dimensions
// ldx / ldy at leaf size L = 2^lg: each row is its own reduction — leaves of L
// elements (the last one partial), then the balanced tree over the row's leaf
// pairs padded with (+0, +0) to a power of two (tf_reduce_rows' row tree; a
// single-leaf row is its leaf pair).
template <int M, bool DOT>
void rows(int dtype, const void* x, const void* y, int64_t lo, int64_t hi, int64_t cols, int64_t ldx, int64_t ldy,
          int lg, void* pairs) {
  const int64_t L = int64_t(1) << lg;
  const int64_t npl = cols > 0 ? (cols + L - 1) / L : 1;  // leaves per row
  int64_t P2 = 1;
  while (P2 < npl) P2 <<= 1;
  const bool wide_acc = (M == kWide) || dtype == 1;  // accumulator binary64
  std::vector<double> lp(2 * P2);
  for (int64_t r = lo; r < hi; ++r) {
    std::fill(lp.begin(), lp.end(), 0.0);
    for (int64_t l = 0; l < npl; ++l) {
      const int64_t n = std::min(L, cols - l * L);
      if (n <= 0) continue;
      if (dtype == 1) {
        if constexpr (M != kWide)
          leaf_f64<M, DOT>(static_cast<const double*>(x) + r * ldx + l * L,
                           DOT ? static_cast<const double*>(y) + r * ldy + l * L : nullptr, n, &lp[2 * l]);
      } else {
        leaf_f32<M, DOT>(static_cast<const float*>(x) + r * ldx + l * L,
                         DOT ? static_cast<const float*>(y) + r * ldy + l * L : nullptr, n, &lp[2 * l]);
      }
    }
    double o[2];
    if (npl == 1) {
      o[0] = lp[0];
      o[1] = lp[1];
    } else if (wide_acc) {
      std::vector<P<double>> t(P2);
      for (int64_t i = 0; i < P2; ++i) t[i] = P<double>{lp[2 * i], lp[2 * i + 1]};
      const P<double> root = tree_pow2<M, double>(t.data(), P2);
      o[0] = root.s;
      o[1] = root.e;
    } else {
      std::vector<P<float>> t(P2);
      for (int64_t i = 0; i < P2; ++i) t[i] = P<float>{static_cast<float>(lp[2 * i]), static_cast<float>(lp[2 * i + 1])};
      const P<float> root = tree_pow2<M, float>(t.data(), P2);
      o[0] = root.s;
      o[1] = root.e;
    }
    if (wide_acc) {
      static_cast<double*>(pairs)[2 * (r - lo)] = o[0];
      static_cast<double*>(pairs)[2 * (r - lo) + 1] = o[1];
    } else {
      static_cast<float*>(pairs)[2 * (r - lo)] = static_cast<float>(o[0]);
      static_cast<float*>(pairs)[2 * (r - lo) + 1] = static_cast<float>(o[1]);
    }
  }
}

}  // namespace

extern "C" int TFB_HL_NAME(tfb_host_rows)(int method, int dtype, const void* x, const void* y, int64_t lo, int64_t hi,
                                          int64_t cols, int64_t ldx, int64_t ldy, int lg, void* pairs) {
  if (lg < (dtype == 1 ? 9 : 10)) return -1;
  const bool dot = y != nullptr;
  switch (method) {
#define TFB_HR_CASE(M)                                                               \
  case M:                                                                            \
    if (dot) rows<M, true>(dtype, x, y, lo, hi, cols, ldx, ldy, lg, pairs);          \
    else rows<M, false>(dtype, x, y, lo, hi, cols, ldx, ldy, lg, pairs);             \
    return 0;
    TFB_HR_CASE(kDirect)
    TFB_HR_CASE(kWide)
    TFB_HR_CASE(kFast)
    TFB_HR_CASE(kRigorous)
    TFB_HR_CASE(kKahan)
#undef TFB_HR_CASE
    default:
      return -1;
  }
}

// Leaf pairs of the FULL leaves [lo, hi) of x (and y): pairs[l - lo] in the
// accumulator type.  The caller guarantees lg >= log2(256 V), full leaves,
// method in 0..4 (no TwoProduct) and no WIDE on binary64.  Returns 0 or -1.
extern "C" int TFB_HL_NAME(tfb_host_leaves)(int method, int dtype, const void* x, const void* y, int lg, int64_t lo,
                                            int64_t hi, void* pairs) {
  if (lg < (dtype == 1 ? 9 : 10)) return -1;
  const bool dot = y != nullptr;
  switch (method) {
#define TFB_HL_CASE(M)                                                              \
  case M:                                                                           \
    if (dot) leaves<M, true>(dtype, x, y, lg, lo, hi, pairs);                       \
    else leaves<M, false>(dtype, x, y, lg, lo, hi, pairs);                          \
    return 0;
    TFB_HL_CASE(kDirect)
    TFB_HL_CASE(kWide)
    TFB_HL_CASE(kFast)
    TFB_HL_CASE(kRigorous)
    TFB_HL_CASE(kKahan)
#undef TFB_HL_CASE
    default:
      return -1;
  }
}
