// exact.cu — exact (correctly rounded) sum / dot on the GPU: SURVEY.md §8(f) f2,
// the device counterpart of the reference's expansion oracle
// (expansion.py:79-140: exact_sum, exact_dot, Expansion.hi/.lo, relative_error).
//
// Method (ExBLAS-style, all integer steps exact and associative):
//   * each thread keeps a K=4-component floating-point expansion; every addend
//     goes through a TwoSum cascade (exact: the multiset value never changes);
//     whatever falls out of the last component is deposited into the CTA's
//     fixed-point superaccumulator in shared memory;
//   * the superaccumulator anchors bit 0 at 2^-1074 and stores 32-bit digits
//     in int64 limbs (carry-save; 2^31 deposits per limb before overflow);
//   * at the end every thread deposits its expansion, the CTA normalises its
//     limbs and adds them into a grid accumulator in global memory with integer
//     atomics (exact and order-independent, hence bit-reproducible for any
//     grid); the last CTA (retire ticket) reads the total, zeroes the
//     accumulator, normalises, and rounds to hi = fl(S), lo = fl(S - hi) (round
//     to nearest even; the reference's relative_error uses exactly these two
//     leading components, expansion.py:129-140).  (A per-CTA record summed by the
//     last CTA cost ~100 µs at 592 CTAs; bit-by-bit rounding another ~50 µs.)
#include <cuda_runtime.h>

#include <cstdint>

#include "eft.cuh"
#include "status.h"
#include "twofold_b200.h"

namespace tfb {

constexpr int kExactThreads = 256;
constexpr int kLimbs = 72;   // 72 * 32 = 2304 bit positions >= 2098 + 64 carry bits
#ifndef TFB_EXACT_K
#define TFB_EXACT_K 4
#endif
#ifndef TFB_EXACT_DUAL
#define TFB_EXACT_DUAL 0
#endif
#ifndef TFB_EXACT_U
#define TFB_EXACT_U 0  // 16-byte vectors per operand loaded ahead of the cascades (0: sums 4, dots 2)
#endif
#ifndef TFB_EXACT_MINB
#define TFB_EXACT_MINB 4
#endif
#ifndef TFB_EXACT_MINB_SUM
#define TFB_EXACT_MINB_SUM TFB_EXACT_MINB  // sums (one operand) may fit more CTAs per SM
#endif
constexpr int kExactMinBlocks = TFB_EXACT_MINB;  // CTAs per SM (register cap) and grid = SMs x this
constexpr int kExpK = TFB_EXACT_K;        // per-thread expansion length
constexpr int kExpN = 1 + TFB_EXACT_DUAL;  // independent expansions per thread (ILP)

// Grid accumulator (caller scratch, zero on entry, left zero): kLimbs digit sums,
// the top carry sum and the non-finite count.
constexpr int kAccWords = kLimbs + 2;

__device__ __noinline__ void deposit(long long* acc, double v) {
  if (v == 0.0) return;
  const unsigned long long bits = __double_as_longlong(v);
  const bool neg = bits >> 63;
  const int ebits = static_cast<int>((bits >> 52) & 0x7FF);
  unsigned long long m = bits & 0xFFFFFFFFFFFFFull;
  int s;  // bit position of the significand's LSB above 2^-1074
  if (ebits == 0) {
    s = 0;  // subnormal: m * 2^-1074
  } else {
    m |= 1ull << 52;
    s = ebits - 1;  // normal: m * 2^(ebits - 1075) = m * 2^(ebits-1 - 1074)
  }
  const int d = s >> 5, r = s & 31;
  TFB_CHECK(d >= 0 && d + 2 < kLimbs);
  const unsigned long long lo = m << r;                       // bits 0..63 of m << r
  const unsigned long long hi = r ? (m >> (64 - r)) : 0ull;    // bits 64..84
  long long c0 = static_cast<long long>(lo & 0xFFFFFFFFull);
  long long c1 = static_cast<long long>(lo >> 32);
  long long c2 = static_cast<long long>(hi);
  if (neg) { c0 = -c0; c1 = -c1; c2 = -c2; }
  auto* u = reinterpret_cast<unsigned long long*>(acc);
  if (c0) atomicAdd(u + d, static_cast<unsigned long long>(c0));
  if (c1) atomicAdd(u + d + 1, static_cast<unsigned long long>(c1));
  if (c2) atomicAdd(u + d + 2, static_cast<unsigned long long>(c2));
}

__device__ __forceinline__ void cascade(double (&a)[kExpK], double x, long long* acc) {
  // Keep every expansion component below 2^1001 so no TwoSum can overflow:
  // huge addends (or a huge leading component) go straight to the fixed-point
  // accumulator, which represents any finite sum of finite doubles exactly.
  if (fabs(x) >= 0x1p1000 || fabs(a[0]) >= 0x1p1000) {
    deposit(acc, x);
    return;
  }
  // Early exit: once a TwoSum is exact nothing is left to carry (typical data
  // settles after two components, halving the FP64 work per addend).
#pragma unroll
  for (int i = 0; i < kExpK; ++i) {
    double s, e;
    two_sum<double>(a[i], x, s, e);
    a[i] = s;
    x = e;
    if (x == 0.0) return;
  }
  deposit(acc, x);
}

template <typename T> struct ExVec;
template <> struct ExVec<float> { using type = float4; static constexpr int V = 4; };
template <> struct ExVec<double> { using type = double2; static constexpr int V = 2; };
__device__ __forceinline__ float4 ex_ld(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ex_ld(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ float ex_get(const float4& v, int j) {
  return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
}
__device__ __forceinline__ double ex_get(const double2& v, int j) { return j == 0 ? v.x : v.y; }

// Addends: 0 = x_i, 1 = fl_T(x_i*y_i) (the twofold kernels' addends), 2 = exact
// products (fl(x*y) and fma(x, y, -fl(x*y)) for binary64; exact in binary64 for
// binary32 data).  abs: |addend| (A = sum |y_i| of the tolerances).
// MODE / ABS are template parameters: the per-element path has no runtime
// branches besides the cascade's early exit.
template <typename T, int MODE, bool ABS>
__device__ __forceinline__ void add_element(double (&a)[kExpK], long long* acc, T xv, T yv, int& nonfinite) {
  constexpr bool kResidual = MODE == 2 && sizeof(T) == 8;  // binary64 true products carry fma residuals
  double p, r = 0.0;
  if constexpr (MODE == 0) {
    p = static_cast<double>(xv);
  } else if constexpr (MODE == 1) {
    p = static_cast<double>(Ar<T>::mul(xv, yv));
  } else {
    p = __dmul_rn(static_cast<double>(xv), static_cast<double>(yv));  // exact for binary32 data
    if constexpr (kResidual) r = __fma_rn(static_cast<double>(xv), static_cast<double>(yv), -p);
  }
  if (!isfinite(p) || (kResidual && !isfinite(r))) {
    ++nonfinite;
    return;
  }
  if constexpr (ABS) {
    if (p < 0.0) {  // |p + r| = -(p + r) when p < 0 (|r| <= ulp(p)/2)
      p = -p;
      r = -r;
    }
  }
  cascade(a, p, acc);
  if constexpr (kResidual) {
    if (r != 0.0) cascade(a, r, acc);
  }
}

// Normalise limbs (digits -> [0, 2^32), signed carry out) by one thread.
__device__ void normalise(long long* limb, long long& top) {
  long long carry = 0;
  for (int k = 0; k < kLimbs; ++k) {
    const long long v = limb[k] + carry;  // |v| < 2^63 by the deposit bound
    limb[k] = v & 0xFFFFFFFFll;
    carry = v >> 32;                      // arithmetic shift: floor division
  }
  top += carry;
}

// Digits of a magnitude (kDig words in [0, 2^32), value * 2^-1074): the 53-bit
// significand is read as one 64-bit window (bits64), not bit by bit.
__device__ __forceinline__ unsigned long long dig(const unsigned long long* mag, int ndig, int i) {
  return (i >= 0 && i < ndig) ? mag[i] : 0ull;
}
// bits [lo, lo + 64) of the magnitude (bits below 0 read as zero)
__device__ unsigned long long bits64(const unsigned long long* mag, int ndig, int lo) {
  const int d = lo >= 0 ? lo >> 5 : -((31 - lo) >> 5);  // floor(lo / 32)
  const int r = lo - 32 * d;                           // 0..31
  const unsigned __int128 w = static_cast<unsigned __int128>(dig(mag, ndig, d)) |
                              (static_cast<unsigned __int128>(dig(mag, ndig, d + 1)) << 32) |
                              (static_cast<unsigned __int128>(dig(mag, ndig, d + 2)) << 64) |
                              (static_cast<unsigned __int128>(dig(mag, ndig, d + 3)) << 96);
  return static_cast<unsigned long long>(w >> r);
}
// ---- the last CTA's finish, by warp 0 (32 lanes; digit arrays in shared memory,
// slot k owned by lane k % 32): carry propagation in rounds, sign/magnitude and
// both roundings with ballot scans instead of one thread walking 74 digits
// (that serial form cost ~17 µs per call).

constexpr int kDig = kLimbs + 2;  // magnitude digits: 72 limbs + the top carry's two

__device__ __forceinline__ int warp_highest_nonzero(const unsigned long long* a, int n) {
  int best = -1;
  for (int base = 0; base < n; base += 32) {
    const int k = base + static_cast<int>(threadIdx.x & 31);
    const unsigned b = __ballot_sync(0xffffffffu, k < n && a[k] != 0);
    if (b) best = base + 31 - __clz(b);
  }
  return best;
}
__device__ __forceinline__ int warp_lowest_nonzero(const unsigned long long* a, int n) {
  for (int base = 0; base < n; base += 32) {
    const int k = base + static_cast<int>(threadIdx.x & 31);
    const unsigned b = __ballot_sync(0xffffffffu, k < n && a[k] != 0);
    if (b) return base + __ffs(b) - 1;
  }
  return n;
}
__device__ __forceinline__ bool warp_any_nonzero_below(const unsigned long long* a, int n) {
  bool any = false;
  for (int base = 0; base < n; base += 32) {
    const int k = base + static_cast<int>(threadIdx.x & 31);
    any |= __any_sync(0xffffffffu, k < n && a[k] != 0);
  }
  return any;
}

// Round mag (kDig digits, warp-visible) * 2^-1074 to binary64, nearest-even; also
// reports the significand's last-bit weight `lsb` (-1: exact, no remainder) and
// whether it rounded up.  Uniform across the warp.
__device__ double round_digits_warp(const unsigned long long* mag, bool neg, int& lsb_out, bool& up) {
  lsb_out = -1;
  up = false;
  const int hd = warp_highest_nonzero(mag, kDig);
  if (hd < 0) return 0.0;
  const int p = hd * 32 + (63 - __clzll(mag[hd]));
  double out;
  if (p < 53) {  // exactly representable: integer < 2^53 times 2^-1074
    out = scalbn(static_cast<double>(bits64(mag, kDig, 0)), -1074);
  } else {
    const int lsb = p - 52;
    unsigned long long m = bits64(mag, kDig, lsb) & ((1ull << 53) - 1);
    const unsigned long long guard = bits64(mag, kDig, lsb - 1) & 1ull;
    const int se = lsb - 1;  // sticky range [0, se)
    bool sticky = warp_any_nonzero_below(mag, se >> 5);
    if (!sticky && (se & 31)) sticky = (dig(mag, kDig, se >> 5) & ((1ull << (se & 31)) - 1)) != 0;
    if (guard && (sticky || (m & 1ull))) {
      ++m;  // may carry to 2^53: still exact in scalbn
      up = true;
    }
    lsb_out = lsb;
    out = scalbn(static_cast<double>(m), lsb - 1074);
  }
  return neg ? -out : out;
}

// tot: kLimbs digit sums (>= 0) + top carry sum + non-finite count, in shared memory.
// mag, rem: kDig-word shared scratch.  Called by all 32 lanes of one warp.
__device__ void finish_warp(long long* tot, unsigned long long* mag, unsigned long long* rem, double* out,
                            long long* limbs_out, unsigned* counter) {
  const int lane = static_cast<int>(threadIdx.x & 31);
  __shared__ long long s_carry_top;
  long long top = tot[kLimbs];
  const long long nonfin = tot[kLimbs + 1];
  // normalise: digits to [0, 2^32) in rounds (the first moves < 2^10 per digit, later
  // rounds only ripple through all-ones digits)
  for (;;) {
    long long c[3];
#pragma unroll
    for (int sl = 0; sl < 3; ++sl) {
      const int k = lane + 32 * sl;
      c[sl] = 0;
      if (k < kLimbs) {
        c[sl] = tot[k] >> 32;  // tot[k] >= 0
        tot[k] &= 0xFFFFFFFFll;
      }
    }
    if (lane == 0) s_carry_top = 0;
    __syncwarp();
#pragma unroll
    for (int sl = 0; sl < 3; ++sl) {
      const int k = lane + 32 * sl;
      if (k < kLimbs && c[sl]) {
        if (k + 1 < kLimbs) tot[k + 1] += c[sl];
        else s_carry_top = c[sl];
      }
    }
    const bool more = __any_sync(0xffffffffu, (c[0] | c[1] | c[2]) != 0);
    __syncwarp();
    top += s_carry_top;
    __syncwarp();
    if (!more) break;
  }
  if (limbs_out) {
    for (int k = lane; k < kLimbs; k += 32) limbs_out[k] = tot[k];
    if (lane == 0) limbs_out[kLimbs] = top;
  }
  // sign and magnitude: value = D + top * 2^(32 kLimbs), 0 <= D < 2^(32 kLimbs)
  const bool neg = top < 0;
  for (int k = lane; k < kLimbs; k += 32) mag[k] = static_cast<unsigned long long>(tot[k]);
  __syncwarp();
  unsigned long long utop = static_cast<unsigned long long>(top);
  if (neg) {  // |value| = (|top| - 1) 2^(32 kLimbs) + (2^(32 kLimbs) - D), or |top| 2^(32 kLimbs) if D = 0
    const int z = warp_lowest_nonzero(mag, kLimbs);
    __syncwarp();
    for (int k = lane; k < kLimbs; k += 32)
      mag[k] = k < z ? 0ull : (k == z ? (1ull << 32) - mag[k] : 0xFFFFFFFFull - mag[k]);
    utop = static_cast<unsigned long long>(-top) - (z < kLimbs ? 1ull : 0ull);
  }
  if (lane == 0) {
    mag[kLimbs] = utop & 0xFFFFFFFFull;
    mag[kLimbs + 1] = utop >> 32;
  }
  __syncwarp();
  if (nonfin) {
    if (lane == 0) {
      out[0] = __longlong_as_double(0x7FF8000000000000ll);
      out[1] = out[0];
      *counter = 0u;
    }
    return;
  }
  int lsb;
  bool up;
  const double hi = round_digits_warp(mag, neg, lsb, up);
  if (!isfinite(hi) || lsb < 0) {  // beyond binary64 (no meaningful remainder) or exact
    if (lane == 0) {
      out[0] = hi;
      out[1] = 0.0;
      *counter = 0u;
    }
    return;
  }
  // lo = fl(S - hi).  |S| = m0 2^lsb + low (m0 the truncated significand); hi took
  // m0 or m0 + 1, so S - hi = +-low or -+(2^lsb - low), 0 < low < 2^lsb when rounded up.
  const int q = lsb >> 5, qb = lsb & 31;
  for (int k = lane; k < kDig; k += 32)
    rem[k] = k < q ? mag[k] : (k == q && qb ? (mag[k] & ((1ull << qb) - 1)) : 0ull);
  __syncwarp();
  bool rneg = neg;
  if (up) {  // 2^lsb - low, complemented within lsb bits
    const int z = warp_lowest_nonzero(rem, kDig);
    __syncwarp();
    for (int k = lane; k < kDig; k += 32) {
      const unsigned long long full = k < q ? 0xFFFFFFFFull : (k == q && qb ? (1ull << qb) - 1 : 0ull);
      rem[k] = k < z ? 0ull : (k == z ? full + 1 - rem[k] : full - rem[k]);
    }
    rneg = !neg;
    __syncwarp();
  }
  int lsb2;
  bool up2;
  const double lo = round_digits_warp(rem, rneg, lsb2, up2);
  if (lane == 0) {
    out[0] = hi;
    out[1] = lo;
    *counter = 0u;  // leave the workspace reusable
  }
}

template <typename T, int MODE, bool ABS>
__global__ void __launch_bounds__(kExactThreads, MODE == 0 ? TFB_EXACT_MINB_SUM : kExactMinBlocks) exact_kernel(
    const T* __restrict__ x, const T* __restrict__ y, int64_t n,
    long long* __restrict__ gacc, unsigned* __restrict__ counter, double* __restrict__ out,
    long long* __restrict__ limbs_out) {
  constexpr bool DOT = MODE != 0;
  // one fixed-point accumulator per warp: the end-of-thread deposits of all 256
  // expansions would otherwise serialise on the same few shared-memory words
  __shared__ long long accw[kExactThreads / 32][kLimbs];
  long long* acc = accw[threadIdx.x >> 5];
  __shared__ long long s_top;
  __shared__ int s_last;
  __shared__ int s_nonfinite;
  for (int k = threadIdx.x; k < kLimbs * (kExactThreads / 32); k += blockDim.x) (&accw[0][0])[k] = 0;
  if (threadIdx.x == 0) s_nonfinite = 0;
  __syncthreads();
  double a[kExpN][kExpK];
#pragma unroll
  for (int q = 0; q < kExpN; ++q)
#pragma unroll
    for (int i = 0; i < kExpK; ++i) a[q][i] = 0.0;
  int nonfinite = 0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t gtid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  // 16-byte vector loads, U vectors per operand in flight before the cascades
  // run (the flush atomics keep the compiler from prefetching on its own).
  using VT = typename ExVec<T>::type;
  constexpr int VB = ExVec<T>::V;
  // measured (scripts/build_exact_variants.sh): sums 4 (f64 2^28 0.589 -> 0.548 ms), dots 2
  // (f64 dot 2^27 at 4: 0.397 -> 0.440 ms, the second operand's registers)
  constexpr int U = TFB_EXACT_U > 0 ? TFB_EXACT_U : (DOT ? 2 : 4);
  const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15u) == 0 &&
                       (!DOT || (reinterpret_cast<uintptr_t>(y) & 15u) == 0);
  int64_t scalar_from = 0;
  if (aligned) {
    const int64_t nv = n / VB;
    const VT* xv = reinterpret_cast<const VT*>(x);
    const VT* yv = reinterpret_cast<const VT*>(y);
    int64_t v = gtid;
    for (; v + (U - 1) * stride < nv; v += U * stride) {
      VT va[U], vb[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        va[k] = ex_ld(xv + v + k * stride);
        if constexpr (DOT) vb[k] = ex_ld(yv + v + k * stride);
      }
#pragma unroll
      for (int k = 0; k < U; ++k)
#pragma unroll
        for (int j = 0; j < VB; ++j)
          add_element<T, MODE, ABS>(a[j % kExpN], acc, ex_get(va[k], j), DOT ? ex_get(vb[k], j) : T(0),
                                    nonfinite);
    }
    for (; v < nv; v += stride) {
      const VT va = ex_ld(xv + v);
      VT vb;
      if constexpr (DOT) vb = ex_ld(yv + v);
#pragma unroll
      for (int j = 0; j < VB; ++j)
        add_element<T, MODE, ABS>(a[j % kExpN], acc, ex_get(va, j), DOT ? ex_get(vb, j) : T(0), nonfinite);
    }
    scalar_from = nv * VB;
  }
  for (int64_t i = scalar_from + gtid; i < n; i += stride)
    add_element<T, MODE, ABS>(a[0], acc, x[i], DOT ? y[i] : T(0), nonfinite);
#pragma unroll
  for (int q = 0; q < kExpN; ++q)
#pragma unroll
    for (int i = 0; i < kExpK; ++i) deposit(acc, a[q][i]);
  if (nonfinite) atomicAdd(&s_nonfinite, nonfinite);
  __syncthreads();
  for (int k = threadIdx.x; k < kLimbs; k += blockDim.x) {  // the CTA's sum of the warp accumulators
    long long v = 0;
#pragma unroll
    for (int w = 0; w < kExactThreads / 32; ++w) v += accw[w][k];
    accw[0][k] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long top = 0;
    normalise(accw[0], top);  // digits in [0, 2^32): the grid total stays far below 2^63
    s_top = top;
  }
  __syncthreads();
  // this CTA's digits into the grid accumulator: integer adds, exact and order-free
  for (int k = threadIdx.x; k < kLimbs + 2; k += blockDim.x) {
    const long long v = k < kLimbs ? accw[0][k] : (k == kLimbs ? s_top : static_cast<long long>(s_nonfinite));
    if (v) atomicAdd(reinterpret_cast<unsigned long long*>(&gacc[k]), static_cast<unsigned long long>(v));
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // last CTA: read the total, leave the accumulator zero for the next call, finish
  __shared__ long long tot[kLimbs + 2];
  __shared__ unsigned long long mag[kDig], rem[kDig];
  for (int k = threadIdx.x; k < kLimbs + 2; k += blockDim.x) {
    tot[k] = __ldcg(&gacc[k]);
    gacc[k] = 0;
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  finish_warp(tot, mag, rem, out, limbs_out, counter);
}

}  // namespace tfb

using namespace tfb;

extern "C" {

int tf_exact_workspace(int64_t* records, size_t* bytes) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t g = static_cast<int64_t>(sms) * kExactMinBlocks;
  if (records) *records = g;
  if (bytes) *bytes = static_cast<size_t>(kAccWords) * sizeof(long long);
  return TF_OK;
}

int tf_exact(int dtype, const void* x, const void* y, int64_t n, int flags, void* out2,
             void* limbs_out, void* records, size_t records_bytes, void* counter, void* stream) {
  if (dtype != TF_F32 && dtype != TF_F64) return TF_EINVAL_DTYPE;
  if (n < 0) return TF_EINVAL_SHAPE;
  if (!out2 || !counter || (n > 0 && !x)) return TF_EINVAL_ARG;
  if ((flags & TF_EXACT_TRUE_PRODUCTS) && !y) return TF_EINVAL_ARG;
  const int mode = y ? ((flags & TF_EXACT_TRUE_PRODUCTS) ? 2 : 1) : 0;
  int64_t g = 0;
  size_t need = 0;
  tf_exact_workspace(&g, &need);
  if (mode == 0) g = g / kExactMinBlocks * TFB_EXACT_MINB_SUM;  // sums: their own CTAs per SM
  const int64_t per = (n + kExactThreads - 1) / kExactThreads;
  if (g > per && per > 0) g = per;  // tiny inputs: fewer CTAs
  if (g < 1) g = 1;
  if (!records || records_bytes < static_cast<size_t>(kAccWords) * sizeof(long long)) return TF_EWORKSPACE;
  auto s = static_cast<cudaStream_t>(stream);
  const bool absval = (flags & TF_EXACT_ABS) != 0;
  const dim3 grid(static_cast<unsigned>(g));
  auto* rec = static_cast<long long*>(records);
  auto* ctr = static_cast<unsigned*>(counter);
  auto* o = static_cast<double*>(out2);
  auto* lo = static_cast<long long*>(limbs_out);
#define TFB_EXACT(T, MODE, ABS)                                                                            \
  exact_kernel<T, MODE, ABS><<<grid, kExactThreads, 0, s>>>(static_cast<const T*>(x), static_cast<const T*>(y), \
                                                           n, rec, ctr, o, lo)
#define TFB_EXACT_T(T)                                                                                     \
  do {                                                                                                     \
    if (mode == 0) { if (absval) TFB_EXACT(T, 0, true); else TFB_EXACT(T, 0, false); }                   \
    else if (mode == 1) { if (absval) TFB_EXACT(T, 1, true); else TFB_EXACT(T, 1, false); }              \
    else { if (absval) TFB_EXACT(T, 2, true); else TFB_EXACT(T, 2, false); }                             \
  } while (0)
  if (dtype == TF_F32) TFB_EXACT_T(float);
  else TFB_EXACT_T(double);
#undef TFB_EXACT_T
#undef TFB_EXACT
  return check_launch();
}

}  // extern "C"
