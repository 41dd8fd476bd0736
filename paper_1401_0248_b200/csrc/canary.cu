// canary.cu — the device strict-rounding canary (replaces kernels.py:545-568).
//
// Operands live in device memory so nothing is constant-folded; the kernel
// runs the same step/merge templates the reductions use.  The product build
// (-fmad=false, explicit _rn intrinsics) must pass.  The Makefile also builds
// this file a second time as a NEGATIVE CONTROL (libtfb_canary_unsafe.so:
// -DTFB_PLAIN_OPS=1 so eft.cuh uses plain operators, plus --use_fast_math so
// the compiler may contract products into FMAs) — the analogue of the
// reference's fastmath=True kernel in test_acceptance.py:243-258 — and
// tests/test_canary_negative.py proves the canary rejects that build.
#include <cuda_runtime.h>

#include <cstdio>

#include "eft.cuh"
#include "status.h"
#include "twofold_b200.h"

namespace tfb {

#if TFB_CANARY_STANDALONE  // the negative-control library carries its own status plumbing
static thread_local char g_cuda_err[256] = {0};
std::atomic<uint64_t>& launch_counter() {
  static std::atomic<uint64_t> c{0};
  return c;
}
void set_cuda_error(cudaError_t e) {
  std::snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
}
#endif

__device__ double g_canary_in[8];
__device__ double g_canary_out[8];

__global__ void canary_kernel() {
  const double* in = g_canary_in;
  double* out = g_canary_out;
  double x, y;
  fast_two_sum<double>(in[0], in[1], x, y);  // (1, 2^-53) -> (1, 2^-53)
  out[0] = x;
  out[1] = y;
  float xf, yf;
  fast_two_sum<float>(static_cast<float>(in[0]), static_cast<float>(in[2]), xf, yf);  // (1, 2^-24)
  out[2] = xf;
  out[3] = yf;
  // fl(fl(a*b) + s) == 0 exactly; a contracted fma(a, b, s) would give 2^-60.
  Pair<double> st{in[4], 0.0};
  step<kFast, double>(st, addend<kFast, double, true>(in[3], in[3]));
  out[4] = st.s;
  // binary32 twin: a = 1 + 2^-13, s = -(1 + 2^-12); fma would give 2^-26.
  Pair<float> sf{static_cast<float>(in[6]), 0.0f};
  step<kRigorous, float>(sf, addend<kRigorous, float, true>(static_cast<float>(in[5]),
                                                            static_cast<float>(in[5])));
  out[5] = sf.s;
  // twofold merge keeps the absorbed addend: (1,0) (+) (2^-53,0) -> (1, 2^-53)
  Pair<double> m = merge<kFast, double>(Pair<double>{in[0], 0.0}, Pair<double>{in[1], 0.0});
  out[6] = m.s;
  out[7] = m.e;
}

}  // namespace tfb

using namespace tfb;

extern "C" {

int tf_canary(void) {
  const double in[8] = {1.0, 0x1p-53, 0x1p-24, 1.0 + 0x1p-30, -(1.0 + 0x1p-29),
                        1.0 + 0x1p-13, -(1.0 + 0x1p-12), 0.0};
  if (cudaMemcpyToSymbol(g_canary_in, in, sizeof(in)) != cudaSuccess) return record_cuda_error();
  canary_kernel<<<1, 1>>>();
  if (int rc = check_launch()) return rc;
  double out[8];
  if (cudaMemcpyFromSymbol(out, g_canary_out, sizeof(out)) != cudaSuccess) return record_cuda_error();
  const bool ok = out[0] == 1.0 && out[1] == 0x1p-53 && out[2] == 1.0 && out[3] == 0x1p-24 &&
                  out[4] == 0.0 && out[5] == 0.0 && out[6] == 1.0 && out[7] == 0x1p-53;
  return ok ? TF_OK : TF_ECANARY;
}

#if TFB_CANARY_STANDALONE
int tf_canary_raw(double* out8) {  // the eight canary outputs, for the negative-control test's report
  const double in[8] = {1.0, 0x1p-53, 0x1p-24, 1.0 + 0x1p-30, -(1.0 + 0x1p-29),
                        1.0 + 0x1p-13, -(1.0 + 0x1p-12), 0.0};
  if (cudaMemcpyToSymbol(g_canary_in, in, sizeof(in)) != cudaSuccess) return record_cuda_error();
  canary_kernel<<<1, 1>>>();
  if (int rc = check_launch()) return rc;
  if (cudaMemcpyFromSymbol(out8, g_canary_out, 8 * sizeof(double)) != cudaSuccess) return record_cuda_error();
  return TF_OK;
}
#endif

}  // extern "C"
