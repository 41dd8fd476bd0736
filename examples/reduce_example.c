/* Native caller of the C ABI (include/twofold_b200.h): generate cfg5-like data on
 * the device, run the twofold dot through tf_reduce on a user stream, print the
 * (value, error) pair and the exact sum from tf_exact; then reduce the same data
 * from plain malloc'd host arrays through the host-buffer engine
 * (tf_host_reduce) and check the pair is bit-identical.
 *
 *   cc reduce_example.c -I../include -I/usr/local/cuda/include \
 *      -L../paper_1401_0248_b200 -ltwofold_b200 -L/usr/local/cuda/lib64 -lcudart \
 *      -Wl,-rpath,../paper_1401_0248_b200:/usr/local/cuda/lib64
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "twofold_b200.h"

#define CK(call)                                                                   \
  do {                                                                             \
    int rc_ = (call);                                                              \
    if (rc_) {                                                                     \
      fprintf(stderr, "%s -> %s %s\n", #call, tf_strerror(rc_), tf_last_cuda_error()); \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : (int64_t)1 << 24;
  CK(tf_canary());
  cudaStream_t s;
  if (cudaStreamCreate(&s) != cudaSuccess) return 1;
  double *x, *y, *pair, *exact;
  size_t pbytes = 0;
  int64_t ncounters = 0, leaves = 0;
  CK(tf_workspace_size(TF_TWOFOLD_FAST, TF_F64, 1, n, 0, &pbytes, &ncounters, &leaves));
  void *partials, *counters, *records;
  int64_t nrec = 0;
  size_t rbytes = 0;
  CK(tf_exact_workspace(&nrec, &rbytes));
  if (cudaMalloc((void**)&x, n * sizeof(double)) || cudaMalloc((void**)&y, n * sizeof(double)) ||
      cudaMalloc((void**)&pair, 2 * sizeof(double)) || cudaMalloc((void**)&exact, 2 * sizeof(double)) ||
      cudaMalloc(&partials, pbytes ? pbytes : 16) || cudaMalloc(&counters, 4 * (ncounters + 1)) ||
      cudaMalloc(&records, rbytes))
    return 1;
  cudaMemsetAsync(counters, 0, 4 * (ncounters + 1), s);  /* zero once; kernels leave them zero */
  cudaMemsetAsync(records, 0, rbytes, s);                  /* the exact oracle's accumulator, likewise */
  CK(tf_fill(TF_DIST_UNIFORM_SYM, TF_F64, 4, 0, 0, n, 0, 0, 0, n, x, s));
  CK(tf_fill(TF_DIST_UNIFORM_SYM, TF_F64, 4, 1, 0, n, 0, 0, 0, n, y, s));
  CK(tf_reduce(TF_TWOFOLD_FAST, TF_F64, x, y, n, 0, pair, partials, pbytes, counters, ncounters, s));
  CK(tf_exact(TF_F64, x, y, n, 0, exact, NULL, records, rbytes, (char*)counters + 4 * ncounters, s));
  double h[2], e[2];
  cudaMemcpyAsync(h, pair, sizeof(h), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(e, exact, sizeof(e), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return 1;
  printf("n=%lld leaves=%lld value=%.17g error=%.17g exact_hi=%.17g exact_lo=%.17g\n", (long long)n,
         (long long)leaves, h[0], h[1], e[0], e[1]);
  printf("launch: %s\n", tf_last_launch());
  /* v + e must equal the exact sum to well below one ulp of it */
  const double dev = (h[0] - e[0]) + (h[1] - e[1]);
  if ((dev < 0 ? -dev : dev) > 1e-13 * (e[0] < 0 ? -e[0] : e[0]) + 1e-300) return 2;

  /* the same dot from pageable host memory: one blocking call */
  double* hx = (double*)malloc(n * sizeof(double));
  double* hy = (double*)malloc(n * sizeof(double));
  if (!hx || !hy) return 1;
  if (cudaMemcpy(hx, x, n * sizeof(double), cudaMemcpyDeviceToHost) ||
      cudaMemcpy(hy, y, n * sizeof(double), cudaMemcpyDeviceToHost))
    return 1;
  void* engine = NULL;
  double hp[2];
  CK(tf_host_engine_create(0, 0, 0, &engine));
  CK(tf_host_reduce(engine, TF_TWOFOLD_FAST, TF_F64, hx, hy, n, 0, hp, NULL));
  printf("host engine (%d copy threads): value=%.17g error=%.17g %s\n", tf_host_engine_threads(engine), hp[0],
         hp[1], (hp[0] == h[0] && hp[1] == h[1]) ? "bit-identical" : "MISMATCH");
  CK(tf_host_engine_destroy(engine));
  free(hx);
  free(hy);
  return (hp[0] == h[0] && hp[1] == h[1]) ? 0 : 3;
}
