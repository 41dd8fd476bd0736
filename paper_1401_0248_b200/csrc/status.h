// status.h — CUDA error capture shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include "twofold_b200.h"

namespace tfb {

// Per-thread text of the last CUDA failure (tf_last_cuda_error()).
void set_cuda_error(cudaError_t e);

inline int record_cuda_error() {
  set_cuda_error(cudaGetLastError());
  return TF_ECUDA;
}

inline int check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_cuda_error(e);
    return TF_ECUDA;
  }
  return TF_OK;
}

}  // namespace tfb
