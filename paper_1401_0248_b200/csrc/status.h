// status.h — CUDA error capture shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "twofold_b200.h"

namespace tfb {

// Per-thread text of the last CUDA failure (tf_last_cuda_error()).
void set_cuda_error(cudaError_t e);

inline int record_cuda_error() {
  set_cuda_error(cudaGetLastError());
  return TF_ECUDA;
}

// Process-wide count of kernels this library launched (tf_launch_count()).
std::atomic<uint64_t>& launch_counter();

// Called right after every kernel launch.
inline int check_launch() {
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_cuda_error(e);
    return TF_ECUDA;
  }
  return TF_OK;
}

}  // namespace tfb
