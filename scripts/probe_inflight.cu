// probe_inflight.cu — standalone HBM probe (not part of the library): does the
// leaf-per-CTA access pattern of leaves_kernel reach the grid-stride read roof
// at mid sizes, and how many bytes in flight per thread does it need?
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/build/probe_inflight scripts/probe_inflight.cu
//   ./probe_inflight            (one line per case: µs per launch, GB/s; graph-replayed, rotating buffers)
//
// Kernels only XOR-fold the bytes (no FP chain), so the numbers isolate the
// memory side: grid-stride (tf_read_roof's shape) vs one leaf per CTA (two
// operands, batches of U 16-byte vectors per thread per operand, with or
// without a one-batch software prefetch).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));  \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

__device__ __forceinline__ uint4 ldv(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

template <int U>
__global__ void __launch_bounds__(256) gs_kernel(const uint4* __restrict__ p, int64_t nvec, unsigned* sink) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  unsigned acc = 0;
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  for (; i + (U - 1) * stride < nvec; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldv(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < nvec; i += stride) {
    uint4 v = ldv(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9E3779B9u) sink[0] = acc;
}

// Grid-stride with 32-byte loads per thread (LDG...256): U loads of 32 B in flight.
struct u8v { uint4 a, b; };
__device__ __forceinline__ u8v ldv32(const uint4* p) {
  u8v v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.a.x), "=r"(v.a.y), "=r"(v.a.z), "=r"(v.a.w), "=r"(v.b.x), "=r"(v.b.y), "=r"(v.b.z),
                 "=r"(v.b.w)
               : "l"(p));
  return v;
}
template <int U>
__global__ void __launch_bounds__(256) gs32_kernel(const uint4* __restrict__ p, int64_t npairs, unsigned* sink) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  unsigned acc = 0;
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  for (; i + (U - 1) * stride < npairs; i += U * stride) {
    u8v v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldv32(p + 2 * (i + u * stride));
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].a.x ^ v[u].a.w ^ v[u].b.y ^ v[u].b.z;
  }
  for (; i < npairs; i += stride) {
    const u8v v = ldv32(p + 2 * i);
    acc ^= v.a.x ^ v.a.w ^ v.b.y ^ v.b.z;
  }
  if (acc == 0x9E3779B9u) sink[0] = acc;
}

// One leaf (R vectors per thread per operand, 256 threads) per CTA iteration.
template <int U, bool PF>
__global__ void __launch_bounds__(256) leaf_kernel(const uint4* __restrict__ x, const uint4* __restrict__ y,
                                                   int R, int64_t P, unsigned* sink) {
  unsigned acc = 0;
  for (int64_t l = blockIdx.x; l < P; l += gridDim.x) {
    const uint4* xv = x + l * int64_t(R) * 256 + threadIdx.x;
    const uint4* yv = y + l * int64_t(R) * 256 + threadIdx.x;
    if (!PF) {
      for (int k = 0; k < R; k += U) {
        uint4 a[U], b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          a[u] = ldv(xv + (k + u) * 256);
          b[u] = ldv(yv + (k + u) * 256);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= a[u].x ^ a[u].w ^ b[u].y ^ b[u].z;
      }
    } else {
      uint4 a[U], b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a[u] = ldv(xv + u * 256);
        b[u] = ldv(yv + u * 256);
      }
      for (int k = 0; k < R; k += U) {
        uint4 a2[U], b2[U];
        if (k + U < R) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            a2[u] = ldv(xv + (k + U + u) * 256);
            b2[u] = ldv(yv + (k + U + u) * 256);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= a[u].x ^ a[u].w ^ b[u].y ^ b[u].z;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          a[u] = a2[u];
          b[u] = b2[u];
        }
      }
    }
  }
  if (acc == 0x9E3779B9u) sink[0] = acc;
}

// Two leaves per 256-thread CTA, 32-byte loads: thread tt (0..127) of half h
// reads vectors 2tt, 2tt+1 of every 256-vector row of leaf (2*l2 + h).
template <int U>
__global__ void __launch_bounds__(256) leaf32_kernel(const uint4* __restrict__ x, const uint4* __restrict__ y,
                                                     int R, int64_t P, unsigned* sink) {
  unsigned acc = 0;
  const int h = threadIdx.x >> 7, tt = threadIdx.x & 127;
  for (int64_t l2 = blockIdx.x; 2 * l2 < P; l2 += gridDim.x) {
    const int64_t l = 2 * l2 + h;
    if (l >= P) break;
    const uint4* xv = x + l * int64_t(R) * 256 + 2 * tt;
    const uint4* yv = y + l * int64_t(R) * 256 + 2 * tt;
    for (int k = 0; k < R; k += U) {
      u8v a[U], b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a[u] = ldv32(xv + (k + u) * 256);
        b[u] = ldv32(yv + (k + u) * 256);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc ^= a[u].a.x ^ a[u].b.w ^ b[u].a.y ^ b[u].b.z;
    }
  }
  if (acc == 0x9E3779B9u) sink[0] = acc;
}

struct Pool {
  char* base;
  size_t bytes;
};

template <typename F>
static float graph_us(F launch, int reps, cudaStream_t s) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < reps; ++i) launch(i);
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int t = 0; t < 4; ++t) {
    CK(cudaGraphLaunch(ge, s));
    CK(cudaEventRecord(e0, s));
    CK(cudaGraphLaunch(ge, s));
    CK(cudaEventRecord(e1, s));
    CK(cudaStreamSynchronize(s));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (t > 0 && ms < best) best = ms;
  }
  CK(cudaGraphExecDestroy(ge));
  CK(cudaGraphDestroy(g));
  return best * 1e3f / reps;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t pool_bytes = size_t(4) << 30;
  char* pool;
  CK(cudaMalloc(&pool, pool_bytes));
  CK(cudaMemset(pool, 0x5a, pool_bytes));
  unsigned* sink;
  CK(cudaMalloc(&sink, 4));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));

  // total bytes per launch (both operands)
  const size_t sizes[] = {size_t(8) << 20, size_t(32) << 20, size_t(128) << 20, size_t(512) << 20,
                          size_t(2048) << 20};
  for (size_t total : sizes) {
    const int slots = static_cast<int>(pool_bytes / total);
    const int reps = slots < 8 ? 8 : (slots > 40 ? 40 : slots);
    auto buf = [&](int i) { return reinterpret_cast<const uint4*>(pool + size_t(i % slots) * total); };
    const int64_t nvec = total / 16;
    printf("== %zu MB per launch (rotating over %d buffers)\n", total >> 20, slots);
    for (int mult : {4, 8, 16}) {
      const unsigned grid = sms * mult;
      float us4 = graph_us([&](int i) { gs_kernel<4><<<grid, 256, 0, s>>>(buf(i), nvec, sink); }, reps, s);
      float us8 = graph_us([&](int i) { gs_kernel<8><<<grid, 256, 0, s>>>(buf(i), nvec, sink); }, reps, s);
      printf("grid-stride grid=%u U4 %.2f us %.0f GB/s | U8 %.2f us %.0f GB/s\n", grid, us4, total / us4 / 1e3, us8,
             total / us8 / 1e3);
    }
    for (int mult : {4, 8}) {
      const unsigned grid = sms * mult;
      float a2 = graph_us([&](int i) { gs32_kernel<2><<<grid, 256, 0, s>>>(buf(i), nvec / 2, sink); }, reps, s);
      float a4 = graph_us([&](int i) { gs32_kernel<4><<<grid, 256, 0, s>>>(buf(i), nvec / 2, sink); }, reps, s);
      printf("grid-stride 32B grid=%u U2 %.2f us %.0f GB/s | U4 %.2f us %.0f GB/s\n", grid, a2, total / a2 / 1e3, a4,
             total / a4 / 1e3);
    }
    if (getenv("PROBE_GS_ONLY")) continue;
    for (int leaf_kb : {16, 32, 64, 128}) {
      const int64_t leaf_bytes = int64_t(leaf_kb) << 10;
      const int64_t P = (total / 2) / leaf_bytes;
      const int R = static_cast<int>(leaf_bytes / (16 * 256));
      if (P < 64) continue;
      for (int U : {2, 4}) {
        if (U > R) continue;
        for (int64_t occ : {int64_t(4), int64_t(8)}) {
          const int64_t cap = int64_t(sms) * occ;
          const unsigned grid = static_cast<unsigned>((P + 1) / 2 < cap ? (P + 1) / 2 : cap);
          auto L = [&](int i) {
            const uint4* x = buf(i);
            const uint4* y = x + nvec / 2;
            if (U == 2) leaf32_kernel<2><<<grid, 256, 0, s>>>(x, y, R, P, sink);
            else leaf32_kernel<4><<<grid, 256, 0, s>>>(x, y, R, P, sink);
          };
          float us = graph_us(L, reps, s);
          printf("leaf32 %3d KB/operand P=%5lld grid=%u U=%d: %.2f us %.0f GB/s\n", leaf_kb,
                 static_cast<long long>(P), grid, U, us, total / us / 1e3);
        }
      }
    }
    if (getenv("PROBE_LEAF32_ONLY")) continue;
    // leaves: operand bytes = total/2; leaf bytes per operand = 2^leaf_log2 * 4 (f32 view)
    for (int leaf_kb : {8, 16, 32, 64, 128, 256}) {
      const int64_t leaf_bytes = int64_t(leaf_kb) << 10;
      const int64_t P = (total / 2) / leaf_bytes;
      if (P < 32) continue;
      const int R = static_cast<int>(leaf_bytes / (16 * 256));
      for (int mode = 0; mode < 6; ++mode) {
        const int U = mode % 3 == 0 ? 2 : mode % 3 == 1 ? 4 : 8;
        const bool pf = mode >= 3;
        if (U > R) continue;
        const int64_t occ_cap = int64_t(sms) * 8;
        const unsigned grid = static_cast<unsigned>(P < occ_cap ? P : occ_cap);
        auto L = [&](int i) {
          const uint4* x = buf(i);
          const uint4* y = x + nvec / 2;
          if (!pf) {
            if (U == 2) leaf_kernel<2, false><<<grid, 256, 0, s>>>(x, y, R, P, sink);
            else if (U == 4) leaf_kernel<4, false><<<grid, 256, 0, s>>>(x, y, R, P, sink);
            else leaf_kernel<8, false><<<grid, 256, 0, s>>>(x, y, R, P, sink);
          } else {
            if (U == 2) leaf_kernel<2, true><<<grid, 256, 0, s>>>(x, y, R, P, sink);
            else if (U == 4) leaf_kernel<4, true><<<grid, 256, 0, s>>>(x, y, R, P, sink);
            else leaf_kernel<8, true><<<grid, 256, 0, s>>>(x, y, R, P, sink);
          }
        };
        float us = graph_us(L, reps, s);
        printf("leaf %3d KB/operand P=%5lld grid=%u U=%d pf=%d: %.2f us %.0f GB/s\n", leaf_kb,
               static_cast<long long>(P), grid, U, pf ? 1 : 0, us, total / us / 1e3);
      }
    }
    fflush(stdout);
  }
  CK(cudaGetLastError());
  return 0;
}
