// ubench_read.cu — read-only HBM ceiling (NOT product code): how fast can a
// kernel stream 512 MiB (cfg3's 8192^2 f64 matrix) through the SMs?  Rotates
// over 2 buffers (> L2), K launches per event pair.  Variants: grid-stride
// 16-B loads with U loads in flight per thread, 8 / 16 / 32 resident warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ubench_read scripts/ubench_read.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

template <int U>
__global__ void __launch_bounds__(256) k_read(const uint4* __restrict__ a, size_t n, unsigned* sink) {
  unsigned acc = 0;
  const size_t stride = (size_t)gridDim.x * 256 * U;
  for (size_t i = (size_t)blockIdx.x * 256 * U + threadIdx.x; i < n; i += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(a + i + u * 256);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

// double sum with the same access pattern (the FP64 add pipe in the loop)
template <int U>
__global__ void __launch_bounds__(256) k_sum(const double2* __restrict__ a, size_t n, double* out) {
  double s0 = 0, s1 = 0;
  const size_t stride = (size_t)gridDim.x * 256 * U;
  for (size_t i = (size_t)blockIdx.x * 256 * U + threadIdx.x; i < n; i += stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(a + i + u * 256);
#pragma unroll
    for (int u = 0; u < U; ++u) { s0 += v[u].x; s1 += v[u].y; }
  }
  if (s0 + s1 == 1234.5) *out = s0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t bytes = (size_t)8192 * 8192 * 8;
  void* buf[2];
  for (int r = 0; r < 2; ++r) {
    CK(cudaMalloc(&buf[r], bytes));
    CK(cudaMemset(buf[r], r + 1, bytes));
  }
  unsigned* sink;
  CK(cudaMalloc(&sink, 64));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch) {
    for (int r = 0; r < 4; ++r) launch(r % 2);
    CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      for (int k = 0; k < 20; ++k) launch(k % 2);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms / 20 < best ? ms / 20 : best;
    }
    CK(cudaGetLastError());
    printf("%-44s %8.2f us %8.1f GB/s\n", name, best * 1e3, bytes / best / 1e6);
    fflush(stdout);
  };
  const size_t n16 = bytes / 16;
  for (int mult : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, sizeof nm, "xor-read U=4 grid=sms*%d", mult);
    timeit(nm, [&](int r) { k_read<4><<<sms * mult, 256>>>((const uint4*)buf[r], n16, sink); });
    snprintf(nm, sizeof nm, "xor-read U=8 grid=sms*%d", mult);
    timeit(nm, [&](int r) { k_read<8><<<sms * mult, 256>>>((const uint4*)buf[r], n16, sink); });
    snprintf(nm, sizeof nm, "f64 sum U=4 grid=sms*%d", mult);
    timeit(nm, [&](int r) { k_sum<4><<<sms * mult, 256>>>((const double2*)buf[r], n16, (double*)sink); });
  }
  timeit("xor-read U=1 one 16-B load per thread", [&](int r) {
    k_read<1><<<(unsigned)(n16 / 256), 256>>>((const uint4*)buf[r], n16, sink);
  });
  return 0;
}
