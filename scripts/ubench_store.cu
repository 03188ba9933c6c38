// ubench_store.cu — store-path microbenchmark (not product code): how fast
// can 64 MiB of float32 be written after an L2 flush, with st.global.v4
// (streaming / default) vs cp.async.bulk (bulk async smem->global, the
// TMA store path)?  Sizes = the cfg2 output.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ubench_store scripts/ubench_store.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr size_t NB = 64ull << 20;

__global__ void st_cs(float4* out, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(out + i, make_float4(1.f, 2.f, 3.f, (float)i));
}
__global__ void st_wb(float4* out, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = make_float4(1.f, 2.f, 3.f, (float)i);
}
// each block owns contiguous CH-byte chunks; smem staging buffer filled by
// threads, then one thread issues cp.async.bulk global<-shared
template <int CH>
__global__ void __launch_bounds__(256) st_bulk(char* out, size_t nch) {
  extern __shared__ __align__(128) char buf[];
  const int NBUF = 2;
  for (size_t c = blockIdx.x, it = 0; c < nch; c += gridDim.x, ++it) {
    char* b = buf + (it % NBUF) * CH;
    if (threadIdx.x == 0 && it >= NBUF)
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    for (int o = threadIdx.x * 16; o < CH; o += 256 * 16)
      *(float4*)(b + o) = make_float4(1.f, 2.f, 3.f, (float)o);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + c * CH),
                   "r"((uint32_t)__cvta_generic_to_shared(b)), "r"(CH) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__global__ void rd(const double* a, size_t n, double* sink) {
  double s = 0;
  for (size_t i = (size_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256) s += __ldcg(a + i);
  if (s == 12345.678) *sink = s;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  char *out, *flush, *clean;
  CK(cudaMalloc(&out, NB));
  CK(cudaMalloc(&flush, 256 << 20));
  CK(cudaMalloc(&clean, 256 << 20));
  CK(cudaMemset(clean, 0, 256 << 20));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch) {
    float best = 1e9;
    for (int r = 0; r < 15; ++r) {
      cudaMemsetAsync(flush, r, 256 << 20);
      rd<<<sms * 8, 256>>>((const double*)clean, (256 << 20) / 8, (double*)flush);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 3 && ms < best) best = ms;
    }
    printf("%-40s best %7.2f us  %8.1f GB/s  err=%s\n", name, best * 1e3, NB / best / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int g : {4, 8, 16})
    timeit(g == 4 ? "st.global.cs v4 grid sms*4" : g == 8 ? "st.global.cs v4 grid sms*8" : "st.global.cs v4 grid sms*16",
           [&] { st_cs<<<sms * g, 256>>>((float4*)out, NB / 16); });
  timeit("st.global (wb) v4 grid sms*8", [&] { st_wb<<<sms * 8, 256>>>((float4*)out, NB / 16); });
  cudaFuncSetAttribute(st_bulk<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 16384);
  cudaFuncSetAttribute(st_bulk<32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 32768);
  timeit("cp.async.bulk 16K chunks sms*4", [&] { st_bulk<16384><<<sms * 4, 256, 2 * 16384>>>(out, NB / 16384); });
  timeit("cp.async.bulk 16K chunks sms*6", [&] { st_bulk<16384><<<sms * 6, 256, 2 * 16384>>>(out, NB / 16384); });
  timeit("cp.async.bulk 32K chunks sms*3", [&] { st_bulk<32768><<<sms * 3, 256, 2 * 32768>>>(out, NB / 32768); });
  timeit("cudaMemsetAsync 64 MiB", [&] { cudaMemsetAsync(out, 7, NB); });
  return 0;
}
