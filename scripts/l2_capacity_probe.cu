// l2_capacity_probe.cu -- diagnostic (NOT product code): effective L2
// capacity seen by all 148 SMs reading one shared working set repeatedly.
// Read bandwidth per pass vs working-set size: the knee is where the set
// stops fitting (126 MB nominal; ~half if lines are duplicated per die).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/l2_capacity_probe scripts/l2_capacity_probe.cu
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void k_read(const float4* __restrict__ p, size_t n4, int passes, float* out) {
  float acc = 0.f;
  for (int it = 0; it < passes; ++it)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
         i += (size_t)gridDim.x * blockDim.x) {
      float4 v = __ldcg(p + i);
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 123.456f) *out = acc;
}

int main() {
  const size_t maxb = (size_t)512 << 20;
  float4* buf;
  float* out;
  cudaMalloc(&buf, maxb);
  cudaMalloc(&out, 4);
  cudaMemset(buf, 0, maxb);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t sizes_mb[] = {16, 32, 48, 56, 64, 72, 80, 96, 112, 128, 160, 256, 512};
  for (size_t mb : sizes_mb) {
    const size_t n4 = (mb << 20) / 16;
    const int passes = 20;
    k_read<<<sms * 8, 256>>>(buf, n4, 2, out);  // warm
    cudaEventRecord(a);
    k_read<<<sms * 8, 256>>>(buf, n4, passes, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("working set %4zu MB: %7.1f GB/s\n", mb, (double)(mb << 20) * passes / ms / 1e6);
  }
  return 0;
}
