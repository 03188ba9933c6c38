// ubench_rowred.cu — design-space microbenchmark (not product code) for the
// cfg3 axis-0 reduction: f64 (8192 x 8192) column-major, each output reduces
// one contiguous 64 KiB column.  Warp items (one warp per column, lanes read
// consecutive 16-B vectors, three rotating batches of U vectors), like
// k_red_rows_wv, with variants: cyclic vs blocked item assignment, warps per
// SM, and a variant that streams a warp's columns back to back without a
// pipeline refill between items.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_rowred scripts/ubench_rowred.cu
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

constexpr int64_t N = 8192;
constexpr int U = 4;

__device__ __forceinline__ double2 ldv(const double* p) {
  double2 r;
  asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ double warp_sum(double v) {
  for (int s = 16; s; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
  return v;
}

// V 0: per-item pipeline (refill per column), cyclic items
// V 1: per-item pipeline, blocked items (warp w gets columns [w*per, ...))
// V 2: continuous stream across the warp's blocked columns (no refill)
template <int V, int BPS>
__global__ void __launch_bounds__(256, BPS) rowred(const double* __restrict__ src, double* out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int64_t NV = N / 2;              // 16-B vectors per column
  constexpr int64_t NB = NV / (32 * U);      // batches per column (32)
  if (V < 2) {
    const int64_t per = (N + nw - 1) / nw;
    const int64_t o0 = V == 0 ? gw : gw * per, o1 = V == 0 ? N : min(N, o0 + per), st = V == 0 ? nw : 1;
    for (int64_t o = o0; o < o1; o += st) {
      const double* col = src + o * N;
      double a0 = 0, a1 = 0;
      double2 bA[U], bB[U], bC[U];
      auto ld = [&](double2(&b)[U], int64_t k) {
#pragma unroll
        for (int u = 0; u < U; ++u) b[u] = ldv(col + 2 * (lane + (k * U + u) * 32));
      };
      auto fold = [&](const double2(&b)[U]) {
#pragma unroll
        for (int u = 0; u < U; ++u) { a0 += b[u].x; a1 += b[u].y; }
      };
      ld(bA, 0);
      ld(bB, 1);
      int64_t k = 0;
      for (; k + 3 <= NB; k += 3) {
        if (k + 2 < NB) ld(bC, k + 2);
        fold(bA);
        if (k + 3 < NB) ld(bA, k + 3);
        fold(bB);
        if (k + 4 < NB) ld(bB, k + 4);
        fold(bC);
      }
      if (k < NB) fold(bA);
      if (k + 1 < NB) fold(bB);
      const double s = warp_sum(a0 + a1);
      if (lane == 0) out[o] = s;
    }
  } else {
    const int64_t per = (N + nw - 1) / nw;
    const int64_t o0 = gw * per, o1 = min(N, o0 + per);
    if (o0 >= o1) return;
    const int64_t total = (o1 - o0) * NB;  // batches in the warp's stream
    const double* base = src + o0 * N;
    double a0 = 0, a1 = 0;
    double2 bA[U], bB[U], bC[U];
    auto ld = [&](double2(&b)[U], int64_t g) {
      const int64_t o = g / NB, k = g - o * NB;
#pragma unroll
      for (int u = 0; u < U; ++u) b[u] = ldv(base + o * N + 2 * (lane + (k * U + u) * 32));
    };
    auto fold = [&](const double2(&b)[U], int64_t g) {
#pragma unroll
      for (int u = 0; u < U; ++u) { a0 += b[u].x; a1 += b[u].y; }
      if ((g + 1) % NB == 0) {
        const double s = warp_sum(a0 + a1);
        if (lane == 0) out[o0 + g / NB] = s;
        a0 = a1 = 0;
      }
    };
    ld(bA, 0);
    if (total > 1) ld(bB, 1);
    int64_t g = 0;
    for (; g + 3 <= total; g += 3) {
      if (g + 2 < total) ld(bC, g + 2);
      fold(bA, g);
      if (g + 3 < total) ld(bA, g + 3);
      fold(bB, g + 1);
      if (g + 4 < total) ld(bB, g + 4);
      fold(bC, g + 2);
    }
    if (g < total) fold(bA, g);
    if (g + 1 < total) fold(bB, g + 1);
  }
}

__global__ void flush_k(double* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = p[i] * 0.5 + 1.0;
}

template <int V, int BPS>
void run(const char* name, const double* src, double* out, double* fl, size_t nfl, int grid) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e9, tot = 0;
  const int reps = 12;
  for (int r = 0; r < reps + 3; ++r) {
    flush_k<<<1184, 512>>>(fl, nfl);
    CK(cudaEventRecord(a));
    rowred<V, BPS><<<grid, 256>>>(src, out);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (r >= 3) {
      best = ms < best ? ms : best;
      tot += ms;
    }
  }
  const double bytes = 8.0 * N * N;
  printf("%-44s grid %5d  best %7.2f us %7.1f GB/s  mean %7.2f us %7.1f GB/s\n", name, grid,
         best * 1e3, bytes / best / 1e6, tot / reps * 1e3, bytes / (tot / reps) / 1e6);
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double *src, *out, *fl;
  const size_t nfl = (256u << 20) / 8;
  CK(cudaMalloc(&src, 8 * N * N));
  CK(cudaMalloc(&out, 8 * N));
  CK(cudaMalloc(&fl, nfl * 8));
  CK(cudaMemset(src, 0x3f, 8 * N * N));
  CK(cudaMemset(fl, 0, nfl * 8));
  run<0, 2>("cyclic items, 2 blocks/SM", src, out, fl, nfl, sms * 2);
  run<1, 2>("blocked items, 2 blocks/SM", src, out, fl, nfl, sms * 2);
  run<2, 2>("continuous stream, 2 blocks/SM", src, out, fl, nfl, sms * 2);
  run<0, 4>("cyclic items, 4 blocks/SM", src, out, fl, nfl, sms * 4);
  run<2, 4>("continuous stream, 4 blocks/SM", src, out, fl, nfl, sms * 4);
  run<0, 2>("cyclic items, 1024 warps (one item each x8)", src, out, fl, nfl, 128);
  run<0, 4>("cyclic items, 8192 warps (one item each)", src, out, fl, nfl, 1024);
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
