// ubench_colred.cu — design-space microbenchmark (not product code) for the
// cfg3 axis-1 reduction: f64 (8192 x 8192) column-major, reduce over the
// strided axis, outputs adjacent (k_red_cols_v's layout).  Each thread owns
// two adjacent outputs (one 16-B vector per row); a block covers NT*2
// outputs x one row chunk and writes 16-B partials chunk-major.  Variants
// compare the fold of the extreme (fmax vs compare-select vs two chains)
// against the compensated sum under the same streaming.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_colred scripts/ubench_colred.cu
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

__device__ __forceinline__ void dd_add(double& hi, double& lo, double v) {
  const double s = hi + v, bp = s - hi;
  lo += (hi - (s - bp)) + (v - bp);
  hi = s;
}
__device__ __forceinline__ double2 ldv(const char* p) {
  double2 r;
  asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

// V: 0 sum (dd), 1 fmax, 2 compare-select (v > m), 3 fmax on two chains,
//    4 fmax with 4-row batches x 4 in flight (deeper)
template <int V, int NT, int U>
__global__ void __launch_bounds__(NT, 512 / NT) colred(const char* __restrict__ src, int64_t chunk,
                                                       int64_t nob, double2* ws) {
  const int64_t nwork = nob * ((N + chunk - 1) / chunk);
  for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int64_t ob = w % nob, c = w / nob;
    const int64_t o = (ob * NT + threadIdx.x) * 2;
    const int64_t j0 = c * chunk, j1 = min(N, j0 + chunk);
    const int64_t s0 = N * 8;
    const char* ptr = src + o * 8 + j0 * s0;
    double a0 = V == 0 ? 0.0 : -INFINITY, a1 = a0, l0 = 0.0, l1 = 0.0;
    double b0 = a0, b1 = a0;
    const int64_t nfull = (j1 - j0) / U;
    double2 bA[U], bB[U], bC[U];
    auto ld = [&](double2(&b)[U], int64_t k) {
#pragma unroll
      for (int u = 0; u < U; ++u) b[u] = ldv(ptr + (k * U + u) * s0);
    };
    auto fold = [&](const double2(&b)[U]) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double x = b[u].x, y = b[u].y;
        if (V == 0) {
          dd_add(a0, l0, x);
          dd_add(a1, l1, y);
        } else if (V == 1 || V == 4) {
          a0 = fmax(a0, x);
          a1 = fmax(a1, y);
        } else if (V == 2) {
          a0 = x > a0 ? x : a0;
          a1 = y > a1 ? y : a1;
        } else {
          if (u & 1) {
            b0 = fmax(b0, x);
            b1 = fmax(b1, y);
          } else {
            a0 = fmax(a0, x);
            a1 = fmax(a1, y);
          }
        }
      }
    };
    if (nfull > 0) ld(bA, 0);
    if (nfull > 1) ld(bB, 1);
    int64_t k = 0;
    for (; k + 3 <= nfull; k += 3) {
      if (k + 2 < nfull) ld(bC, k + 2);
      fold(bA);
      if (k + 3 < nfull) ld(bA, k + 3);
      fold(bB);
      if (k + 4 < nfull) ld(bB, k + 4);
      fold(bC);
    }
    if (k < nfull) fold(bA);
    if (k + 1 < nfull) fold(bB);
    if (V == 3) {
      a0 = fmax(a0, b0);
      a1 = fmax(a1, b1);
    }
    const int64_t O = N;
    ws[c * O + o] = make_double2(a0, l0);
    ws[c * O + o + 1] = make_double2(a1, l1);
  }
}

__global__ void flush_k(double* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = p[i] * 0.5 + 1.0;
}

template <int V, int NT, int U>
void run(const char* name, const char* src, double2* ws, double* fl, size_t nfl, int sms, int C) {
  const int64_t nob = N / (NT * 2);
  const int64_t chunk = (N + C - 1) / C;
  const int64_t work = nob * ((N + chunk - 1) / chunk);
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e9, tot = 0;
  const int reps = 12;
  for (int r = 0; r < reps + 3; ++r) {
    flush_k<<<sms * 4, 512>>>(fl, nfl);
    CK(cudaEventRecord(a));
    colred<V, NT, U><<<(int)work, NT>>>(src, chunk, nob, ws);
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
  printf("%-40s C=%3d grid %6lld  best %7.2f us %7.1f GB/s  mean %7.2f us %7.1f GB/s\n", name, C,
         (long long)work, best * 1e3, bytes / best / 1e6, tot / reps * 1e3, bytes / (tot / reps) / 1e6);
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  char* src;
  double2* ws;
  double* fl;
  const size_t nfl = (256u << 20) / 8;
  CK(cudaMalloc(&src, 8 * N * N));
  CK(cudaMalloc(&ws, 16 * N * 128));
  CK(cudaMalloc(&fl, nfl * 8));
  CK(cudaMemset(src, 0x3f, 8 * N * N));
  CK(cudaMemset(fl, 0, nfl * 8));
  for (int C : {32, 64, 128}) {
    run<0, 64, 4>("sum dd   NT64 U4", src, ws, fl, nfl, sms, C);
    run<1, 64, 4>("max fmax NT64 U4", src, ws, fl, nfl, sms, C);
    run<2, 64, 4>("max sel  NT64 U4", src, ws, fl, nfl, sms, C);
    run<3, 64, 4>("max 2ch  NT64 U4", src, ws, fl, nfl, sms, C);
    run<1, 64, 8>("max fmax NT64 U8", src, ws, fl, nfl, sms, C);
    run<1, 128, 4>("max fmax NT128 U4", src, ws, fl, nfl, sms, C);
    run<0, 128, 4>("sum dd   NT128 U4", src, ws, fl, nfl, sms, C);
  }
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
