// ubench.cu — design-space microbenchmarks (not product code) for the two
// HBM-bound hot kernels: column reductions of an f64 8192x8192 matrix
// (SURVEY cfg3 axis 0) and the transposing int16->f32 broadcast add (cfg2).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench scripts/ubench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}
__device__ __forceinline__ void dd_add(double& hi, double& lo, double v) {
  double s, e;
  two_sum(hi, v, s, e);
  hi = s;
  lo = __dadd_rn(lo, e);
}

// block per column, 8-B loads, U=8, 4 dd accumulators (the r01 kernel shape)
__global__ void __launch_bounds__(256) red_a(const double* x, double* out, int n, int ncol) {
  for (int col = blockIdx.x; col < ncol; col += gridDim.x) {
    const double* c = x + (size_t)col * n;
    double hi[4] = {0, 0, 0, 0}, lo[4] = {0, 0, 0, 0};
    for (int jb = threadIdx.x; jb < n; jb += 256 * 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcs(c + jb + u * 256);
#pragma unroll
      for (int u = 0; u < 8; ++u) dd_add(hi[u & 3], lo[u & 3], v[u]);
    }
    double s = hi[0] + hi[1] + hi[2] + hi[3] + lo[0] + lo[1] + lo[2] + lo[3];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
    __shared__ double sh[8];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0;
      for (int k = 0; k < 8; ++k) t += sh[k];
      out[col] = t;
    }
    __syncthreads();
  }
}

// block per column, 16-B loads (double2), 8 vectors per iteration, 4 dd accs
template <int U>
__global__ void __launch_bounds__(256) red_b(const double* x, double* out, int n, int ncol) {
  for (int col = blockIdx.x; col < ncol; col += gridDim.x) {
    const double2* c = (const double2*)(x + (size_t)col * n);
    const int n2 = n / 2;
    double hi[4] = {0, 0, 0, 0}, lo[4] = {0, 0, 0, 0};
    for (int jb = threadIdx.x; jb < n2; jb += 256 * U) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = jb + u * 256 < n2 ? __ldcs(c + jb + u * 256) : make_double2(0, 0);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        dd_add(hi[(2 * u) & 3], lo[(2 * u) & 3], v[u].x);
        dd_add(hi[(2 * u + 1) & 3], lo[(2 * u + 1) & 3], v[u].y);
      }
    }
    double s = hi[0] + hi[1] + hi[2] + hi[3] + lo[0] + lo[1] + lo[2] + lo[3];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
    __shared__ double sh[8];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0;
      for (int k = 0; k < 8; ++k) t += sh[k];
      out[col] = t;
    }
    __syncthreads();
  }
}

// plain double sum with 16-B loads (memory-bound reference)
__global__ void __launch_bounds__(256) red_c(const double* x, double* out, int n, int ncol) {
  for (int col = blockIdx.x; col < ncol; col += gridDim.x) {
    const double2* c = (const double2*)(x + (size_t)col * n);
    const int n2 = n / 2;
    double s0 = 0, s1 = 0;
    for (int jb = threadIdx.x; jb < n2; jb += 256 * 8) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcs(c + jb + u * 256);
#pragma unroll
      for (int u = 0; u < 8; ++u) { s0 += v[u].x; s1 += v[u].y; }
    }
    double s = s0 + s1;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
    __shared__ double sh[8];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0;
      for (int k = 0; k < 8; ++k) t += sh[k];
      out[col] = t;
    }
    __syncthreads();
  }
}

// axis-1 style: thread per row, strided columns (col-major; rows adjacent)
template <int U>
__global__ void __launch_bounds__(256) red_rows_strided(const double* x, double* out, int n,
                                                        int chunks) {
  // grid: (n/256 row-blocks) x chunks; partial per (row, chunk)
  const int row = blockIdx.x * 256 + threadIdx.x;
  const int per = n / chunks;
  const int c0 = blockIdx.y * per;
  double hi[2] = {0, 0}, lo[2] = {0, 0};
  for (int j = c0; j < c0 + per; j += U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(x + (size_t)(j + u) * n + row);
#pragma unroll
    for (int u = 0; u < U; ++u) dd_add(hi[u & 1], lo[u & 1], v[u]);
  }
  out[(size_t)blockIdx.y * n + row] = hi[0] + hi[1] + lo[0] + lo[1];
}

__global__ void copy_ref(const uint4* a, uint4* b, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}

// ---- cfg2: out[i0 + q*N] = float(X[q + (N-1-i0)*N]) + R[q], N = 4096
// (V = reversed transpose of column-major X; out column-major)
template <int TQ>
__global__ void __launch_bounds__(256) tile_f32(const int16_t* X, const float* R, float* out, int N) {
  // tile: 64 (i0) x TQ (q)
  __shared__ __align__(16) int16_t sm[TQ][64];
  const int nt0 = N / 64, ntq = N / TQ;
  for (int w = blockIdx.x; w < nt0 * ntq; w += gridDim.x) {
    const int t0 = w % nt0, tq = w / nt0;
    // phase 1: X rows (fixed V-row i0 = X column N-1-i0): TQ int16 contiguous
#pragma unroll
    for (int pass = 0; pass < TQ / 32; ++pass) {
      const int i0 = threadIdx.x % 64, c = threadIdx.x / 64 + 4 * pass;  // 16-B chunk index
      const int col = N - 1 - (t0 * 64 + i0);
      const uint4 v = __ldcs((const uint4*)(X + (size_t)col * N + tq * TQ) + c);
      const int16_t* e = (const int16_t*)&v;
#pragma unroll
      for (int j = 0; j < 8; ++j) sm[c * 8 + j][i0] = e[j];
    }
    __syncthreads();
#pragma unroll
    for (int pass = 0; pass < TQ / 16; ++pass) {
      const int ig = threadIdx.x % 16, qq = threadIdx.x / 16 + 16 * pass;
      const int q = tq * TQ + qq;
      const float r = __ldg(R + q);
      const uint2 raw = *(const uint2*)&sm[qq][ig * 4];
      const float f0 = (float)(int16_t)(raw.x & 0xffff) + r;
      const float f1 = (float)(int16_t)(raw.x >> 16) + r;
      const float f2 = (float)(int16_t)(raw.y & 0xffff) + r;
      const float f3 = (float)(int16_t)(raw.y >> 16) + r;
      __stcs((float4*)(out + (size_t)q * N + t0 * 64 + ig * 4), make_float4(f0, f1, f2, f3));
    }
    __syncthreads();
  }
}

// same, computing in double (the r01 semantics path)
__global__ void __launch_bounds__(256) tile_f64(const int16_t* X, const float* R, float* out, int N) {
  constexpr int TQ = 64;
  __shared__ __align__(16) int16_t sm[TQ][64];
  const int nt0 = N / 64, ntq = N / TQ;
  for (int w = blockIdx.x; w < nt0 * ntq; w += gridDim.x) {
    const int t0 = w % nt0, tq = w / nt0;
#pragma unroll
    for (int pass = 0; pass < TQ / 32; ++pass) {
      const int i0 = threadIdx.x % 64, c = threadIdx.x / 64 + 4 * pass;
      const int col = N - 1 - (t0 * 64 + i0);
      const uint4 v = __ldcs((const uint4*)(X + (size_t)col * N + tq * TQ) + c);
      const int16_t* e = (const int16_t*)&v;
#pragma unroll
      for (int j = 0; j < 8; ++j) sm[c * 8 + j][i0] = e[j];
    }
    __syncthreads();
#pragma unroll
    for (int pass = 0; pass < TQ / 16; ++pass) {
      const int ig = threadIdx.x % 16, qq = threadIdx.x / 16 + 16 * pass;
      const int q = tq * TQ + qq;
      const double r = __ldg(R + q);
      const uint2 raw = *(const uint2*)&sm[qq][ig * 4];
      const float f0 = __double2float_rn((double)(int16_t)(raw.x & 0xffff) + r);
      const float f1 = __double2float_rn((double)(int16_t)(raw.x >> 16) + r);
      const float f2 = __double2float_rn((double)(int16_t)(raw.y & 0xffff) + r);
      const float f3 = __double2float_rn((double)(int16_t)(raw.y >> 16) + r);
      __stcs((float4*)(out + (size_t)q * N + t0 * 64 + ig * 4), make_float4(f0, f1, f2, f3));
    }
    __syncthreads();
  }
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int n = 8192;
  const size_t nb = (size_t)n * n * 8;
  double* x;
  double* out;
  char* flush;
  CK(cudaMalloc(&x, nb));
  CK(cudaMalloc(&out, (size_t)n * 64 * 8));
  CK(cudaMalloc(&flush, 512 << 20));
  {
    std::vector<double> h((size_t)n * n);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)((i * 2654435761u) % 1000) * 1e-3;
    CK(cudaMemcpy(x, h.data(), nb, cudaMemcpyHostToDevice));
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, double bytes, auto launch) {
    float best = 1e9, sum = 0;
    for (int r = 0; r < 8; ++r) {
      cudaMemsetAsync(flush, r, 512 << 20);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 2) { best = ms < best ? ms : best; sum += ms; }
    }
    CK(cudaGetLastError());
    printf("%-44s best %8.4f ms  %8.1f GB/s   mean %8.1f GB/s\n", name, best, bytes / best / 1e6,
           bytes / (sum / 6) / 1e6);
  };
  timeit("copy_ref f64 536MB (r+w bytes)", 2.0 * nb, [&] {
    copy_ref<<<sms * 16, 256>>>((const uint4*)x, (uint4*)flush, (256u << 20) / 16);
  });
  timeit("red_a block/col ldg64 U8 dd4 grid=n", nb, [&] { red_a<<<n, 256>>>(x, out, n, n); });
  timeit("red_b<8> block/col ldg128 dd4 grid=n", nb, [&] { red_b<8><<<n, 256>>>(x, out, n, n); });
  timeit("red_b<4> block/col ldg128 dd4 grid=n", nb, [&] { red_b<4><<<n, 256>>>(x, out, n, n); });
  timeit("red_b<8> persistent grid=sms*8", nb, [&] { red_b<8><<<sms * 8, 256>>>(x, out, n, n); });
  timeit("red_b<16> block/col", nb, [&] { red_b<16><<<n, 256>>>(x, out, n, n); });
  timeit("red_c plain sum ldg128", nb, [&] { red_c<<<n, 256>>>(x, out, n, n); });
  timeit("red_rows_strided<8> chunks=32", nb, [&] {
    red_rows_strided<8><<<dim3(n / 256, 32), 256>>>(x, out, n, 32);
  });
  timeit("red_rows_strided<16> chunks=32", nb, [&] {
    red_rows_strided<16><<<dim3(n / 256, 32), 256>>>(x, out, n, 32);
  });
  timeit("red_rows_strided<8> chunks=64", nb, [&] {
    red_rows_strided<8><<<dim3(n / 256, 64), 256>>>(x, out, n, 64);
  });
  // cfg2
  const int N = 4096;
  int16_t* X;
  float* R;
  float* o;
  CK(cudaMalloc(&X, (size_t)N * N * 2));
  CK(cudaMalloc(&R, N * 4));
  CK(cudaMalloc(&o, (size_t)N * N * 4));
  CK(cudaMemset(X, 1, (size_t)N * N * 2));
  CK(cudaMemset(R, 0, N * 4));
  const double b2 = (double)N * N * 6 + N * 4;
  for (int per : {4, 8, 16}) {
    char name[64];
    snprintf(name, 64, "tile_f32<64> grid=sms*%d", per);
    timeit(name, b2, [&] { tile_f32<64><<<sms * per, 256>>>(X, R, o, N); });
  }
  timeit("tile_f32<128> grid=sms*8", b2, [&] { tile_f32<128><<<sms * 8, 256>>>(X, R, o, N); });
  timeit("tile_f32<128> grid=all tiles", b2, [&] { tile_f32<128><<<(N / 64) * (N / 128), 256>>>(X, R, o, N); });
  timeit("tile_f32<64> grid=all tiles", b2, [&] { tile_f32<64><<<(N / 64) * (N / 64), 256>>>(X, R, o, N); });
  timeit("tile_f64 grid=sms*8", b2, [&] { tile_f64<<<sms * 8, 256>>>(X, R, o, N); });
  timeit("tile_f64 grid=all tiles", b2, [&] { tile_f64<<<(N / 64) * (N / 64), 256>>>(X, R, o, N); });
  return 0;
}
