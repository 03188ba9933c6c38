// ubench_tile_rot.cu — design-space microbenchmark (NOT product code) for the
// cfg2 transposing int16 -> f32 broadcast add under the bench's steady-state
// methodology (back-to-back launches rotating over 4 input/output sets,
// 4 x 100.7 MB > 126 MB L2, one event pair around K launches):
//   out[i + j*N] = float(X[j + (N-1-i)*N]) + R[j],  N = 4096
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/ubench_tile_rot scripts/ubench_tile_rot.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

#include "../include/tidepool_gpu.h"

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

constexpr int N = 4096;
constexpr int ROT = 4;

// TI x TJ tile (i = output row = fast axis of out; j = output column = fast
// axis of X).  Phase 1: each lane loads 16 B (8 int16 along j) of one X
// column segment, converts, adds R[j], writes sm[j][i ^ swz].  Phase 2:
// float4 along i per lane -> 16-B coalesced stores of output columns.
// ORDER 0: i-tiles fastest across the work index (write locality);
// ORDER 1: j-tiles fastest.  DYN: work items claimed from an atomic counter.
template <int TI, int TJ, int MINB, int ORDER, int DYN, int PF>
__global__ void __launch_bounds__(256, MINB)
    k_var(const int16_t* __restrict__ X, const float* __restrict__ R, float* __restrict__ out,
          int* counter) {
  constexpr int LPR = TJ * 2 / 16;   // lanes per i-row segment
  constexpr int RPW = 32 / LPR;      // i-rows per warp load
  constexpr int NLD = TI / (8 * RPW);
  constexpr int SWM = RPW > 4 ? RPW : 4;
  static_assert(NLD >= 1, "tile too small");
  __shared__ __align__(16) float sm[TJ][TI];
  __shared__ int next_w;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane % LPR;
  const int r0 = warp * RPW + lane / LPR;
  const int swz1 = (c * SWM) & 31;
  constexpr int nti = N / TI, ntj = N / TJ;
  const int nwork = nti * ntj;
  uint4 xb[PF][NLD];
  float yr[PF][8];
  auto tile_of = [&](int w, int& ti, int& tj) {
    if (ORDER == 0) { ti = w % nti; tj = w / nti; }
    else if (ORDER == 1) { tj = w % ntj; ti = w / ntj; }
    else {  // grouped raster: ORDER consecutive i-tiles, then the next j-tile
      const int g = w / (ORDER * ntj), r = w % (ORDER * ntj);
      ti = g * ORDER + r % ORDER;
      tj = r / ORDER;
    }
  };
  auto load = [&](int w, int s) {
    int ti, tj;
    tile_of(w, ti, tj);
#pragma unroll
    for (int l = 0; l < NLD; ++l) {
      const int i = ti * TI + r0 + l * 8 * RPW;
      xb[s][l] = __ldcs((const uint4*)(X + (size_t)(N - 1 - i) * N + tj * TJ) + c);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) yr[s][k] = __ldg(R + tj * TJ + c * 8 + k);
  };
  int w = blockIdx.x;
  if (DYN) {
    if (threadIdx.x == 0) next_w = atomicAdd(counter, 1) + gridDim.x;
  }
  int wq[PF];
  wq[0] = w;
#pragma unroll
  for (int s = 1; s < PF; ++s) wq[s] = wq[s - 1] + gridDim.x;
  if (DYN && PF > 1) {
    __syncthreads();
    // (PF > 1 with DYN not used)
  }
#pragma unroll
  for (int s = 0; s < PF; ++s)
    if (wq[s] < nwork) load(wq[s], s);
  int slot = 0;
  while (w < nwork) {
    int ti, tj;
    tile_of(w, ti, tj);
#pragma unroll
    for (int l = 0; l < NLD; ++l) {
      const int i = r0 + l * 8 * RPW;
      const int16_t* e = (const int16_t*)&xb[slot][l];
#pragma unroll
      for (int k = 0; k < 8; ++k) sm[c * 8 + k][i ^ swz1] = (float)e[k] + yr[slot][k];
    }
    int wn;
    if (DYN) {
      __syncthreads();
      wn = next_w;
      __syncthreads();
      if (threadIdx.x == 0) next_w = atomicAdd(counter, 1) + gridDim.x;
    } else {
      __syncthreads();
      wn = w + PF * gridDim.x;
    }
    if (wn < nwork) load(wn, slot);
    constexpr int TPC = TI / 4;          // threads per output column
    constexpr int CPP = 256 / TPC;       // columns per pass
    const int ig = threadIdx.x % TPC;
#pragma unroll
    for (int pass = 0; pass < TJ / CPP; ++pass) {
      const int j = threadIdx.x / TPC + CPP * pass;
      const int swz = ((j / 8) * SWM) & 31;
      const float4 f = *(const float4*)&sm[j][(ig * 4) ^ swz];
      __stcs((float4*)(out + (size_t)(tj * TJ + j) * N + ti * TI + ig * 4), f);
    }
    __syncthreads();
    if (DYN) {
      w = wn;
    } else {
      w += gridDim.x;
      slot = (slot + 1) % PF;
    }
  }
}

__global__ void k_contig(const int16_t* __restrict__ X, float* __restrict__ out, size_t n8) {
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n8;
       t += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldcs((const uint4*)X + t);
    const int16_t* e = (const int16_t*)&v;
    __stcs((float4*)out + 2 * t, make_float4(e[0], e[1], e[2], e[3]));
    __stcs((float4*)out + 2 * t + 1, make_float4(e[4], e[5], e[6], e[7]));
  }
}

// one 8-element chunk per thread, no grid-stride loop (the product k_contig shape)
__global__ void k_contig1(const int16_t* __restrict__ X, float* __restrict__ out) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const uint4 v = __ldcs((const uint4*)X + t);
  const int16_t* e = (const int16_t*)&v;
  __stcs((float4*)out + 2 * t, make_float4(e[0], e[1], e[2], e[3]));
  __stcs((float4*)out + 2 * t + 1, make_float4(e[4], e[5], e[6], e[7]));
}

// grid-stride contiguous cast with a configurable number of resident threads
// (memory-level concurrency sweep); DBL: convert through double like the
// product's Tier-A path (I2F.F64), which lowers the issue rate
template <int DBL>
__global__ void __launch_bounds__(256) k_contig_gs(const int16_t* __restrict__ X,
                                                   float* __restrict__ out, size_t n8) {
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n8;
       t += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldcs((const uint4*)X + t);
    const int16_t* e = (const int16_t*)&v;
    float f[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = DBL ? (float)(double)(long long)e[k] : (float)e[k];
    __stcs((float4*)out + 2 * t, make_float4(f[0], f[1], f[2], f[3]));
    __stcs((float4*)out + 2 * t + 1, make_float4(f[4], f[5], f[6], f[7]));
  }
}

// one chunk per thread, double conversion (the product's instruction mix)
__global__ void k_contig1d(const int16_t* __restrict__ X, float* __restrict__ out) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const uint4 v = __ldcs((const uint4*)X + t);
  const int16_t* e = (const int16_t*)&v;
  float f[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) f[k] = (float)(double)(long long)e[k];
  __stcs((float4*)out + 2 * t, make_float4(f[0], f[1], f[2], f[3]));
  __stcs((float4*)out + 2 * t + 1, make_float4(f[4], f[5], f[6], f[7]));
}

// column-streaming order: block b owns output column group tj = b % ntj and
// walks SPAN consecutive i-tiles of it (each block writes SPAN*TI*4
// contiguous bytes per output column, sequentially), next tile prefetched
template <int TI, int TJ, int MINB, int SPAN>
__global__ void __launch_bounds__(256, MINB)
    k_cols(const int16_t* __restrict__ X, const float* __restrict__ R, float* __restrict__ out) {
  constexpr int LPR = TJ * 2 / 16, RPW = 32 / LPR, NLD = TI / (8 * RPW);
  constexpr int SWM = RPW > 4 ? RPW : 4;
  constexpr int ntj = N / TJ;
  __shared__ __align__(16) float sm[TJ][TI];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane % LPR, r0 = warp * RPW + lane / LPR;
  const int swz1 = (c * SWM) & 31;
  const int tj = blockIdx.x % ntj, ti0 = (blockIdx.x / ntj) * SPAN;
  float yr[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) yr[k] = __ldg(R + tj * TJ + c * 8 + k);
  uint4 xb[NLD];
  auto load = [&](int ti) {
#pragma unroll
    for (int l = 0; l < NLD; ++l) {
      const int i = ti * TI + r0 + l * 8 * RPW;
      xb[l] = __ldcs((const uint4*)(X + (size_t)(N - 1 - i) * N + tj * TJ) + c);
    }
  };
  load(ti0);
  for (int s = 0; s < SPAN; ++s) {
    const int ti = ti0 + s;
#pragma unroll
    for (int l = 0; l < NLD; ++l) {
      const int i = r0 + l * 8 * RPW;
      const int16_t* e = (const int16_t*)&xb[l];
#pragma unroll
      for (int k = 0; k < 8; ++k) sm[c * 8 + k][i ^ swz1] = (float)e[k] + yr[k];
    }
    __syncthreads();
    if (s + 1 < SPAN) load(ti + 1);
    constexpr int TPC = TI / 4, CPP = 256 / TPC;
    const int ig = threadIdx.x % TPC;
#pragma unroll
    for (int pass = 0; pass < TJ / CPP; ++pass) {
      const int j = threadIdx.x / TPC + CPP * pass;
      const int swz = ((j / 8) * SWM) & 31;
      const float4 f = *(const float4*)&sm[j][(ig * 4) ^ swz];
      __stcs((float4*)(out + (size_t)(tj * TJ + j) * N + ti * TI + ig * 4), f);
    }
    __syncthreads();
  }
}

// strip kernel: block = TJ consecutive output columns (contiguous TJ*16 KiB
// of the output) x IH consecutive rows.  Phase A: the X segments (TJ int16
// = TJ*2 B per X column, IH X columns) -> smem int16 [IH][TJ] (padded);
// phase B: the block writes its columns one after another, each warp
// instruction 512 B contiguous (a single sequential write stream per block).
template <int TJ, int IH, int MINB>
__global__ void __launch_bounds__(256, MINB)
    k_strip(const int16_t* __restrict__ X, const float* __restrict__ R, float* __restrict__ out) {
  constexpr int PAD = 2;                       // int16 of padding per smem row
  constexpr int ROW = TJ + PAD;
  extern __shared__ __align__(16) int16_t ssm[];
  constexpr int NIH = N / IH;
  const int sj = blockIdx.x / NIH, ih = blockIdx.x % NIH;
  const int j0 = sj * TJ, i0 = ih * IH;
  // phase A: lanes load 4 B (2 int16) each; TJ/2 lanes per X column segment
  constexpr int LPS = TJ / 2;
  for (int t = threadIdx.x; t < IH * LPS; t += 256) {
    const int ii = t / LPS, q = t % LPS;
    const int i = i0 + ii;
    const uint32_t v = __ldcs((const uint32_t*)(X + (size_t)(N - 1 - i) * N + j0) + q);
    *(uint32_t*)&ssm[ii * ROW + 2 * q] = v;   // ROW even -> 4-B aligned
  }
  __syncthreads();
  // phase B: column by column; thread handles 4 consecutive i (float4)
  for (int jj = 0; jj < TJ; ++jj) {
    const float r = __ldg(R + j0 + jj);
    float* col = out + (size_t)(j0 + jj) * N + i0;
    for (int t = threadIdx.x; t < IH / 4; t += 256) {
      const int ii = 4 * t;
      float4 f;
      f.x = (float)ssm[(ii + 0) * ROW + jj] + r;
      f.y = (float)ssm[(ii + 1) * ROW + jj] + r;
      f.z = (float)ssm[(ii + 2) * ROW + jj] + r;
      f.w = (float)ssm[(ii + 3) * ROW + jj] + r;
      __stcs((float4*)(col + ii), f);
    }
  }
}

// full-sector stores: each warp store instruction covers 512 contiguous
// bytes (lane l: 4 int16 in, one float4 out), U independent chunks per thread
template <int U>
__global__ void __launch_bounds__(256) k_contig2(const int16_t* __restrict__ X,
                                                 float* __restrict__ out) {
  const size_t base = (size_t)blockIdx.x * 256 * U + threadIdx.x;
  uint2 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = __ldcs((const uint2*)X + base + u * 256);
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int16_t* e = (const int16_t*)&v[u];
    __stcs((float4*)out + base + u * 256, make_float4(e[0], e[1], e[2], e[3]));
  }
}

// reads in the cfg2 tile pattern (64 x 128-B X segments per 64x64 tile),
// writes contiguous (each tile's 4096 floats to a contiguous 16 KiB block)
__global__ void __launch_bounds__(256) k_tread(const int16_t* __restrict__ X,
                                               float* __restrict__ out) {
  const int w = blockIdx.x, ti = w % 64, tj = w / 64;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane % 8, r0 = warp * 4 + lane / 8;
#pragma unroll
  for (int l = 0; l < 2; ++l) {
    const int i = ti * 64 + r0 + l * 32;
    const uint4 v = __ldcs((const uint4*)(X + (size_t)(N - 1 - i) * N + tj * 64) + c);
    const int16_t* e = (const int16_t*)&v;
    float* o = out + (size_t)w * 4096 + (r0 + l * 32) * 64 + c * 8;
    __stcs((float4*)o, make_float4(e[0], e[1], e[2], e[3]));
    __stcs((float4*)o + 1, make_float4(e[4], e[5], e[6], e[7]));
  }
}

// tile-pattern reads with full-sector contiguous writes: a warp's 32 lanes
// each hold 4 int16 of one 128-B X segment half... lane l loads 8 B (4 j's)
// of row i = l / 16 (2 rows x 16 lanes per instruction), writes 16 B
// contiguous: the warp writes 512 B contiguous per instruction
__global__ void __launch_bounds__(256) k_tread2(const int16_t* __restrict__ X,
                                                float* __restrict__ out) {
  const int w = blockIdx.x, ti = w % 64, tj = w / 64;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const int row = warp * 8 + l * 2 + lane / 16;       // 0..63
    const int i = ti * 64 + row;
    const uint2 v = __ldcs((const uint2*)(X + (size_t)(N - 1 - i) * N + tj * 64) + (lane % 16));
    const int16_t* e = (const int16_t*)&v;
    float* o = out + (size_t)w * 4096 + row * 64 + (lane % 16) * 4;
    __stcs((float4*)o, make_float4(e[0], e[1], e[2], e[3]));
  }
}

// k_twrite with a padded output leading dimension LD (floats): does the
// 16-KiB column stride alias the write pattern onto few memory channels?
template <int LD>
__global__ void __launch_bounds__(256) k_twrite_ld(const int16_t* __restrict__ X,
                                                   float* __restrict__ out) {
  const int w = blockIdx.x, ti = w % 64, tj = w / 64;
  const int ig = threadIdx.x % 16;
#pragma unroll
  for (int pass = 0; pass < 4; ++pass) {
    const int j = threadIdx.x / 16 + 16 * pass;
    const uint2 v = __ldcs((const uint2*)(X + (size_t)w * 4096 + j * 64 + ig * 4));
    const int16_t* e = (const int16_t*)&v;
    __stcs((float4*)(out + (size_t)(tj * 64 + j) * LD + ti * 64 + ig * 4),
           make_float4(e[0], e[1], e[2], e[3]));
  }
}

// write-side shape sweep: each block writes NC output columns x SEG floats
// (SEG * NC = 4096 elements, contiguous reads); block w covers column group
// w / (N / SEG) and row segment w % (N / SEG)
template <int SEG, int NC>
__global__ void __launch_bounds__(256) k_wshape(const int16_t* __restrict__ X,
                                                float* __restrict__ out) {
  const int w = blockIdx.x, ns = N / SEG;
  const int ts = w % ns, tc = w / ns;
  for (int e = threadIdx.x * 4; e < 4096; e += 1024) {
    const int j = e / SEG, i = e % SEG;
    const uint2 v = __ldcs((const uint2*)(X + (size_t)w * 4096 + e));
    const int16_t* q = (const int16_t*)&v;
    __stcs((float4*)(out + (size_t)(tc * NC + j) * N + ts * SEG + i),
           make_float4(q[0], q[1], q[2], q[3]));
  }
}

// k_wshape with all of a thread's loads issued before its stores
template <int SEG, int NC>
__global__ void __launch_bounds__(256) k_wshape_u(const int16_t* __restrict__ X,
                                                  float* __restrict__ out) {
  const int w = blockIdx.x, ns = N / SEG;
  const int ts = w % ns, tc = w / ns;
  uint2 v[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = __ldcs((const uint2*)(X + (size_t)w * 4096 + threadIdx.x * 4 + k * 1024));
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int e = threadIdx.x * 4 + k * 1024;
    const int j = e / SEG, i = e % SEG;
    const int16_t* q = (const int16_t*)&v[k];
    __stcs((float4*)(out + (size_t)(tc * NC + j) * N + ts * SEG + i),
           make_float4(q[0], q[1], q[2], q[3]));
  }
}

// tile-pattern reads (64 X columns x 128 B) issued all before any store,
// contiguous full-sector writes: the read side with full memory-level
// parallelism
__global__ void __launch_bounds__(256) k_tread_u(const int16_t* __restrict__ X,
                                                 float* __restrict__ out) {
  const int w = blockIdx.x, ti = w % 64, tj = w / 64;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane % 8, r0 = warp * 4 + lane / 8;
  uint4 v[2];
#pragma unroll
  for (int l = 0; l < 2; ++l)
    v[l] = __ldcs((const uint4*)(X + (size_t)(N - 1 - (ti * 64 + r0 + l * 32)) * N + tj * 64) + c);
#pragma unroll
  for (int l = 0; l < 2; ++l) {
    const int16_t* e = (const int16_t*)&v[l];
    // 8 lanes x 2 float4 = 256 B contiguous per row; rows of a warp adjacent
    float* o = out + (size_t)w * 4096 + (r0 + l * 32) * 64 + c * 8;
    __stcs((float4*)o, make_float4(e[0], e[1], e[2], e[3]));
    __stcs((float4*)o + 1, make_float4(e[4], e[5], e[6], e[7]));
  }
}

// the full cfg2 tile op, one tile per block, 8 blocks / SM (32 regs),
// loads issued first; smem transpose; tile-pattern writes
__global__ void __launch_bounds__(256, 8) k_tile_hi(const int16_t* __restrict__ X,
                                                    const float* __restrict__ R,
                                                    float* __restrict__ out) {
  __shared__ __align__(16) float sm[64][64];
  const int w = blockIdx.x, ti = w % 64, tj = w / 64;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane % 8, r0 = warp * 4 + lane / 8;
  const int swz1 = (c * 4) & 31;
  uint4 v[2];
#pragma unroll
  for (int l = 0; l < 2; ++l)
    v[l] = __ldcs((const uint4*)(X + (size_t)(N - 1 - (ti * 64 + r0 + l * 32)) * N + tj * 64) + c);
  float y[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) y[k] = __ldg(R + tj * 64 + c * 8 + k);
#pragma unroll
  for (int l = 0; l < 2; ++l) {
    const int16_t* e = (const int16_t*)&v[l];
#pragma unroll
    for (int k = 0; k < 8; ++k) sm[c * 8 + k][(r0 + l * 32) ^ swz1] = (float)e[k] + y[k];
  }
  __syncthreads();
  const int ig = threadIdx.x % 16;
#pragma unroll
  for (int pass = 0; pass < 4; ++pass) {
    const int j = threadIdx.x / 16 + 16 * pass;
    const int swz = ((j / 8) * 4) & 31;
    const float4 f = *(const float4*)&sm[j][(ig * 4) ^ swz];
    __stcs((float4*)(out + (size_t)(tj * 64 + j) * N + ti * 64 + ig * 4), f);
  }
}

// the full cfg2 op with T tiles per block (adjacent i-tiles of one column
// group), ALL 2*T loads of a thread issued before any conversion: 32*T
// bytes in flight per thread; smem T x 16 KiB
template <int T, int MINB>
__global__ void __launch_bounds__(256, MINB) k_tile_mt(const int16_t* __restrict__ X,
                                                       const float* __restrict__ R,
                                                       float* __restrict__ out) {
  extern __shared__ __align__(16) float smt[];
  const int w0 = blockIdx.x * T;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane % 8, r0 = warp * 4 + lane / 8;
  const int swz1 = (c * 4) & 31;
  uint4 v[T][2];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int w = w0 + t, ti = w % 64, tj = w / 64;
#pragma unroll
    for (int l = 0; l < 2; ++l)
      v[t][l] = __ldcs((const uint4*)(X + (size_t)(N - 1 - (ti * 64 + r0 + l * 32)) * N + tj * 64) + c);
  }
  const int tj0 = w0 / 64;
  float y[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) y[k] = __ldg(R + tj0 * 64 + c * 8 + k);
#pragma unroll
  for (int t = 0; t < T; ++t) {
    float(*sm)[64] = (float(*)[64])(smt + t * 4096);
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      const int16_t* e = (const int16_t*)&v[t][l];
#pragma unroll
      for (int k = 0; k < 8; ++k) sm[c * 8 + k][(r0 + l * 32) ^ swz1] = (float)e[k] + y[k];
    }
  }
  __syncthreads();
  const int ig = threadIdx.x % 16;
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int w = w0 + t, ti = w % 64, tj = w / 64;
    float(*sm)[64] = (float(*)[64])(smt + t * 4096);
#pragma unroll
    for (int pass = 0; pass < 4; ++pass) {
      const int j = threadIdx.x / 16 + 16 * pass;
      const int swz = ((j / 8) * 4) & 31;
      const float4 f = *(const float4*)&sm[j][(ig * 4) ^ swz];
      __stcs((float4*)(out + (size_t)(tj * 64 + j) * N + ti * 64 + ig * 4), f);
    }
  }
}

// tile-pattern reads (hoisted) with X column stride LDX int16, contiguous
// full-sector writes: read-side aliasing check
template <int LDX>
__global__ void __launch_bounds__(256) k_tread_ld(const int16_t* __restrict__ X,
                                                  float* __restrict__ out) {
  const int w = blockIdx.x, ti = w % 64, tj = w / 64;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane % 8, r0 = warp * 4 + lane / 8;
  uint4 v[2];
#pragma unroll
  for (int l = 0; l < 2; ++l)
    v[l] = __ldcs((const uint4*)(X + (size_t)(N - 1 - (ti * 64 + r0 + l * 32)) * LDX + tj * 64) + c);
#pragma unroll
  for (int l = 0; l < 2; ++l) {
    const int16_t* e = (const int16_t*)&v[l];
    float* o = out + (size_t)w * 4096 + (r0 + l * 32) * 64 + c * 8;
    __stcs((float4*)o, make_float4(e[0], e[1], e[2], e[3]));
    __stcs((float4*)o + 1, make_float4(e[4], e[5], e[6], e[7]));
  }
}

// tile-pattern reads (8-B loads, 16 lanes per 128-B X segment, all 4
// issued first) + one 16-B store per lane, 512 contiguous bytes per warp
// instruction: the read side alone
__global__ void __launch_bounds__(256) k_tread3(const int16_t* __restrict__ X,
                                                float* __restrict__ out) {
  const int w = blockIdx.x, ti = w % 64, tj = w / 64;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint2 v[4];
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const int row = warp * 8 + l * 2 + lane / 16;
    v[l] = __ldcs((const uint2*)(X + (size_t)(N - 1 - (ti * 64 + row)) * N + tj * 64) + (lane % 16));
  }
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const int row = warp * 8 + l * 2 + lane / 16;
    const int16_t* e = (const int16_t*)&v[l];
    __stcs((float4*)(out + (size_t)w * 4096 + row * 64 + (lane % 16) * 4),
           make_float4(e[0], e[1], e[2], e[3]));
  }
}

// the full cfg2 op (k_tile_hi shape) with an L2 sector-promotion hint on
// the X loads: PROMO 0 = ld.global.cs, 1 = L2::128B, 2 = L2::256B; ORD as k_var
__device__ __forceinline__ uint4 ld_promo(const void* p, int promo) {
  uint4 v;
  if (promo == 2)
    asm volatile("ld.global.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if (promo == 1)
    asm volatile("ld.global.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else
    v = __ldcs((const uint4*)p);
  return v;
}
template <int PROMO, int ORD>
__global__ void __launch_bounds__(256, 8) k_tile_promo(const int16_t* __restrict__ X,
                                                       const float* __restrict__ R,
                                                       float* __restrict__ out) {
  __shared__ __align__(16) float sm[64][64];
  const int w = blockIdx.x;
  const int ti = ORD == 0 ? w % 64 : w / 64, tj = ORD == 0 ? w / 64 : w % 64;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane % 8, r0 = warp * 4 + lane / 8;
  const int swz1 = (c * 4) & 31;
  uint4 v[2];
#pragma unroll
  for (int l = 0; l < 2; ++l)
    v[l] = ld_promo((const uint4*)(X + (size_t)(N - 1 - (ti * 64 + r0 + l * 32)) * N + tj * 64) + c, PROMO);
  float y[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) y[k] = __ldg(R + tj * 64 + c * 8 + k);
#pragma unroll
  for (int l = 0; l < 2; ++l) {
    const int16_t* e = (const int16_t*)&v[l];
#pragma unroll
    for (int k = 0; k < 8; ++k) sm[c * 8 + k][(r0 + l * 32) ^ swz1] = (float)e[k] + y[k];
  }
  __syncthreads();
  const int ig = threadIdx.x % 16;
#pragma unroll
  for (int pass = 0; pass < 4; ++pass) {
    const int j = threadIdx.x / 16 + 16 * pass;
    const int swz = ((j / 8) * 4) & 31;
    const float4 f = *(const float4*)&sm[j][(ig * 4) ^ swz];
    __stcs((float4*)(out + (size_t)(tj * 64 + j) * N + ti * 64 + ig * 4), f);
  }
}

// the full cfg2 op, one tile per block, with the float tile written by ONE
// TMA bulk tensor store (box 64 i x 64 j of the column-major output) from a
// dense [j][i] staging tile instead of 4 x 16-B st.global per thread
__global__ void __launch_bounds__(256, 4) k_tile_tmast(const __grid_constant__ CUtensorMap omap,
                                                       const int16_t* __restrict__ X,
                                                       const float* __restrict__ R, int ord) {
  __shared__ __align__(16) float sm[64][64];
  __shared__ __align__(128) float stg[64][64];
  const int w = blockIdx.x;
  const int ti = ord == 0 ? w % 64 : w / 64, tj = ord == 0 ? w / 64 : w % 64;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane % 8, r0 = warp * 4 + lane / 8;
  const int swz1 = (c * 4) & 31;
  uint4 v[2];
#pragma unroll
  for (int l = 0; l < 2; ++l)
    v[l] = __ldcs((const uint4*)(X + (size_t)(N - 1 - (ti * 64 + r0 + l * 32)) * N + tj * 64) + c);
  float y[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) y[k] = __ldg(R + tj * 64 + c * 8 + k);
#pragma unroll
  for (int l = 0; l < 2; ++l) {
    const int16_t* e = (const int16_t*)&v[l];
#pragma unroll
    for (int k = 0; k < 8; ++k) sm[c * 8 + k][(r0 + l * 32) ^ swz1] = (float)e[k] + y[k];
  }
  __syncthreads();
  const int ig = threadIdx.x % 16;
#pragma unroll
  for (int pass = 0; pass < 4; ++pass) {
    const int j = threadIdx.x / 16 + 16 * pass;
    const int swz = ((j / 8) * 4) & 31;
    *(float4*)&stg[j][ig * 4] = *(const float4*)&sm[j][(ig * 4) ^ swz];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
            (uint64_t)&omap),
        "r"(ti * 64), "r"(tj * 64), "r"((uint32_t)__cvta_generic_to_shared(&stg[0][0]))
        : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

// the full cfg2 op with 8-B loads: a warp instruction reads 2 X segments
// (16 lanes x 8 B = 128 B each), all 4 loads of a thread issued first;
// smem [j][i ^ s(j)], s(j) = ((j >> 2) & 7) * 4 keeps float4 groups intact
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_tile8(const int16_t* __restrict__ X,
                                                     const float* __restrict__ R,
                                                     float* __restrict__ out) {
  __shared__ __align__(16) float sm[64][64];
  const int w = blockIdx.x, ti = w % 64, tj = w / 64;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane % 16;  // j = 4q .. 4q+3
  uint2 v[4];
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const int row = warp * 8 + l * 2 + lane / 16;
    v[l] = __ldcs((const uint2*)(X + (size_t)(N - 1 - (ti * 64 + row)) * N + tj * 64) + q);
  }
  float y[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) y[k] = __ldg(R + tj * 64 + 4 * q + k);
  const int s1 = (q & 7) * 4;
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const int row = warp * 8 + l * 2 + lane / 16;
    const int16_t* e = (const int16_t*)&v[l];
#pragma unroll
    for (int k = 0; k < 4; ++k) sm[4 * q + k][row ^ s1] = (float)e[k] + y[k];
  }
  __syncthreads();
  const int ig = threadIdx.x % 16;
#pragma unroll
  for (int pass = 0; pass < 4; ++pass) {
    const int j = threadIdx.x / 16 + 16 * pass;
    const int s2 = ((j >> 2) & 7) * 4;
    const float4 f = *(const float4*)&sm[j][(ig * 4) ^ s2];
    __stcs((float4*)(out + (size_t)(tj * 64 + j) * N + ti * 64 + ig * 4), f);
  }
}

// reads contiguous (each tile's 4096 int16 from a contiguous 8 KiB block),
// writes in the cfg2 tile pattern (64 output columns x 256 B per tile)
__global__ void __launch_bounds__(256) k_twrite(const int16_t* __restrict__ X,
                                                float* __restrict__ out) {
  const int w = blockIdx.x, ti = w % 64, tj = w / 64;
  const int ig = threadIdx.x % 16;
#pragma unroll
  for (int pass = 0; pass < 4; ++pass) {
    const int j = threadIdx.x / 16 + 16 * pass;
    const uint2 v = __ldcs((const uint2*)(X + (size_t)w * 4096 + j * 64 + ig * 4));
    const int16_t* e = (const int16_t*)&v;
    __stcs((float4*)(out + (size_t)(tj * 64 + j) * N + ti * 64 + ig * 4),
           make_float4(e[0], e[1], e[2], e[3]));
  }
}

int main(int argc, char** argv) {
  const bool pool = argc > 1 && argv[1][0] == 'p';  // cudaMallocAsync (stream-ordered pool)
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int16_t* X[ROT];
  float* O[ROT];
  float* R;
  int* ctr;
  CK(cudaMalloc(&R, N * 4));
  CK(cudaMalloc(&ctr, 4096 * 4));
  CK(cudaMemset(ctr, 0, 4096 * 4));
  std::vector<int16_t> hx((size_t)N * N);
  std::vector<float> hr(N);
  for (size_t i = 0; i < hx.size(); ++i) hx[i] = (int16_t)((i * 2654435761u) % 2001) - 1000;
  for (int j = 0; j < N; ++j) hr[j] = (float)((j * 7919) % 1000) * 0.001f - 0.5f;
  for (int r = 0; r < ROT; ++r) {
    if (pool) {
      CK(cudaMallocAsync(&X[r], (size_t)N * 5120 * 2, 0));
      CK(cudaMallocAsync(&O[r], (size_t)N * 4608 * 4, 0));
      CK(cudaDeviceSynchronize());
    } else {
      CK(cudaMalloc(&X[r], (size_t)N * 5120 * 2));
      CK(cudaMalloc(&O[r], (size_t)N * 4608 * 4));
    }
    printf("set %d: X %p O %p\n", r, (void*)X[r], (void*)O[r]);
    CK(cudaMemcpy(X[r], hx.data(), hx.size() * 2, cudaMemcpyHostToDevice));
  }
  CK(cudaMemcpy(R, hr.data(), N * 4, cudaMemcpyHostToDevice));
  std::vector<float> ho((size_t)N * N);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = (double)N * N * 6 + N * 4;
  const int K = 40;
  int ctr_i = 0;
  auto timeit = [&](const char* name, auto launch, bool verify) {
    for (int r = 0; r < 8; ++r) launch(r % ROT, ctr + (ctr_i++ % 4096));
    CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      for (int k = 0; k < K; ++k) launch(k % ROT, ctr + (ctr_i++ % 4096));
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms / K < best ? ms / K : best;
    }
    CK(cudaGetLastError());
    size_t bad = 0;
    if (verify) {
      CK(cudaMemcpy(ho.data(), O[1], ho.size() * 4, cudaMemcpyDeviceToHost));
      for (int j = 0; j < N; ++j)
        for (int i = 0; i < N; ++i) {
          const float want = (float)hx[(size_t)j + (size_t)(N - 1 - i) * N] + hr[j];
          if (ho[(size_t)i + (size_t)j * N] != want) ++bad;
        }
      CK(cudaMemset(O[1], 0, (size_t)N * N * 4));
    }
    printf("%-52s %7.2f us %8.1f GB/s %s\n", name, best * 1e3, bytes / best / 1e6,
           verify ? (bad ? "MISMATCH" : "ok") : "");
    fflush(stdout);
  };
  // note: the counter array gives every launch a fresh zeroed counter (4096 launches max)
  timeit("contig i16->f32 same bytes (SOL for the mix)",
         [&](int r, int*) { k_contig<<<sms * 8, 256>>>(X[r], O[r], (size_t)N * N / 8); }, false);
  // the product kernels through the C ABI, same buffers, same stream (0 = the
  // library's default stream; events below are recorded on it)
  tpg_init();
  tpg_stream lib_stream = nullptr;
  tpg_default_stream(0, &lib_stream);
  cudaStream_t ls = *(cudaStream_t*)((char*)lib_stream + 8);
  {
    tpg_plan cp{};
    cp.ndim = 1; cp.nviews = 2; cp.extent[0] = (int64_t)N * N; cp.stride[0][0] = 4; cp.stride[1][0] = 2;
    tpg_plan hp{};
    hp.ndim = 2; hp.nviews = 3; hp.extent[0] = N; hp.extent[1] = N;
    hp.stride[0][0] = 4; hp.stride[0][1] = 4 * N; hp.stride[1][0] = -2 * N; hp.stride[1][1] = 2;
    hp.stride[2][0] = 0; hp.stride[2][1] = 4;
    auto timels = [&](const char* name, auto launch) {
      for (int r = 0; r < 8; ++r) launch(r % ROT);
      CK(cudaStreamSynchronize(ls));
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0, ls);
        for (int k = 0; k < K; ++k) launch(k % ROT);
        cudaEventRecord(e1, ls);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms / K < best ? ms / K : best;
      }
      printf("%-52s %7.2f us %8.1f GB/s\n", name, best * 1e3, bytes / best / 1e6);
      fflush(stdout);
    };
    timels("PRODUCT tpg_unary contiguous i16->f32 (k_contig)", [&](int r) {
      tpg_operand d{}, a{};
      d.base = O[r]; d.dtype = TPG_FLOAT; a.base = X[r]; a.dtype = TPG_INT16;
      tpg_unary(lib_stream, TPG_IDENTITY, &cp, &d, &a, TPG_INT16, 0, 0);
    });
    timels("PRODUCT tpg_binary cfg2 (k_tile_f32)", [&](int r) {
      tpg_operand d{}, a{}, b{};
      d.base = O[r]; d.dtype = TPG_FLOAT;
      a.base = X[r]; a.offset = (int64_t)(N - 1) * 2 * N; a.dtype = TPG_INT16;
      b.base = R; b.dtype = TPG_FLOAT;
      tpg_binary(lib_stream, TPG_ADD, &hp, &d, &a, &b, TPG_FLOAT, 0);
    });
    timels("ubench contig1 on the library stream", [&](int r) {
      k_contig1<<<N * N / 8 / 256, 256, 0, ls>>>(X[r], O[r]);
    });
    timels("ubench persist 64x64 on the library stream", [&](int r) {
      k_var<64, 64, 5, 0, 0, 1><<<sms * 5, 256, 0, ls>>>(X[r], R, O[r], ctr);
    });
  }
#define COLS(TI, TJ, MINB, SPAN)                                                               \
  timeit("cols " #TI "x" #TJ " minb" #MINB " span" #SPAN,                                     \
         [&](int r, int*) {                                                                    \
           k_cols<TI, TJ, MINB, SPAN><<<(N / TI) * (N / TJ) / SPAN, 256>>>(X[r], R, O[r]);     \
         },                                                                                    \
         true)
  COLS(64, 64, 5, 1);
  COLS(64, 64, 5, 2);
  COLS(64, 64, 5, 4);
  COLS(64, 64, 5, 8);
  COLS(64, 64, 5, 16);
  COLS(128, 64, 3, 4);
  COLS(128, 64, 3, 8);
  COLS(64, 128, 3, 4);
  COLS(64, 128, 3, 8);
  COLS(32, 128, 6, 8);
  COLS(32, 128, 6, 16);
#define WSHAPE(SEG, NC)                                                                        \
  timeit("write shape " #SEG " rows x " #NC " cols per block",                                 \
         [&](int r, int*) { k_wshape<SEG, NC><<<4096, 256>>>(X[r], O[r]); }, false)
  {
    CUtensorMap maps[ROT];
    for (int r = 0; r < ROT; ++r) {
      cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)N};
      cuuint64_t strides[1] = {(cuuint64_t)N * 4};
      cuuint32_t box[2] = {64, 64};
      cuuint32_t estr[2] = {1, 1};
      CUresult cr = cuTensorMapEncodeTiled(&maps[r], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, O[r], dims,
                                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                           CU_TENSOR_MAP_SWIZZLE_NONE,
                                           CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (cr != CUDA_SUCCESS) { printf("tensor map failed %d\n", (int)cr); return 1; }
    }
    timeit("TMA-store tile ord0", [&](int r, int*) { k_tile_tmast<<<4096, 256>>>(maps[r], X[r], R, 0); }, true);
    timeit("TMA-store tile ord1", [&](int r, int*) { k_tile_tmast<<<4096, 256>>>(maps[r], X[r], R, 1); }, true);
  }
  timeit("promo cs ord0", [&](int r, int*) { k_tile_promo<0, 0><<<4096, 256>>>(X[r], R, O[r]); }, true);
  timeit("promo 128B ord0", [&](int r, int*) { k_tile_promo<1, 0><<<4096, 256>>>(X[r], R, O[r]); }, true);
  timeit("promo 256B ord0", [&](int r, int*) { k_tile_promo<2, 0><<<4096, 256>>>(X[r], R, O[r]); }, true);
  timeit("promo cs ord1", [&](int r, int*) { k_tile_promo<0, 1><<<4096, 256>>>(X[r], R, O[r]); }, true);
  timeit("promo 128B ord1", [&](int r, int*) { k_tile_promo<1, 1><<<4096, 256>>>(X[r], R, O[r]); }, true);
  timeit("promo 256B ord1", [&](int r, int*) { k_tile_promo<2, 1><<<4096, 256>>>(X[r], R, O[r]); }, true);
  timeit("k_tile8 full op, 8-B loads, minb8", [&](int r, int*) { k_tile8<8><<<4096, 256>>>(X[r], R, O[r]); }, true);
  timeit("k_tile8 full op, 8-B loads, minb6", [&](int r, int*) { k_tile8<6><<<4096, 256>>>(X[r], R, O[r]); }, true);
  timeit("k_tile8 full op, 8-B loads, minb4", [&](int r, int*) { k_tile8<4><<<4096, 256>>>(X[r], R, O[r]); }, true);
  timeit("tile reads (8-B, hoisted) + contig2-style writes", [&](int r, int*) { k_tread3<<<4096, 256>>>(X[r], O[r]); }, false);
  timeit("tile reads ldx 4096 (dense)", [&](int r, int*) { k_tread_ld<4096><<<4096, 256>>>(X[r], O[r]); }, false);
  timeit("tile reads ldx 4160 (+128 B)", [&](int r, int*) { k_tread_ld<4160><<<4096, 256>>>(X[r], O[r]); }, false);
  timeit("tile reads ldx 4352 (+512 B)", [&](int r, int*) { k_tread_ld<4352><<<4096, 256>>>(X[r], O[r]); }, false);
  timeit("tile reads ldx 5120 (+2 KiB)", [&](int r, int*) { k_tread_ld<5120><<<4096, 256>>>(X[r], O[r]); }, false);
  timeit("tile-pattern reads hoisted, contiguous writes",
         [&](int r, int*) { k_tread_u<<<4096, 256>>>(X[r], O[r]); }, false);
  timeit("k_tile_hi: full cfg2 op, one tile / block, 8 blocks / SM",
         [&](int r, int*) { k_tile_hi<<<4096, 256>>>(X[r], R, O[r]); }, true);
#define TILEMT(T, MINB)                                                                        \
  {                                                                                            \
    CK(cudaFuncSetAttribute(k_tile_mt<T, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                            T * 16384));                                                       \
    timeit("k_tile_mt T=" #T " minb" #MINB,                                                    \
           [&](int r, int*) { k_tile_mt<T, MINB><<<4096 / T, 256, T * 16384>>>(X[r], R, O[r]); }, \
           true);                                                                              \
  }
  TILEMT(1, 8);
  TILEMT(2, 6);
  TILEMT(2, 4);
  TILEMT(4, 3);
  TILEMT(4, 2);
  TILEMT(8, 1);
  timeit("contig2 U=1 (one load, one store per thread)",
         [&](int r, int*) { k_contig2<1><<<N * N / 4 / 256, 256>>>(X[r], O[r]); }, false);
  timeit("write shape 4096x1, loads hoisted",
         [&](int r, int*) { k_wshape_u<4096, 1><<<4096, 256>>>(X[r], O[r]); }, false);
  timeit("write shape 64x64, loads hoisted",
         [&](int r, int*) { k_wshape_u<64, 64><<<4096, 256>>>(X[r], O[r]); }, false);
  WSHAPE(64, 64);
  WSHAPE(128, 32);
  WSHAPE(256, 16);
  WSHAPE(512, 8);
  WSHAPE(1024, 4);
  WSHAPE(2048, 2);
  WSHAPE(4096, 1);
  timeit("tile-pattern writes, ld 4096 (dense)",
         [&](int r, int*) { k_twrite_ld<4096><<<4096, 256>>>(X[r], O[r]); }, false);
  timeit("tile-pattern writes, ld 4128 (+128 B pad)",
         [&](int r, int*) { k_twrite_ld<4128><<<4096, 256>>>(X[r], O[r]); }, false);
  timeit("tile-pattern writes, ld 4160 (+256 B pad)",
         [&](int r, int*) { k_twrite_ld<4160><<<4096, 256>>>(X[r], O[r]); }, false);
  timeit("tile-pattern writes, ld 4608 (+2 KiB pad)",
         [&](int r, int*) { k_twrite_ld<4608><<<4096, 256>>>(X[r], O[r]); }, false);
  timeit("tile-pattern reads, full-sector contiguous writes",
         [&](int r, int*) { k_tread2<<<4096, 256>>>(X[r], O[r]); }, false);
#define STRIP(TJ, IH, MINB)                                                                    \
  {                                                                                            \
    const int smem = IH * (TJ + 2) * 2;                                                        \
    CK(cudaFuncSetAttribute(k_strip<TJ, IH, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                            smem));                                                            \
    timeit("strip TJ" #TJ " IH" #IH " minb" #MINB,                                             \
           [&](int r, int*) {                                                                  \
             k_strip<TJ, IH, MINB><<<(N / TJ) * (N / IH), 256, smem>>>(X[r], R, O[r]);         \
           },                                                                                  \
           true);                                                                              \
  }
  STRIP(16, 4096, 1);
  STRIP(16, 2048, 2);
  STRIP(16, 1024, 4);
  STRIP(16, 512, 8);
  STRIP(32, 1024, 2);
  STRIP(32, 512, 4);
  STRIP(64, 512, 2);
  STRIP(64, 256, 4);
  timeit("contig2 full-sector stores U=2",
         [&](int r, int*) { k_contig2<2><<<N * N / 4 / 512, 256>>>(X[r], O[r]); }, false);
  timeit("contig2 full-sector stores U=4",
         [&](int r, int*) { k_contig2<4><<<N * N / 4 / 1024, 256>>>(X[r], O[r]); }, false);
  timeit("contig1d one chunk per thread, via double",
         [&](int r, int*) { k_contig1d<<<N * N / 8 / 256, 256>>>(X[r], O[r]); }, false);
  for (int mult : {1, 2, 3, 4, 6, 8, 16}) {
    char nm[96];
    snprintf(nm, sizeof nm, "contig grid-stride float  grid=sms*%d", mult);
    timeit(nm, [&](int r, int*) { k_contig_gs<0><<<sms * mult, 256>>>(X[r], O[r], (size_t)N * N / 8); }, false);
    snprintf(nm, sizeof nm, "contig grid-stride double grid=sms*%d", mult);
    timeit(nm, [&](int r, int*) { k_contig_gs<1><<<sms * mult, 256>>>(X[r], O[r], (size_t)N * N / 8); }, false);
  }
  for (int mult : {1, 2, 3, 4}) {
    char nm[96];
    snprintf(nm, sizeof nm, "persist 64x64 grid=sms*%d", mult);
    timeit(nm, [&](int r, int* c) { k_var<64, 64, 5, 0, 0, 1><<<sms * mult, 256>>>(X[r], R, O[r], c); }, true);
  }
  timeit("contig1 one chunk per thread (product k_contig shape)",
         [&](int r, int*) { k_contig1<<<N * N / 8 / 256, 256>>>(X[r], O[r]); }, false);
  timeit("tile-pattern reads, contiguous writes",
         [&](int r, int*) { k_tread<<<4096, 256>>>(X[r], O[r]); }, false);
  timeit("contiguous reads, tile-pattern writes",
         [&](int r, int*) { k_twrite<<<4096, 256>>>(X[r], O[r]); }, false);
#define PERSIST(TI, TJ, MINB, ORD, PF, MULT)                                                  \
  timeit("persist " #TI "x" #TJ " minb" #MINB " ord" #ORD " pf" #PF " grid=sms*" #MULT,       \
         [&](int r, int* c) {                                                                  \
           k_var<TI, TJ, MINB, ORD, 0, PF><<<sms * MULT, 256>>>(X[r], R, O[r], c);             \
         },                                                                                    \
         true)
#define ONESHOT(TI, TJ, MINB, ORD)                                                             \
  timeit("oneshot " #TI "x" #TJ " minb" #MINB " ord" #ORD,                                     \
         [&](int r, int* c) {                                                                  \
           k_var<TI, TJ, MINB, ORD, 0, 1><<<(N / TI) * (N / TJ), 256>>>(X[r], R, O[r], c);     \
         },                                                                                    \
         true)
#define DYNQ(TI, TJ, MINB, ORD, MULT)                                                          \
  timeit("dynamic " #TI "x" #TJ " minb" #MINB " ord" #ORD " grid=sms*" #MULT,                 \
         [&](int r, int* c) {                                                                  \
           k_var<TI, TJ, MINB, ORD, 1, 1><<<sms * MULT, 256>>>(X[r], R, O[r], c);              \
         },                                                                                    \
         true)
  PERSIST(64, 64, 5, 0, 1, 5);
  PERSIST(64, 64, 5, 1, 1, 5);
  PERSIST(64, 64, 5, 4, 1, 5);
  PERSIST(64, 64, 5, 8, 1, 5);
  PERSIST(64, 64, 5, 16, 1, 5);
  PERSIST(64, 64, 5, 32, 1, 5);
  ONESHOT(64, 64, 8, 8);
  ONESHOT(64, 64, 8, 16);
  ONESHOT(64, 64, 8, 32);
  PERSIST(64, 128, 3, 8, 1, 3);
  PERSIST(64, 128, 3, 16, 1, 3);
  PERSIST(128, 64, 3, 8, 1, 3);
  PERSIST(128, 64, 3, 16, 1, 3);
  PERSIST(64, 64, 4, 0, 2, 4);
  PERSIST(64, 64, 6, 0, 1, 6);
  PERSIST(64, 64, 8, 0, 1, 8);
  ONESHOT(64, 64, 5, 0);
  ONESHOT(64, 64, 8, 0);
  ONESHOT(64, 64, 8, 1);
  DYNQ(64, 64, 5, 0, 5);
  DYNQ(64, 64, 6, 0, 6);
  PERSIST(128, 64, 3, 0, 1, 3);
  ONESHOT(128, 64, 4, 0);
  PERSIST(64, 128, 3, 0, 1, 3);
  ONESHOT(64, 128, 4, 0);
  ONESHOT(64, 128, 4, 1);
  ONESHOT(32, 64, 8, 0);
  ONESHOT(32, 128, 6, 0);
  ONESHOT(32, 128, 6, 1);
  PERSIST(32, 128, 6, 0, 1, 6);
  return 0;
}
