// ubench_cfg2_tma.cu — design-space microbenchmark (NOT product code): the
// cfg2 transposing int16 -> f32 broadcast add with LARGE tiles fed by TMA,
// under the bench's steady-state methodology (back-to-back launches rotating
// over 4 input/output sets, 4 x 100.7 MB > 126 MB L2, one event pair around
// K launches):
//   out[i + j*N] = float(X[j + (N-1-i)*N]) + R[j],  N = 4096
// The register-staged 64x64 tiles of the product read 128-B X segments and
// write 256-B output segments; here one TMA 2-D load per 64-column box brings
// a TI x TJ int16 tile (TJ*2-byte X runs) into 128-B-swizzled shared memory,
// and each warp writes whole TI*4-byte output column runs: lane l holds row
// i0+l of 8 adjacent columns (one conflict-free LDS.128 thanks to the
// swizzle), so each of its 8 stores is one full 128-B line per warp.
// Persistent CTAs, STAGES-deep TMA ring (mbarrier complete_tx).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda \
//   -o scripts/ubench_cfg2_tma scripts/ubench_cfg2_tma.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

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

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// TI rows (i, output fast axis) x TJ columns (j, X fast axis) per tile.
// ORDER 0: i-tiles fastest across the work index; 1: j-tiles fastest.
// ST: 0 plain stores, 1 st.global.cs (evict-first).
template <int TI, int TJ, int STAGES, int ORDER, int ST>
__global__ void __launch_bounds__(256, 1)
    k_tma_tile(const __grid_constant__ CUtensorMap xmap, const float* __restrict__ R,
               float* __restrict__ out) {
  constexpr int NB = TJ / 64;                  // 64-column boxes per tile
  constexpr int BOX_BYTES = TI * 128;
  constexpr int STAGE_BYTES = NB * BOX_BYTES;
  constexpr int NTI = N / TI, NTJ = N / TJ, NT = NTI * NTJ;
  constexpr int ITEMS = (TI / 32) * (TJ / 8);  // (32-row group, 8-column chunk)
  extern __shared__ __align__(1024) uint8_t dyn[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)dyn + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[STAGES];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto coords = [&](int t, int& ti, int& tj) {
    if (ORDER == 0) { ti = t % NTI; tj = t / NTI; }
    else { tj = t % NTJ; ti = t / NTJ; }
  };
  auto issue = [&](int t, int s) {
    int ti, tj;
    coords(t, ti, tj);
    mbar_expect(&full[s], STAGE_BYTES);
#pragma unroll
    for (int b = 0; b < NB; ++b)
      tma_load_2d(sm + s * STAGE_BYTES + b * BOX_BYTES, &xmap, tj * TJ + b * 64,
                  N - (ti + 1) * TI, &full[s]);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&xmap) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      const int t = blockIdx.x + s * gridDim.x;
      if (t < NT) issue(t, s);
    }
  }
  int k = 0;
  for (int t = blockIdx.x; t < NT; t += gridDim.x, ++k) {
    const int s = k % STAGES;
    mbar_wait(&full[s], (k / STAGES) & 1);
    int ti, tj;
    coords(t, ti, tj);
    const uint8_t* st = sm + s * STAGE_BYTES;
    for (int it = warp; it < ITEMS; it += 8) {
      const int g = it % (TI / 32), cidx = it / (TI / 32);
      const int b = cidx / 8, c = cidx % 8;
      const int il = 32 * g + lane;
      const int rl = TI - 1 - il;  // tile row of X holding output row il
      const uint4 v = *(const uint4*)(st + b * BOX_BYTES + rl * 128 + ((c ^ (rl & 7)) << 4));
      const int j0 = tj * TJ + 8 * cidx;
      const float4 y0 = __ldg((const float4*)(R + j0));
      const float4 y1 = __ldg((const float4*)(R + j0 + 4));
      const float y[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
      const int16_t* e = (const int16_t*)&v;
      float* o = out + (size_t)j0 * N + ti * TI + il;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float f = (float)e[q] + y[q];
        if (ST) __stcs(o + (size_t)q * N, f);
        else o[(size_t)q * N] = f;
      }
    }
    __syncthreads();  // stage s consumed by every warp
    if (threadIdx.x == 0) {
      const int tn = t + STAGES * gridDim.x;
      if (tn < NT) issue(tn, s);
    }
  }
}

// same tile walk, but the 8 columns of a lane are transposed 4x4 across lane
// quads with shuffles so that every store is a 16-B float4 (4 columns x
// 128 B per warp instruction)
template <int TI, int TJ, int STAGES, int ORDER>
__global__ void __launch_bounds__(256, 1)
    k_tma_tile_v4(const __grid_constant__ CUtensorMap xmap, const float* __restrict__ R,
                  float* __restrict__ out) {
  constexpr int NB = TJ / 64;
  constexpr int BOX_BYTES = TI * 128;
  constexpr int STAGE_BYTES = NB * BOX_BYTES;
  constexpr int NTI = N / TI, NTJ = N / TJ, NT = NTI * NTJ;
  constexpr int ITEMS = (TI / 32) * (TJ / 8);
  extern __shared__ __align__(1024) uint8_t dyn[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)dyn + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[STAGES];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto coords = [&](int t, int& ti, int& tj) {
    if (ORDER == 0) { ti = t % NTI; tj = t / NTI; }
    else { tj = t % NTJ; ti = t / NTJ; }
  };
  auto issue = [&](int t, int s) {
    int ti, tj;
    coords(t, ti, tj);
    mbar_expect(&full[s], STAGE_BYTES);
#pragma unroll
    for (int b = 0; b < NB; ++b)
      tma_load_2d(sm + s * STAGE_BYTES + b * BOX_BYTES, &xmap, tj * TJ + b * 64,
                  N - (ti + 1) * TI, &full[s]);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      const int t = blockIdx.x + s * gridDim.x;
      if (t < NT) issue(t, s);
    }
  }
  const int m = lane & 3;  // position in the lane quad
  int k = 0;
  for (int t = blockIdx.x; t < NT; t += gridDim.x, ++k) {
    const int s = k % STAGES;
    mbar_wait(&full[s], (k / STAGES) & 1);
    int ti, tj;
    coords(t, ti, tj);
    const uint8_t* st = sm + s * STAGE_BYTES;
    for (int it = warp; it < ITEMS; it += 8) {
      const int g = it % (TI / 32), cidx = it / (TI / 32);
      const int b = cidx / 8, c = cidx % 8;
      const int il = 32 * g + lane;
      const int rl = TI - 1 - il;
      const uint4 v = *(const uint4*)(st + b * BOX_BYTES + rl * 128 + ((c ^ (rl & 7)) << 4));
      const int j0 = tj * TJ + 8 * cidx;
      const int16_t* e = (const int16_t*)&v;
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // columns j0+4h .. j0+4h+3
        float a[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) a[q] = (float)e[4 * h + q] + __ldg(R + j0 + 4 * h + q);
        // 4x4 transpose in the quad: lane m ends with column m of rows 4p..4p+3
        float r4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          // value of row (quad base + q), column m: lane (base+q) holds a[m]
          const float send = a[(m - q + 4) & 3];  // lane m sends its column (m-q) ...
          const float got = __shfl_sync(0xffffffffu, send, (lane & ~3) | ((m + q) & 3));
          r4[(m + q) & 3] = got;
          (void)send;
        }
        float* o = out + (size_t)(j0 + 4 * h + m) * N + ti * TI + 32 * g + (lane & ~3);
        __stcs((float4*)o, make_float4(r4[0], r4[1], r4[2], r4[3]));
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int tn = t + STAGES * gridDim.x;
      if (tn < NT) issue(tn, s);
    }
  }
}


// product-like variant: runtime column stride (sdq bytes), each lane owns
// one 16-B chunk (8 columns) of RG = TI/32 row groups, so one column address
// serves RG stores (+128 B immediates); warps own chunks w, w+8, ...
template <int TI, int STAGES>
__global__ void __launch_bounds__(256, 1)
    k_tma_rg(const __grid_constant__ CUtensorMap xmap, const float* __restrict__ R,
             float* __restrict__ out, long sdq) {
  constexpr int TJ = 64, RG = TI / 32;
  constexpr int BOX_BYTES = TI * 128;
  constexpr int STAGE_BYTES = BOX_BYTES;
  constexpr int NTI = N / TI, NTJ = N / TJ, NT = NTI * NTJ;
  extern __shared__ __align__(1024) uint8_t dyn[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)dyn + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[STAGES];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto issue = [&](int t, int s) {
    const int ti = t % NTI, tj = t / NTI;
    mbar_expect(&full[s], STAGE_BYTES);
    tma_load_2d(sm + s * STAGE_BYTES, &xmap, tj * TJ, N - (ti + 1) * TI, &full[s]);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < STAGES; ++s) {
      const int t = blockIdx.x + s * gridDim.x;
      if (t < NT) issue(t, s);
    }
  const int c = warp;  // chunk
  uint32_t soff[RG];
#pragma unroll
  for (int g = 0; g < RG; ++g) {
    const int rl = TI - 1 - (32 * g + lane);
    soff[g] = rl * 128 + ((c ^ (rl & 7)) << 4);
  }
  int k = 0;
  for (int t = blockIdx.x; t < NT; t += gridDim.x, ++k) {
    const int s = k % STAGES;
    mbar_wait(&full[s], (k / STAGES) & 1);
    const int ti = t % NTI, tj = t / NTI;
    const uint8_t* st = sm + s * STAGE_BYTES;
    uint4 v[RG];
#pragma unroll
    for (int g = 0; g < RG; ++g) v[g] = *(const uint4*)(st + soff[g]);
    const int j0 = tj * TJ + 8 * c;
    const float4 y0 = __ldg((const float4*)(R + j0));
    const float4 y1 = __ldg((const float4*)(R + j0 + 4));
    const float y[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
    char* dp = (char*)out + (size_t)j0 * sdq + (size_t)(ti * TI + lane) * 4;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float* col = (float*)(dp + q * sdq);
#pragma unroll
      for (int g = 0; g < RG; ++g) __stcs(col + 32 * g, (float)((const int16_t*)&v[g])[q] + y[q]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int tn = t + STAGES * gridDim.x;
      if (tn < NT) issue(tn, s);
    }
  }
}

int main(int argc, char** argv) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int16_t* X[ROT];
  float* O[ROT];
  float* R;
  CK(cudaMalloc(&R, N * 4));
  std::vector<int16_t> hx((size_t)N * N);
  std::vector<float> hr(N);
  for (size_t i = 0; i < hx.size(); ++i) hx[i] = (int16_t)((i * 2654435761u) % 2001) - 1000;
  for (int j = 0; j < N; ++j) hr[j] = (float)((j * 7919) % 1000) * 0.001f - 0.5f;
  CUtensorMap xm[ROT];
  for (int r = 0; r < ROT; ++r) {
    CK(cudaMalloc(&X[r], (size_t)N * N * 2));
    CK(cudaMalloc(&O[r], (size_t)N * N * 4));
    CK(cudaMemcpy(X[r], hx.data(), hx.size() * 2, cudaMemcpyHostToDevice));
  }
  CK(cudaMemcpy(R, hr.data(), N * 4, cudaMemcpyHostToDevice));
  std::vector<float> ho((size_t)N * N);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = (double)N * N * 6 + N * 4;
  const int K = 40;
  auto maps = [&](int ti) {
    for (int r = 0; r < ROT; ++r) {
      cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)N};
      cuuint64_t strides[1] = {(cuuint64_t)N * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)ti};
      cuuint32_t estr[2] = {1, 1};
      CUresult cr = cuTensorMapEncodeTiled(&xm[r], CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, X[r], dims,
                                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                           CU_TENSOR_MAP_SWIZZLE_128B,
                                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (cr != CUDA_SUCCESS) { printf("tensor map failed %d\n", (int)cr); exit(1); }
    }
  };
  auto timeit = [&](const char* name, auto launch) {
    for (int r = 0; r < 8; ++r) launch(r % ROT);
    CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      for (int k = 0; k < K; ++k) launch(k % ROT);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms / K < best ? ms / K : best;
    }
    CK(cudaGetLastError());
    CK(cudaMemcpy(ho.data(), O[1], ho.size() * 4, cudaMemcpyDeviceToHost));
    size_t bad = 0;
    for (int j = 0; j < N; ++j)
      for (int i = 0; i < N; ++i) {
        const float want = (float)hx[(size_t)j + (size_t)(N - 1 - i) * N] + hr[j];
        if (ho[(size_t)i + (size_t)j * N] != want) ++bad;
      }
    CK(cudaMemset(O[1], 0, (size_t)N * N * 4));
    printf("%-52s %7.2f us %8.1f GB/s %s\n", name, best * 1e3, bytes / best / 1e6,
           bad ? "MISMATCH" : "ok");
    fflush(stdout);
  };
#define RUN(TI, TJ, S, ORD, ST, CPS)                                                        \
  {                                                                                         \
    auto kern = k_tma_tile<TI, TJ, S, ORD, ST>;                                             \
    const int smem = S * (TJ / 64) * TI * 128 + 1024;                                       \
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));      \
    maps(TI);                                                                               \
    timeit("tma " #TI "x" #TJ " stages" #S " ord" #ORD " st" #ST " cta/sm" #CPS,            \
           [&](int r) { kern<<<sms * CPS, 256, smem>>>(xm[r], R, O[r]); });                 \
  }
#define RUN4(TI, TJ, S, ORD, CPS)                                                           \
  {                                                                                         \
    auto kern = k_tma_tile_v4<TI, TJ, S, ORD>;                                              \
    const int smem = S * (TJ / 64) * TI * 128 + 1024;                                       \
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));      \
    maps(TI);                                                                               \
    timeit("tma-v4 " #TI "x" #TJ " stages" #S " ord" #ORD " cta/sm" #CPS,                   \
           [&](int r) { kern<<<sms * CPS, 256, smem>>>(xm[r], R, O[r]); });                 \
  }
#define RUNRG(TI, S, CPS)                                                                    \
  {                                                                                         \
    auto kern = k_tma_rg<TI, S>;                                                            \
    const int smem = S * TI * 128 + 1024;                                                   \
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));      \
    maps(TI);                                                                               \
    timeit("rg " #TI "x64 stages" #S " cta/sm" #CPS " (runtime stride)",                    \
           [&](int r) { kern<<<sms * CPS, 256, smem>>>(xm[r], R, O[r], (long)N * 4); });    \
  }
  if (argc > 1 && argv[1][0] == '4') {  // sweep 4: row groups per lane, runtime stride
    RUNRG(64, 6, 4);
    RUNRG(128, 6, 2);
    RUNRG(128, 5, 2);
    RUNRG(128, 4, 3);
    RUNRG(128, 3, 4);
    RUNRG(256, 3, 2);
    RUNRG(256, 6, 1);
    RUNRG(64, 5, 5);
    RUNRG(64, 6, 4);
    RUN(64, 64, 6, 0, 1, 4);
    return 0;
  }
  if (argc > 1 && argv[1][0] == '3') {  // sweep 3: deeper rings
    RUN(64, 64, 6, 0, 1, 4);
    RUN(64, 64, 5, 0, 1, 4);
    RUN(64, 64, 8, 0, 1, 3);
    RUN(64, 64, 12, 0, 1, 2);
    RUN(64, 64, 24, 0, 1, 1);
    RUN(64, 64, 6, 0, 0, 4);
    RUN(32, 64, 12, 0, 1, 4);
    RUN(32, 128, 6, 0, 1, 4);
    RUN(64, 128, 6, 0, 1, 2);
    RUN(64, 64, 6, 0, 1, 4);
    return 0;
  }
  if (argc > 1 && argv[1][0] == '2') {  // sweep 2: around the 64x64 winner
    RUN(64, 64, 4, 0, 1, 4);
    RUN(64, 64, 2, 0, 1, 4);
    RUN(64, 64, 3, 0, 1, 4);
    RUN(64, 64, 6, 0, 1, 4);
    RUN(64, 64, 2, 0, 1, 6);
    RUN(64, 64, 3, 0, 1, 5);
    RUN(64, 64, 4, 0, 1, 5);
    RUN(64, 64, 3, 0, 1, 6);
    RUN(64, 64, 4, 0, 1, 6);
    RUN(64, 64, 2, 0, 1, 8);
    RUN(64, 64, 4, 0, 1, 3);
    RUN(64, 64, 6, 0, 1, 3);
    RUN(64, 64, 4, 1, 1, 4);
    RUN(64, 64, 4, 0, 0, 4);
    RUN(32, 64, 4, 0, 1, 4);
    RUN(32, 64, 4, 0, 1, 8);
    RUN(32, 64, 8, 0, 1, 4);
    RUN(32, 128, 4, 0, 1, 4);
    RUN(32, 128, 3, 0, 1, 6);
    RUN(32, 256, 3, 0, 1, 3);
    RUN(32, 256, 2, 0, 1, 4);
    RUN(64, 128, 3, 0, 1, 3);
    RUN(64, 128, 2, 0, 1, 4);
    RUN(128, 64, 2, 0, 1, 4);
    RUN(64, 64, 4, 0, 1, 4);
    return 0;
  }
  RUN(64, 64, 4, 0, 1, 4);
  RUN(64, 64, 8, 0, 1, 2);
  RUN(128, 64, 4, 0, 1, 2);
  RUN(64, 128, 4, 0, 1, 2);
  RUN(128, 128, 3, 0, 1, 2);
  RUN(128, 128, 3, 0, 0, 2);
  RUN(128, 128, 6, 0, 1, 1);
  RUN(128, 128, 3, 1, 1, 2);
  RUN(128, 256, 3, 0, 1, 1);
  RUN(256, 128, 3, 0, 1, 1);
  RUN(256, 256, 1, 0, 1, 1);
  RUN(256, 64, 3, 0, 1, 2);
  RUN(64, 256, 3, 0, 1, 2);
  RUN(32, 256, 4, 0, 1, 2);
  RUN4(128, 128, 3, 0, 2);
  RUN4(64, 128, 4, 0, 2);
  RUN4(128, 256, 3, 0, 1);
  RUN4(64, 64, 4, 0, 4);
  return 0;
}
