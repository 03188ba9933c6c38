// tpg_gemm_sm100.cu — tcgen05 / TMEM / TMA tensor-core gemm for half and
// bfloat16 operands (fp32 accumulation in tensor memory).
//
// Serves the matmul table entry (reference kernels.matmul,
// pkg/src/tidepool/kernels.py:323-340; ops.matmul ops.py:577-640) and the
// batched extension when both operands are half (or both bfloat16) and the
// destination is half / bfloat16 / float.  Contract vs the reference: the
// reference sums exact double products with Neumaier compensation and
// rounds once; here products are exact in fp32 and accumulate in fp32 in
// TMEM, then round once to the destination (parity tolerance 1e-2 rel to
// sum|a||b| for f16/bf16).  A non-finite accumulator becomes
// NaN, as the reference's compensated sum does.
//
// Kernel shape (persistent: one CTA per SM loops over output tiles in a
// grouped raster; 192 threads; two 128x256 fp32 accumulators in TMEM so
// the epilogue of one tile overlaps the mainloop of the next):
//   warp 0 lane 0   TMA producer: A tile 128x64 and B tile 256x64 (K-major,
//                   128B swizzle) per stage, 4-stage mbarrier ring
//   warp 1 lane 0   MMA issuer: 4 x tcgen05.mma.cta_group::1.kind::f16
//                   (M128 N256 K16) per stage, tcgen05.commit frees the stage
//   warps 2..5      epilogue: tcgen05.ld 32x32b.x32 -> registers -> convert
//                   -> global (coalesced along M for column-major C)
// Operands that are not K-major (or are byte-swapped / misaligned) are
// first packed into a K-major scratch copy by the elementwise engine.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "tpg_common.cuh"
#include "tpg_internal.h"

namespace tpg {

constexpr int GBM = 128, GBN = 256, GBK = 64, GSTAGES = 4;
constexpr int A_STAGE_BYTES = GBM * GBK * 2;
constexpr int B_STAGE_BYTES = GBN * GBK * 2;
constexpr int TMEM_COLS = 256;
constexpr int GEMM_THREADS = 192;
constexpr int GROUP_M = 16;
constexpr size_t GEMM_SMEM =
    1024 + (size_t)GSTAGES * (A_STAGE_BYTES + B_STAGE_BYTES) + 4 * 4096 + 8 * (2 * GSTAGES + 4) + 16;

struct Sm100Args {
  char* d;
  int64_t ds0, ds1, dsb;
  int m, n, k;
  int ddt;
  int epi;  // 0 generic, 1 column-major (M contiguous), 2 row-major (N contiguous)
  int tiles_m, tiles_n;
};

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"((uint64_t)map), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row groups 1024 B
// apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;             // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO
  d |= (uint64_t)1 << 46;             // descriptor version (Blackwell)
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}

#define TMEM_LD32(taddr, v)                                                                     \
  asm volatile(                                                                                 \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "                                                 \
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"                                 \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),     \
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),              \
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),           \
        "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),           \
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),           \
        "=r"(v[31])                                                                             \
      : "r"(taddr))

__device__ __forceinline__ uint32_t cvt_out(int ddt, float f) {
  if (!isfinite(f)) f = __int_as_float(0x7fc00000);
  if (ddt == TPG_HALF) return __half_as_ushort(__float2half_rn(f));
  if (ddt == TPG_BF16) return __bfloat16_as_ushort(__float2bfloat16_rn(f));
  return __float_as_uint(f);
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// grouped raster: GROUP_M row-tiles share the in-flight B tiles in L2
__device__ __forceinline__ void tile_coords(int t, const Sm100Args& g, int& m_tile, int& n_tile,
                                            int& batch) {
  const int per_batch = g.tiles_m * g.tiles_n;
  batch = t / per_batch;
  t -= batch * per_batch;
  const int per_group = GROUP_M * g.tiles_n;
  const int group = t / per_group;
  const int first_m = group * GROUP_M;
  const int gm = min(g.tiles_m - first_m, GROUP_M);
  const int r = t - group * per_group;
  m_tile = first_m + r % gm;
  n_tile = r / gm;
}

// Persistent: one CTA per SM loops over output tiles.  Two TMEM
// accumulators (2 x 256 columns) let the epilogue of tile i overlap the
// mainloop of tile i+1 (tfull/tempty mbarrier pair per accumulator).
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    k_gemm_sm100(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                 Sm100Args g, uint32_t idesc, int ntiles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* As = smem;
  uint8_t* Bs = smem + GSTAGES * A_STAGE_BYTES;
  uint8_t* epi_stage = Bs + GSTAGES * B_STAGE_BYTES;  // 4 warps x 4 KB
  uint64_t* bars = (uint64_t*)(epi_stage + 4 * 4096);
  uint64_t* full = bars;
  uint64_t* empty = bars + GSTAGES;
  uint64_t* tfull = bars + 2 * GSTAGES;       // [2]
  uint64_t* tempty = bars + 2 * GSTAGES + 2;  // [2]
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * GSTAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < GSTAGES; ++s) {
      mbar_init(su32(&full[s]), 1);
      mbar_init(su32(&empty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(su32(&tfull[b]), 1);
      mbar_init(su32(&tempty[b]), 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tma_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tma_b) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_slot)),
                 "r"(2 * TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const int nk = (g.k + GBK - 1) / GBK;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int m_tile, n_tile, batch;
        tile_coords(t, g, m_tile, n_tile, batch);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % GSTAGES;
          const uint32_t ph = (it / GSTAGES) & 1;
          mbar_wait(su32(&empty[s]), ph ^ 1);
          mbar_expect_tx(su32(&full[s]), A_STAGE_BYTES + B_STAGE_BYTES);
          tma_load_3d(su32(As + s * A_STAGE_BYTES), &tma_a, su32(&full[s]), kb * GBK,
                      m_tile * GBM, batch);
          tma_load_3d(su32(Bs + s * B_STAGE_BYTES), &tma_b, su32(&full[s]), kb * GBK,
                      n_tile * GBN, batch);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      uint32_t it = 0, lt = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
        const uint32_t b = lt & 1, use = lt >> 1;
        mbar_wait(su32(&tempty[b]), (use & 1) ^ 1);  // accumulator drained
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + b * TMEM_COLS;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % GSTAGES;
          const uint32_t ph = (it / GSTAGES) & 1;
          mbar_wait(su32(&full[s]), ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t ad = umma_desc_sw128(su32(As + s * A_STAGE_BYTES));
          const uint64_t bd = umma_desc_sw128(su32(Bs + s * B_STAGE_BYTES));
#pragma unroll
          for (int k = 0; k < GBK / 16; ++k)  // +32 B per K16 step inside the swizzle atom
            umma_f16(acc, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          umma_commit(su32(&empty[s]));
        }
        umma_commit(su32(&tfull[b]));
      }
    }
  } else {
    // epilogue: warp w reads TMEM lanes [32*(w%4), 32*(w%4)+32)
    const int q = warp & 3;
    const int es = dt_size(g.ddt);
    uint32_t lt = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      int m_tile, n_tile, batch;
      tile_coords(t, g, m_tile, n_tile, batch);
      const uint32_t b = lt & 1, use = lt >> 1;
      mbar_wait(su32(&tfull[b]), use & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = m_tile * GBM + q * 32 + lane;
      char* dbase = g.d + (int64_t)batch * g.dsb;
#pragma unroll 1
      for (int c = 0; c < GBN / 32; ++c) {
        uint32_t v[32];
        const uint32_t taddr =
            tmem + b * TMEM_COLS + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 32);
        TMEM_LD32(taddr, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c == GBN / 32 - 1) {
          // accumulator fully read: hand it back to the MMA warp
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(su32(&tempty[b]));
        }
        const int n0 = n_tile * GBN + c * 32;
        const int row0 = m_tile * GBM + q * 32;
        if (g.epi == 1 && row0 + 32 <= g.m && n0 + 32 <= g.n) {
          // column-major destination: transpose the warp's 32x32 chunk
          // through shared memory so each lane writes 16-B pieces of columns
          uint8_t* stg = epi_stage + (warp - 2) * 4096;
          if (es == 2) {
            uint16_t* s16 = (uint16_t*)stg;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              s16[j * 32 + lane] = (uint16_t)cvt_out(g.ddt, __uint_as_float(v[j]));
            __syncwarp();
#pragma unroll
            for (int it = 0; it < 4; ++it) {
              const int j = lane / 4 + 8 * it, part = lane % 4;
              const uint4 val = *(const uint4*)(s16 + j * 32 + part * 8);
              *(uint4*)(dbase + (int64_t)(row0 + part * 8) * 2 + (int64_t)(n0 + j) * g.ds1) = val;
            }
          } else {
            uint32_t* s32 = (uint32_t*)stg;
#pragma unroll
            for (int j = 0; j < 32; ++j) s32[j * 32 + lane] = cvt_out(g.ddt, __uint_as_float(v[j]));
            __syncwarp();
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int j = lane / 8 + 4 * it, part = lane % 8;
              const uint4 val = *(const uint4*)(s32 + j * 32 + part * 4);
              *(uint4*)(dbase + (int64_t)(row0 + part * 4) * 4 + (int64_t)(n0 + j) * g.ds1) = val;
            }
          }
          __syncwarp();
          continue;
        }
        if (row < g.m) {
          char* rp = dbase + (int64_t)row * g.ds0;
          if (g.epi == 2 && n0 + 32 <= g.n) {
            // row-major destination: 32 contiguous values per thread
            if (es == 2) {
              uint32_t w[16];
#pragma unroll
              for (int j = 0; j < 16; ++j)
                w[j] = cvt_out(g.ddt, __uint_as_float(v[2 * j])) |
                       (cvt_out(g.ddt, __uint_as_float(v[2 * j + 1])) << 16);
              uint4* dst = (uint4*)(rp + (int64_t)n0 * 2);
#pragma unroll
              for (int j = 0; j < 4; ++j)
                dst[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
            } else {
              uint4* dst = (uint4*)(rp + (int64_t)n0 * 4);
#pragma unroll
              for (int j = 0; j < 8; ++j)
                dst[j] = make_uint4(cvt_out(g.ddt, __uint_as_float(v[4 * j])),
                                    cvt_out(g.ddt, __uint_as_float(v[4 * j + 1])),
                                    cvt_out(g.ddt, __uint_as_float(v[4 * j + 2])),
                                    cvt_out(g.ddt, __uint_as_float(v[4 * j + 3])));
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int n = n0 + j;
              if (n < g.n) {
                const uint32_t o = cvt_out(g.ddt, __uint_as_float(v[j]));
                char* pp = rp + (int64_t)n * g.ds1;
                if (es == 2) *(uint16_t*)pp = (uint16_t)o;
                else *(uint32_t*)pp = o;
              }
            }
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(2 * TMEM_COLS));
  }
}

// ------------------------------------------------------------------ host
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

static bool make_map(CUtensorMap* map, int dt, const void* base, int64_t kdim, int64_t rows,
                     int64_t batch, int64_t row_stride, int64_t batch_stride, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)kdim, (cuuint64_t)rows, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)row_stride, (cuuint64_t)batch_stride};
  cuuint32_t box[3] = {GBK, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, dt == TPG_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                  3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// K-major operand view (rows x k) with row stride rs and unit k stride?
static bool k_major_ok(const tpg_operand* o, int64_t rs, int64_t ks, int64_t bstride, int64_t batch) {
  const uintptr_t base = (uintptr_t)o->base + o->offset;
  return !o->big_endian && ks == 2 && rs > 0 && rs % 16 == 0 && base % 16 == 0 &&
         (batch == 1 || (bstride > 0 && bstride % 16 == 0));
}

extern "C" int tpg_unary(tpg_stream stream, int op, const tpg_plan* plan, const tpg_operand* d,
                         const tpg_operand* a, int compute, int mode, int force_complex);

// pack a (rows x k) operand with strides (rs, ks, bs) into a K-major
// contiguous scratch (row stride kp*2, batch stride rows*kp*2)
static int pack_k_major(Stream* st, const tpg_operand* src, int64_t rows, int64_t k, int64_t batch,
                        int64_t rs, int64_t ks, int64_t bs, void** out, int64_t* out_rs) {
  const int64_t kp = (k + 7) & ~(int64_t)7;
  const size_t bytes = (size_t)(kp * rows * batch * 2);
  TPG_CUDA_CHECK(cudaMallocAsync(out, bytes ? bytes : 16, st->s));
  tpg_plan p{};
  p.ndim = 3;
  p.nviews = 2;
  p.extent[0] = k; p.extent[1] = rows; p.extent[2] = batch;
  p.stride[0][0] = 2; p.stride[0][1] = kp * 2; p.stride[0][2] = kp * rows * 2;
  p.stride[1][0] = ks; p.stride[1][1] = rs; p.stride[1][2] = bs;
  tpg_operand d{};
  d.base = *out;
  d.dtype = src->dtype;
  int rc = tpg_unary(st, TPG_IDENTITY, &p, &d, src, src->dtype, TPG_STANDARD, 0);
  *out_rs = kp * 2;
  return rc;
}

int gemm_sm100(Stream* st, int64_t batch, const tpg_operand* d, const int64_t* ds,
               const tpg_operand* a, const int64_t* as, const tpg_operand* b, const int64_t* bs,
               int64_t m, int64_t n, int64_t k, int compute, int mode) {
  const int adt = a->dtype;
  if (!(adt == TPG_HALF || adt == TPG_BF16) || b->dtype != adt) return 0;
  if (!(d->dtype == TPG_HALF || d->dtype == TPG_BF16 || d->dtype == TPG_FLOAT)) return 0;
  if (dt_kind(compute) != K_FLT || mode != TPG_STANDARD || d->big_endian) return 0;
  if (m < 128 || n < 128 || k < 64 || m > INT32_MAX || n > INT32_MAX || k > INT32_MAX) return 0;
  if (batch * ((m + GBM - 1) / GBM) * ((n + GBN - 1) / GBN) > INT32_MAX) return 0;
  if (sm_count(st->device) <= 0) return 0;
  {
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, st->device);
    if (major != 10) return 0;
  }
  // A is (m x k): rows = m, row stride as[0], k stride as[1]
  // B is (k x n): rows = n, row stride bs[1], k stride bs[0]
  const void* abase = (const char*)a->base + a->offset;
  const void* bbase = (const char*)b->base + b->offset;
  int64_t a_rs = as[0], b_rs = bs[1], a_bs = as[2], b_bs = bs[2];
  void* apack = nullptr;
  void* bpack = nullptr;
  int rc;
  if (!k_major_ok(a, as[0], as[1], as[2], batch)) {
    rc = pack_k_major(st, a, m, k, batch, as[0], as[1], as[2], &apack, &a_rs);
    if (rc) return rc;
    abase = apack;
    a_bs = a_rs * m;
  }
  if (!k_major_ok(b, bs[1], bs[0], bs[2], batch)) {
    rc = pack_k_major(st, b, n, k, batch, bs[1], bs[0], bs[2], &bpack, &b_rs);
    if (rc) return rc;
    bbase = bpack;
    b_bs = b_rs * n;
  }
  if (batch == 1) {
    a_bs = a_rs * m;
    b_bs = b_rs * n;
  }
  CUtensorMap ma, mb;
  if (!make_map(&ma, adt, abase, k, m, batch, a_rs, a_bs, GBM) ||
      !make_map(&mb, adt, bbase, k, n, batch, b_rs, b_bs, GBN)) {
    if (apack) cudaFreeAsync(apack, st->s);
    if (bpack) cudaFreeAsync(bpack, st->s);
    return 0;  // not encodable: SIMT path
  }
  Sm100Args g;
  g.d = (char*)d->base + d->offset;
  g.ds0 = ds[0];
  g.ds1 = ds[1];
  g.dsb = ds[2];
  g.m = (int)m;
  g.n = (int)n;
  g.k = (int)k;
  g.ddt = d->dtype;
  const int es = dt_size(d->dtype);
  const bool al = ((uintptr_t)g.d % 16) == 0;
  g.epi = (ds[1] == es && ds[0] % 16 == 0 && al) ? 2
          : (ds[0] == es && ds[1] % 16 == 0 && al && (batch == 1 || ds[2] % 16 == 0)) ? 1 : 0;
  g.tiles_m = (int)((m + GBM - 1) / GBM);
  g.tiles_n = (int)((n + GBN - 1) / GBN);
  const uint32_t fmt = adt == TPG_BF16 ? 1u : 0u;
  const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(GBN >> 3) << 17) |
                         ((uint32_t)(GBM >> 4) << 24);
  static bool attr_set[64] = {false};
  if (!attr_set[st->device]) {
    TPG_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_sm100, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)GEMM_SMEM));
    attr_set[st->device] = true;
  }
  const int ntiles = g.tiles_m * g.tiles_n * (int)batch;
  const int grid = ntiles < sm_count(st->device) ? ntiles : sm_count(st->device);
  k_gemm_sm100<<<grid, GEMM_THREADS, GEMM_SMEM, st->s>>>(ma, mb, g, idesc, ntiles);
  TPG_LAUNCH_CHECK("gemm sm100");
  if (apack) TPG_CUDA_CHECK(cudaFreeAsync(apack, st->s));
  if (bpack) TPG_CUDA_CHECK(cudaFreeAsync(bpack, st->s));
  return 1;
}

}  // namespace tpg
