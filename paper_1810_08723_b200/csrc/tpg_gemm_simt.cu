// tpg_gemm_simt.cu — general strided matrix product for every dtype.
//
// Replaces kernels.matmul (pkg/src/tidepool/kernels.py:323-340) as driven by
// ops.matmul (ops.py:577-640): C[i,j] = sum_k A[i,k]*B[k,j] over byte-strided
// 2-D operands, products in the compute domain (Python int / float /
// complex), one rounding at the store (ops._make_store).  This SIMT kernel
// is the exact-semantics path for integer, bool, f64 and complex operands
// and for layouts the tensor-core path does not take; f16/bf16 (and the
// TF32x3 f32 path) run on tcgen05 in tpg_gemm_sm100.cu.
//
// Tiling: 64x64 outputs per 256-thread block, 4x4 per thread, K tiles of
// 16 staged through shared memory already decoded to the compute domain.
#include <cuda_runtime.h>

#include "tpg_common.cuh"
#include "tpg_internal.h"

namespace tpg {

struct GemmParams {
  const char* a;
  const char* b;
  char* d;
  int64_t as[3], bs[3], ds[3];  // row, col, batch byte strides
  int64_t m, n, k;
  int adt, bdt, ddt, aswap, bswap, dswap, aal, bal, dal, track;
  uint32_t* flags;
};

template <int KIND>
struct Dom;
template <>
struct Dom<K_INT> {
  typedef int64_t T;
  static __device__ T zero() { return 0; }
  static __device__ T load(int dt, R16 r) { return dec_int(dt, r); }
  static __device__ T mac(T acc, T x, T y) { return (int64_t)((uint64_t)acc + (uint64_t)x * (uint64_t)y); }
  static __device__ R16 enc(int dt, T v, uint32_t* fl) { return enc_from_int(dt, v, false, fl); }
};
template <>
struct Dom<K_UINT> {
  typedef int64_t T;
  static __device__ T zero() { return 0; }
  static __device__ T load(int dt, R16 r) { return dec_int(dt, r); }
  static __device__ T mac(T acc, T x, T y) { return (int64_t)((uint64_t)acc + (uint64_t)x * (uint64_t)y); }
  static __device__ R16 enc(int dt, T v, uint32_t* fl) { return enc_from_int(dt, v, true, fl); }
};
template <>
struct Dom<K_FLT> {
  typedef double T;
  static __device__ T zero() { return 0.0; }
  static __device__ T load(int dt, R16 r) { return dec_flt(dt, r); }
  static __device__ T mac(T acc, T x, T y) { return __dadd_rn(acc, __dmul_rn(x, y)); }
  // the reference accumulates with Neumaier compensation (kernels.py:192-198),
  // which turns any non-finite partial sum into NaN ((s - t) = inf - inf)
  static __device__ R16 enc(int dt, T v, uint32_t* fl) {
    return enc_from_flt(dt, isfinite(v) ? v : __longlong_as_double(0x7ff8000000000000ll), fl);
  }
};
template <>
struct Dom<K_CPX> {
  typedef double2 T;
  static __device__ T zero() { return make_double2(0.0, 0.0); }
  static __device__ T load(int dt, R16 r) { return dec_cpx(dt, r); }
  static __device__ T mac(T acc, T x, T y) {
    const double re = __dsub_rn(__dmul_rn(x.x, y.x), __dmul_rn(x.y, y.y));
    const double im = __dadd_rn(__dmul_rn(x.x, y.y), __dmul_rn(x.y, y.x));
    return make_double2(__dadd_rn(acc.x, re), __dadd_rn(acc.y, im));
  }
  static __device__ R16 enc(int dt, T v, uint32_t* fl) {
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    return enc_from_cpx(dt, isfinite(v.x) ? v.x : nan, isfinite(v.y) ? v.y : nan, fl);
  }
};

constexpr int GT = 64, GK = 16;

template <int KIND>
__global__ void __launch_bounds__(256) k_gemm_simt(GemmParams p) {
  typedef Dom<KIND> D;
  typedef typename D::T T;
  __shared__ T sa[GK][GT + 1];
  __shared__ T sb[GK][GT + 1];
  const int64_t bz = blockIdx.z;
  const char* A = p.a + bz * p.as[2];
  const char* B = p.b + bz * p.bs[2];
  char* Dp = p.d + bz * p.ds[2];
  const int64_t i0 = (int64_t)blockIdx.x * GT, j0 = (int64_t)blockIdx.y * GT;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  T acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = D::zero();
  for (int64_t kk = 0; kk < p.k; kk += GK) {
    for (int idx = threadIdx.x; idx < GT * GK; idx += 256) {
      // A tile: GT rows x GK k; threads sweep rows fastest (M-major)
      const int r = idx % GT, kq = idx / GT;
      const int64_t gi = i0 + r, gk = kk + kq;
      T va = D::zero();
      if (gi < p.m && gk < p.k) {
        R16 raw = load_raw(p.adt, A + gi * p.as[0] + gk * p.as[1], p.aal);
        if (p.aswap) raw = swap_raw(p.adt, raw);
        va = D::load(p.adt, raw);
      }
      sa[kq][r] = va;
      const int c = idx % GT, kb = idx / GT;
      const int64_t gj = j0 + c, gk2 = kk + kb;
      T vb = D::zero();
      if (gj < p.n && gk2 < p.k) {
        R16 raw = load_raw(p.bdt, B + gk2 * p.bs[0] + gj * p.bs[1], p.bal);
        if (p.bswap) raw = swap_raw(p.bdt, raw);
        vb = D::load(p.bdt, raw);
      }
      sb[kb][c] = vb;
    }
    __syncthreads();
#pragma unroll 4
    for (int q = 0; q < GK; ++q) {
      T ra[4], rb[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) ra[r] = sa[q][tx + 16 * r];
#pragma unroll
      for (int c = 0; c < 4; ++c) rb[c] = sb[q][ty + 16 * c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = D::mac(acc[r][c], ra[r], rb[c]);
    }
    __syncthreads();
  }
  uint32_t st = 0;
  uint32_t* fl = p.track ? &st : nullptr;
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t gi = i0 + tx + 16 * r, gj = j0 + ty + 16 * c;
      if (gi < p.m && gj < p.n) {
        R16 o = D::enc(p.ddt, acc[r][c], fl);
        if (p.dswap) o = swap_raw(p.ddt, o);
        store_raw(p.ddt, Dp + gi * p.ds[0] + gj * p.ds[1], o, p.dal);
      }
    }
  if (st) atomicOr(p.flags, st);
}

static bool aligned_op(const char* base, int dt, const int64_t* s, int64_t e0, int64_t e1) {
  const int al = dt_size(dt) < 8 ? dt_size(dt) : 8;
  if ((uintptr_t)base % al) return false;
  if (e0 > 1 && s[0] % al) return false;
  if (e1 > 1 && s[1] % al) return false;
  return true;
}

int gemm_simt(Stream* st, int64_t batch, const tpg_operand* d, const int64_t* ds,
              const tpg_operand* a, const int64_t* as, const tpg_operand* b, const int64_t* bs,
              int64_t m, int64_t n, int64_t k, int compute, int mode) {
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.a = (const char*)a->base + a->offset;
  p.b = (const char*)b->base + b->offset;
  p.d = (char*)d->base + d->offset;
  for (int i = 0; i < 3; ++i) {
    p.as[i] = as[i];
    p.bs[i] = bs[i];
    p.ds[i] = ds[i];
  }
  p.m = m; p.n = n; p.k = k;
  p.adt = a->dtype; p.bdt = b->dtype; p.ddt = d->dtype;
  p.aswap = a->big_endian; p.bswap = b->big_endian; p.dswap = d->big_endian;
  p.aal = aligned_op(p.a, p.adt, as, m, k);
  p.bal = aligned_op(p.b, p.bdt, bs, k, n);
  p.dal = aligned_op(p.d, p.ddt, ds, m, n);
  p.track = mode == TPG_WARNING || mode == TPG_ERROR;
  p.flags = device_flags(st->device);
  dim3 grid((unsigned)((m + GT - 1) / GT), (unsigned)((n + GT - 1) / GT), (unsigned)batch);
  switch (dt_kind(compute)) {
    case K_INT: k_gemm_simt<K_INT><<<grid, 256, 0, st->s>>>(p); break;
    case K_UINT: k_gemm_simt<K_UINT><<<grid, 256, 0, st->s>>>(p); break;
    case K_FLT: k_gemm_simt<K_FLT><<<grid, 256, 0, st->s>>>(p); break;
    default: k_gemm_simt<K_CPX><<<grid, 256, 0, st->s>>>(p); break;
  }
  TPG_LAUNCH_CHECK("gemm simt");
  return TPG_OK;
}

}  // namespace tpg
