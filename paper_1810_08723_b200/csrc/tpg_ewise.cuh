// tpg_ewise.cuh — the strided elementwise / copy-cast engine (shared by the
// tpg_ewise_*.cu translation units).
//
// Replaces the reference loops kernels.binary_elementwise (kernels.py:213-248),
// kernels.unary_elementwise (275-302, also the `copy` entry via ops.py:681),
// kernels.fill (343-352), kernels.arange_fill (377-381),
// kernels.byteswap_inplace (355-357) and kernels.gather (360-363).  The plan
// is the reference IterPlan after canonicalize (tensors.py:570-604): axis 0
// is the destination's fastest axis.
//
// Traversals (picked per call on the host, see choose_traversal):
//   contig  1-D plans whose views are unit-stride (or broadcast): each
//           thread moves 8 elements per operand with 128-bit loads/stores;
//           compile-time-typed fast set (Tier A) only.
//   tile    an input whose fastest axis is not the destination's (a
//           transposed / reversed view, SURVEY cfg2) is staged through a
//           64x64 shared-memory tile so both its loads and the destination
//           stores are coalesced.
//   rows    axis 0 inner, remaining axes decomposed once per block-row.
//   flat    per-element index decomposition (short axis 0).
// Element semantics (decode, compute, cast-on-store) are in tpg_common.cuh.
// Tier A kernels fix op and dtypes at compile time (inlined, small); Tier B
// (dtype -1) calls one out-of-line element function that switches on the
// runtime dtypes (warp-uniform), covering all 15x15 pairs, both byte orders
// and every op with one kernel per (op class, compute kind, traversal).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <thrust/complex.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "tpg_common.cuh"
#include "tpg_internal.h"

namespace tpg {

enum OpClass { OC_BINARY = 0, OC_UNARY = 1, OC_COPY = 2, OC_FILL = 3, OC_ARANGE = 4,
               OC_BSWAP = 5, OC_RAW = 6 };

struct EwParams {
  int ndim;
  int nin;
  int64_t ext[TPG_MAX_DIMS];
  int64_t str[3][TPG_MAX_DIMS];
  char* base[3];
  R16 imm[3];
  int dt[3];
  int swap[3];
  int aligned[3];
  int isimm[3];
  int op;
  int track;
  int dry;
  int force_complex;
  uint32_t* flags;
};

// the per-element descriptor handed (by value) to the out-of-line op
struct EwDesc {
  int dtd, dta, dtb;
  int sd, sa, sb;
  int op, track, fc;
};

// ------------------------------------------------------------ unary math
__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000ll); }

// UNARY_TABLE real branch + unary_scalar_fn domain flag (kernels.py:121-158)
__device__ __forceinline__ double un_flt(int op, double v, uint32_t& st) {
  switch (op) {
    case TPG_NEGATE: return -v;
    case TPG_ABSOLUTE: return fabs(v);
    case TPG_SQRT:
      if (v < 0.0) { st |= TPG_FLAG_DOMAIN; return qnan(); }
      return isnan(v) ? qnan() : sqrt(v);
    case TPG_EXP: return isnan(v) ? qnan() : exp(v);
    case TPG_LOG:
      if (v < 0.0) { st |= TPG_FLAG_DOMAIN; return qnan(); }
      if (isnan(v)) return qnan();
      if (v == 0.0) return -INFINITY;
      return log(v);
    case TPG_SIN: return isnan(v) ? qnan() : sin(v);
    case TPG_COS: return isnan(v) ? qnan() : cos(v);
    case TPG_ASIN:
      if (fabs(v) > 1.0) { st |= TPG_FLAG_DOMAIN; return qnan(); }
      return isnan(v) ? qnan() : asin(v);
    case TPG_ACOS:
      if (fabs(v) > 1.0) { st |= TPG_FLAG_DOMAIN; return qnan(); }
      return isnan(v) ? qnan() : acos(v);
    default: return v;  // conjugate / identity
  }
}

__device__ __forceinline__ int64_t un_int(int op, int64_t v, bool uns) {
  switch (op) {
    case TPG_NEGATE: return (int64_t)(0ull - (uint64_t)v);
    case TPG_ABSOLUTE: return (!uns && v < 0) ? (int64_t)(0ull - (uint64_t)v) : v;
    default: return v;
  }
}

// complex branch (cmath); results are tolerance-level vs CPython's cmath
static __device__ __noinline__ double2 un_cpx(int op, double2 z) {
  typedef thrust::complex<double> C;
  C c(z.x, z.y), r;
  switch (op) {
    case TPG_NEGATE: return make_double2(-z.x, -z.y);
    case TPG_ABSOLUTE: return make_double2(hypot(z.x, z.y), 0.0);
    case TPG_SQRT: r = thrust::sqrt(c); break;
    case TPG_EXP: r = thrust::exp(c); break;
    case TPG_LOG:
      if (z.x == 0.0 && z.y == 0.0) return make_double2(-INFINITY, 0.0);
      r = thrust::log(c);
      break;
    case TPG_SIN: r = thrust::sin(c); break;
    case TPG_COS: r = thrust::cos(c); break;
    case TPG_ASIN: r = thrust::asin(c); break;
    case TPG_ACOS: r = thrust::acos(c); break;
    case TPG_CONJ: return make_double2(z.x, -z.y);
    default: return z;
  }
  return make_double2(r.real(), r.imag());
}

// ------------------------------------------------------------ element op
template <int OC, int KIND>
__device__ __forceinline__ R16 ew_body(const EwDesc& e, R16 ra, R16 rb, int64_t lin, uint32_t& st) {
  const int d_t = e.dtd, a_t = e.dta, b_t = e.dtb, op = e.op;
  uint32_t* fl = e.track ? &st : nullptr;
  R16 out{0, 0};
  if (OC == OC_RAW) return ra;
  if (OC == OC_BSWAP) return swap_raw(d_t, ra);
  if (OC == OC_ARANGE) {
    out = enc_from_int(d_t, lin, false, fl);
  } else if (OC == OC_BINARY) {
    if (e.sa) ra = swap_raw(a_t, ra);
    if (e.sb) rb = swap_raw(b_t, rb);
    if (KIND == K_INT) {
      out = enc_from_int(d_t, bin_int(op, dec_int(a_t, ra), dec_int(b_t, rb), &st), false, fl);
    } else if (KIND == K_UINT) {
      out = enc_from_int(
          d_t, (int64_t)bin_uint(op, (uint64_t)dec_int(a_t, ra), (uint64_t)dec_int(b_t, rb), &st),
          true, fl);
    } else if (KIND == K_FLT) {
      out = enc_from_flt(d_t, bin_flt(op, dec_flt(a_t, ra), dec_flt(b_t, rb)), fl);
    } else {
      double2 r = bin_cpx(op, dec_cpx(a_t, ra), dec_cpx(b_t, rb));
      out = enc_from_cpx(d_t, r.x, r.y, fl);
    }
  } else if (OC == OC_UNARY) {
    if (e.sa) ra = swap_raw(a_t, ra);
    if (KIND == K_CPX || (KIND == K_FLT && e.fc)) {
      double2 r = un_cpx(op, dec_cpx(a_t, ra));
      out = (op == TPG_ABSOLUTE) ? enc_from_flt(d_t, r.x, fl) : enc_from_cpx(d_t, r.x, r.y, fl);
    } else if (KIND == K_FLT) {
      out = enc_from_flt(d_t, un_flt(op, dec_flt(a_t, ra), st), fl);
    } else {
      out = enc_from_int(d_t, un_int(op, dec_int(a_t, ra), KIND == K_UINT), KIND == K_UINT, fl);
    }
  } else {  // OC_COPY: value copy with cast-on-store (ops._run_copy)
    if (e.sa) ra = swap_raw(a_t, ra);
    if (a_t == d_t && a_t != TPG_BOOL) {
      out = ra;  // same dtype: the value round-trips exactly
    } else if (KIND == K_CPX) {
      double2 v = dec_cpx(a_t, ra);
      out = enc_from_cpx(d_t, v.x, v.y, fl);
    } else if (KIND == K_FLT) {
      out = enc_from_flt(d_t, dec_flt(a_t, ra), fl);
    } else {
      out = enc_from_int(d_t, dec_int(a_t, ra), KIND == K_UINT, fl);
    }
  }
  if (e.sd) out = swap_raw(d_t, out);
  return out;
}

// Tier B: one out-of-line copy of the body per (op class, kind)
struct R16S {
  R16 r;
  uint32_t st;
};
template <int OC, int KIND>
__device__ __noinline__ R16S ew_body_gen(EwDesc e, R16 ra, R16 rb, int64_t lin) {
  uint32_t st = 0;
  R16 r = ew_body<OC, KIND>(e, ra, rb, lin, st);
  return R16S{r, st};
}

template <int OC, int NIN, int OP, int KIND, int DTD, int DTA, int DTB>
struct Ew {
  static constexpr bool typed = DTD >= 0 && (DTA >= 0 || NIN < 1) && (DTB >= 0 || NIN < 2);
  static __device__ __forceinline__ int dtd(const EwParams& p) { return DTD >= 0 ? DTD : p.dt[0]; }
  static __device__ __forceinline__ int dta(const EwParams& p) { return DTA >= 0 ? DTA : p.dt[1]; }
  static __device__ __forceinline__ int dtb(const EwParams& p) { return DTB >= 0 ? DTB : p.dt[2]; }

  static __device__ __forceinline__ R16 apply(const EwParams& p, R16 ra, R16 rb, int64_t lin,
                                              uint32_t& st) {
    if (OC == OC_FILL) return p.imm[1];
    EwDesc e;
    e.dtd = dtd(p); e.dta = dta(p); e.dtb = dtb(p);
    e.sd = p.swap[0]; e.sa = p.swap[1]; e.sb = p.swap[2];
    e.op = OP >= 0 ? OP : p.op;
    e.track = p.track;
    e.fc = p.force_complex;
    if (typed || OC == OC_RAW || OC == OC_BSWAP || OC == OC_ARANGE)
      return ew_body<OC, KIND>(e, ra, rb, lin, st);
    R16S x = ew_body_gen<OC, KIND>(e, ra, rb, lin);
    st |= x.st;
    return x.r;
  }
};

// load operand V (1 or 2) at byte offset off
template <class F, int V>
__device__ __forceinline__ R16 ld_op(const EwParams& p, int64_t off) {
  if (p.isimm[V]) return p.imm[V];
  const int dt = V == 1 ? F::dta(p) : F::dtb(p);
  return load_raw(dt, p.base[V] + off, p.aligned[V]);
}

// ------------------------------------------------------------ traversals
// rows: axis 0 inner.  Work item = (tile of axis 0, row over axes 1..).
template <class F, int NIN, int U>
__global__ void __launch_bounds__(256) k_rows(EwParams p, int64_t rows, int64_t ntile) {
  const int64_t e0 = p.ext[0];
  uint32_t st = 0;
  const int dtd = F::dtd(p);
  for (int64_t w = blockIdx.x; w < rows * ntile; w += gridDim.x) {
    const int64_t row = w / ntile, tile = w - row * ntile;
    int64_t od = 0, oa = 0, ob = 0, r = row;
    for (int k = 1; k < p.ndim; ++k) {
      const int64_t e = p.ext[k];
      const int64_t c = r % e;
      r /= e;
      od += c * p.str[0][k];
      if (NIN >= 1) oa += c * p.str[1][k];
      if (NIN >= 2) ob += c * p.str[2][k];
    }
    const int64_t i_base = tile * (256 * U) + threadIdx.x;
    R16 ra[U], rb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i0 = i_base + u * 256;
      ra[u] = rb[u] = R16{0, 0};
      if (i0 < e0) {
        if (NIN >= 1) ra[u] = ld_op<F, 1>(p, oa + i0 * p.str[1][0]);
        if (NIN >= 2) rb[u] = ld_op<F, 2>(p, ob + i0 * p.str[2][0]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i0 = i_base + u * 256;
      if (i0 < e0) {
        R16 o = F::apply(p, ra[u], rb[u], row * e0 + i0, st);
        if (!p.dry) store_raw(dtd, p.base[0] + od + i0 * p.str[0][0], o, p.aligned[0]);
      }
    }
  }
  if (st) atomicOr(p.flags, st);
}

// flat: full index decomposition per element
template <class F, int NIN>
__global__ void __launch_bounds__(256) k_flat(EwParams p, int64_t total) {
  uint32_t st = 0;
  const int dtd = F::dtd(p);
  const int64_t nthreads = (int64_t)gridDim.x * 256;
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < total; i += nthreads) {
    int64_t r = i, d = 0, a = 0, b = 0;
    for (int k = 0; k < p.ndim; ++k) {
      const int64_t e = p.ext[k];
      const int64_t c = r % e;
      r /= e;
      d += c * p.str[0][k];
      if (NIN >= 1) a += c * p.str[1][k];
      if (NIN >= 2) b += c * p.str[2][k];
    }
    R16 ra{0, 0}, rb{0, 0};
    if (NIN >= 1) ra = ld_op<F, 1>(p, a);
    if (NIN >= 2) rb = ld_op<F, 2>(p, b);
    R16 o = F::apply(p, ra, rb, i, st);
    if (!p.dry) store_raw(dtd, p.base[0] + d, o, p.aligned[0]);
  }
  if (st) atomicOr(p.flags, st);
}

// tile: operand X (1 or 2) is coalesced along axis q != 0; stage 64x64
// tiles of it in shared memory, then sweep the tile along axis 0 so the
// destination (and any axis-0-coalesced operand) is written coalesced.
constexpr int TT = 64;

template <class F, int NIN, int X>
__global__ void __launch_bounds__(256) k_tile(EwParams p, int q, int64_t nt0, int64_t ntq,
                                              int64_t nrest) {
  __shared__ uint64_t tile[TT][TT + 1];
  const int64_t e0 = p.ext[0], eq = p.ext[q];
  const int dtd = F::dtd(p);
  const int dtx = X == 1 ? F::dta(p) : F::dtb(p);
  uint32_t st = 0;
  const int64_t nwork = nt0 * ntq * nrest;
  for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int64_t t0 = w % nt0;
    const int64_t tq = (w / nt0) % ntq;
    int64_t rr = w / (nt0 * ntq);
    int64_t off[3] = {0, 0, 0};
    for (int k = 1; k < p.ndim; ++k) {
      if (k == q) continue;
      const int64_t e = p.ext[k];
      const int64_t c = rr % e;
      rr /= e;
#pragma unroll
      for (int v = 0; v < 3; ++v) off[v] += c * p.str[v][k];
    }
    // phase 1: coalesced along q
    {
      constexpr int U = 4;
      for (int idx0 = threadIdx.x; idx0 < TT * TT; idx0 += 256 * U) {
        uint64_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = idx0 + u * 256;
          const int iq = idx % TT, i0 = idx / TT;
          const int64_t g0 = t0 * TT + i0, gq = tq * TT + iq;
          v[u] = 0;
          if (g0 < e0 && gq < eq)
            v[u] = load_raw(dtx, p.base[X] + off[X] + g0 * p.str[X][0] + gq * p.str[X][q],
                            p.aligned[X]).lo;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = idx0 + u * 256;
          tile[idx / TT][idx % TT] = v[u];
        }
      }
    }
    __syncthreads();
    // phase 2: coalesced along axis 0
    {
      constexpr int U = 4;
      constexpr int Y = 3 - X;
      for (int idx0 = threadIdx.x; idx0 < TT * TT; idx0 += 256 * U) {
        R16 ry[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = idx0 + u * 256;
          const int i0 = idx % TT, iq = idx / TT;
          const int64_t g0 = t0 * TT + i0, gq = tq * TT + iq;
          ry[u] = R16{0, 0};
          if (NIN >= 2 && g0 < e0 && gq < eq)
            ry[u] = ld_op<F, Y>(p, off[Y] + g0 * p.str[Y][0] + gq * p.str[Y][q]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = idx0 + u * 256;
          const int i0 = idx % TT, iq = idx / TT;
          const int64_t g0 = t0 * TT + i0, gq = tq * TT + iq;
          if (g0 < e0 && gq < eq) {
            const R16 rx{tile[i0][iq], 0};
            R16 o = (X == 1) ? F::apply(p, rx, ry[u], 0, st) : F::apply(p, ry[u], rx, 0, st);
            if (!p.dry)
              store_raw(dtd, p.base[0] + off[0] + g0 * p.str[0][0] + gq * p.str[0][q], o,
                        p.aligned[0]);
          }
        }
      }
    }
    __syncthreads();
  }
  if (st) atomicOr(p.flags, st);
}

// tile_fast: typed variant of `tile` for full 64x64 tiles with unit-stride,
// 16-B-aligned access along both fast axes (SURVEY cfg2).  Phase 1: each
// thread loads 16 B of X along q (i0 fastest across a warp, so the
// transposing smem writes are conflict-free); phase 2: each thread reads 4
// consecutive i0 of one q column, combines them with Y (imm, broadcast or
// unit-stride along axis 0) and writes 4*SD bytes to the destination.
template <int S>
struct RawT;
template <>
struct RawT<1> { typedef uint8_t T; };
template <>
struct RawT<2> { typedef uint16_t T; };
template <>
struct RawT<4> { typedef uint32_t T; };
template <>
struct RawT<8> { typedef uint64_t T; };

template <class F, int NIN, int X, int SD, int SX, int SY>
__global__ void __launch_bounds__(256) k_tile_fast(EwParams p, int q, int64_t nt0, int64_t ntq,
                                                   int64_t nrest, int ymode) {
  typedef typename RawT<SX>::T TX;
  constexpr int VX = 16 / SX;          // X elements per 16-B load
  constexpr int CHUNKS = TT / VX;      // 16-B chunks per tile row
  __shared__ __align__(16) TX sm[TT][TT];  // [q][i0]
  constexpr int Y = 3 - X;
  const int dtd = F::dtd(p);
  uint32_t st = 0;
  const int64_t nwork = nt0 * ntq * nrest;
  // tile origin offsets of work item w (per view)
  auto origin = [&](int64_t w, int64_t (&off)[3], int64_t& t0, int64_t& tq) {
    t0 = w % nt0;
    tq = (w / nt0) % ntq;
    int64_t rr = w / (nt0 * ntq);
    off[0] = off[1] = off[2] = 0;
    for (int k = 1; k < p.ndim; ++k) {
      if (k == q) continue;
      const int64_t e = p.ext[k];
      const int64_t c = rr % e;
      rr /= e;
#pragma unroll
      for (int v = 0; v < 3; ++v) off[v] += c * p.str[v][k];
    }
  };
  // X chunks of the next tile are prefetched into registers while the
  // current tile is combined and stored (software pipelining)
  constexpr int NP = CHUNKS / 4;
  uint4 pre[NP];
  auto prefetch = [&](int64_t w) {
    int64_t off[3], t0, tq;
    origin(w, off, t0, tq);
    const char* xb = p.base[X] + off[X] + t0 * TT * p.str[X][0] + tq * TT * SX;
#pragma unroll
    for (int pass = 0; pass < NP; ++pass) {
      const int i0 = threadIdx.x % TT, c = threadIdx.x / TT + 4 * pass;
      pre[pass] = __ldcs((const uint4*)(xb + (int64_t)i0 * p.str[X][0] + c * 16));
    }
  };
  if (blockIdx.x < nwork) prefetch(blockIdx.x);
  for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
    int64_t off[3], t0, tq;
    origin(w, off, t0, tq);
    // phase 1: prefetched chunks -> transposed smem tile
#pragma unroll
    for (int pass = 0; pass < NP; ++pass) {
      const int i0 = threadIdx.x % TT, c = threadIdx.x / TT + 4 * pass;
      const TX* e = (const TX*)&pre[pass];
#pragma unroll
      for (int j = 0; j < VX; ++j) sm[c * VX + j][i0] = e[j];
    }
    if (w + gridDim.x < nwork) prefetch(w + gridDim.x);
    __syncthreads();
    // phase 2
    char* db = p.base[0] + off[0] + t0 * TT * SD + tq * TT * p.str[0][q];
    const char* yb = NIN >= 2 ? p.base[Y] + off[Y] + t0 * TT * p.str[Y][0] + tq * TT * p.str[Y][q]
                              : nullptr;
#pragma unroll
    for (int pass = 0; pass < 4; ++pass) {
      const int ig = threadIdx.x % 16, qq = threadIdx.x / 16 + 16 * pass;
      R16 ry[4];
      if (NIN >= 2) {
        if (ymode == 0) {
          ry[0] = ry[1] = ry[2] = ry[3] = p.imm[Y];
        } else if (ymode == 1) {
          ry[0] = load_raw(Y == 1 ? F::dta(p) : F::dtb(p), yb + qq * p.str[Y][q], true);
          ry[1] = ry[2] = ry[3] = ry[0];
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            ry[u] = load_raw(Y == 1 ? F::dta(p) : F::dtb(p),
                             yb + qq * p.str[Y][q] + (int64_t)(ig * 4 + u) * p.str[Y][0], true);
        }
      }
      R16 o[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const R16 rx{(uint64_t)sm[qq][ig * 4 + u], 0};
        o[u] = (X == 1) ? F::apply(p, rx, ry[u], 0, st) : F::apply(p, ry[u], rx, 0, st);
      }
      if (!p.dry) {
        char* dp = db + (int64_t)qq * p.str[0][q] + ig * 4 * SD;
        if constexpr (SD == 4) {
          *(uint4*)dp = make_uint4((uint32_t)o[0].lo, (uint32_t)o[1].lo, (uint32_t)o[2].lo,
                                   (uint32_t)o[3].lo);
        } else if constexpr (SD == 8) {
          *(ulonglong2*)dp = make_ulonglong2(o[0].lo, o[1].lo);
          *(ulonglong2*)(dp + 16) = make_ulonglong2(o[2].lo, o[3].lo);
        } else if constexpr (SD == 2) {
          *(uint2*)dp = make_uint2((uint32_t)(o[0].lo & 0xffff) | ((uint32_t)o[1].lo << 16),
                                   (uint32_t)(o[2].lo & 0xffff) | ((uint32_t)o[3].lo << 16));
        } else {
          *(uint32_t*)dp = (uint32_t)(o[0].lo & 0xff) | ((uint32_t)(o[1].lo & 0xff) << 8) |
                           ((uint32_t)(o[2].lo & 0xff) << 16) | ((uint32_t)(o[3].lo & 0xff) << 24);
        }
      }
    }
    __syncthreads();
  }
  if (st) atomicOr(p.flags, st);
}

// tile_native: the cfg2 family in native float arithmetic.  When every
// operand value is exactly representable in float and the destination is
// float, a float +,-,*,/,min,max is bit-identical to the reference's
// double compute followed by one rounding to float (p_double = 53 >=
// 2*24+2, so the double rounding is innocuous), and NaN inputs give NaN
// either way.  Native types instead of R16 keep registers (occupancy) and
// instruction count low.  No byte swaps, standard mode only.
__host__ __device__ constexpr bool f32_exact(int dt) {
  return dt == TPG_INT8 || dt == TPG_UINT8 || dt == TPG_INT16 || dt == TPG_UINT16 ||
         dt == TPG_HALF || dt == TPG_FLOAT;
}
template <int DT>
struct Native { typedef float T; };
template <>
struct Native<TPG_INT8> { typedef int8_t T; };
template <>
struct Native<TPG_UINT8> { typedef uint8_t T; };
template <>
struct Native<TPG_INT16> { typedef int16_t T; };
template <>
struct Native<TPG_UINT16> { typedef uint16_t T; };
template <>
struct Native<TPG_HALF> { typedef __half T; };

template <typename T>
__device__ __forceinline__ float to_f(T v) { return (float)v; }
template <typename T>
__device__ __forceinline__ T from_bits(uint64_t b) { return (T)b; }
template <>
__device__ __forceinline__ float from_bits<float>(uint64_t b) { return __uint_as_float((uint32_t)b); }
template <>
__device__ __forceinline__ __half from_bits<__half>(uint64_t b) { return __ushort_as_half((uint16_t)b); }
template <>
__device__ __forceinline__ float to_f<__half>(__half v) { return __half2float(v); }

template <int OP>
__device__ __forceinline__ float fop(float a, float b) {
  if (OP == TPG_ADD) return __fadd_rn(a, b);
  if (OP == TPG_SUBTRACT) return __fsub_rn(a, b);
  if (OP == TPG_MULTIPLY) return __fmul_rn(a, b);
  if (OP == TPG_DIVIDE) {
    if (b == 0.0f) {
      if (a == 0.0f || isnan(a)) return __int_as_float(0x7fc00000);
      return copysignf(INFINITY, a) * copysignf(1.0f, b);
    }
    return __fdiv_rn(a, b);
  }
  if (OP == TPG_MINIMUM) return a <= b ? a : b;
  return a >= b ? a : b;
}

// k_tile_f32: the transposing float kernel (SURVEY cfg2).  X (operand XI,
// coalesced along plan axis q) is read a 64(i) x 64(j) tile at a time with
// LPR lanes per tile row, so every warp load covers whole 128-B lines; the
// conversion to float and any Y that is constant along axis 0 (immediate
// or broadcast row) are applied in registers right after the load, and the
// float results go to a shared tile [j][i ^ swz(j)] (XOR swizzle: the
// transposing stores and the float4 reads are both bank-conflict free).
// Phase 2 streams float4 columns to the destination (16-B coalesced
// stores), applying a Y that varies along axis 0 (ymode 2).  Persistent
// grid; the next tile's X chunks (and its Y row slice) are loaded into
// registers before the current tile is stored.
// Y: 0 imm, 1 broadcast along axis 0, 2 unit stride along axis 0;
// NIN == 1: cast-copy of X.
template <int OP, int NIN, int XI, typename TX, typename TY>
__global__ void __launch_bounds__(256, sizeof(TX) >= 4 ? 4 : 5) k_tile_f32(EwParams p, int q, int nt0, int ntq, int ymode) {
  constexpr int SX = sizeof(TX);
  constexpr int VX = 16 / SX;          // X elements per 16-B chunk
  constexpr int LPR = TT * SX / 16;    // lanes per tile row (4, 8 or 16)
  constexpr int RPW = 32 / LPR;        // tile rows per warp load
  constexpr int NLD = TT / (8 * RPW);  // 16-B X loads per thread per tile
  constexpr int SWM = RPW > 4 ? RPW : 4;
  constexpr int Y = 3 - XI;
  __shared__ __align__(16) float sm[TT][TT];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane % LPR;
  const int r0 = warp * RPW + lane / LPR;
  const int swz1 = (c * SWM) & 31;
  // the plan's remaining axes (other than 0 and q) index blockIdx.y
  const char* xs;
  const char* ys = nullptr;
  char* ds;
  {
    int64_t off[3] = {0, 0, 0};
    int64_t rr = blockIdx.y;
    for (int k = 1; k < p.ndim; ++k) {
      if (k == q) continue;
      const int64_t e = p.ext[k];
      const int64_t cc = rr % e;
      rr /= e;
#pragma unroll
      for (int v = 0; v < 3; ++v) off[v] += cc * p.str[v][k];
    }
    xs = p.base[XI] + off[XI];
    if (NIN >= 2) ys = p.base[Y] + off[Y];
    ds = p.base[0] + off[0];
  }
  const int64_t sx0 = p.str[XI][0], sdq = p.str[0][q];
  const int64_t syq = NIN >= 2 ? p.str[Y][q] : 0;
  const int nwork = nt0 * ntq;
  float yimm = 0.0f;
  if (NIN >= 2 && ymode == 0) yimm = to_f<TY>(from_bits<TY>(p.imm[Y].lo));
  uint4 xb[NLD];
  float yr[VX];
  auto load = [&](int w) {
    const int t0 = w % nt0, tq = w / nt0;
    const char* x = xs + (int64_t)(t0 * TT + r0) * sx0 + tq * TT * SX + c * 16;
#pragma unroll
    for (int l = 0; l < NLD; ++l) xb[l] = __ldcs((const uint4*)(x + (int64_t)(l * 8 * RPW) * sx0));
    if (NIN >= 2 && ymode == 1) {
      const char* y = ys + (int64_t)(tq * TT + c * VX) * syq;
#pragma unroll
      for (int k = 0; k < VX; ++k) yr[k] = to_f<TY>(__ldg((const TY*)(y + k * syq)));
    }
  };
  if ((int)blockIdx.x < nwork) load(blockIdx.x);
  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
    // phase 1: registers -> float tile (convert, combine with a row-constant Y)
#pragma unroll
    for (int l = 0; l < NLD; ++l) {
      const int i = r0 + l * 8 * RPW;
      const TX* e = (const TX*)&xb[l];
#pragma unroll
      for (int k = 0; k < VX; ++k) {
        const float x = to_f<TX>(e[k]);
        float v = x;
        if (NIN >= 2 && ymode <= 1) {
          const float y = ymode == 0 ? yimm : yr[k];
          v = XI == 1 ? fop<OP>(x, y) : fop<OP>(y, x);
        }
        sm[c * VX + k][i ^ swz1] = v;
      }
    }
    __syncthreads();
    const int t0 = w % nt0, tq = w / nt0;
    if (w + (int)gridDim.x < nwork) load(w + gridDim.x);
    // phase 2: float4 columns -> destination
    const int ig = threadIdx.x % 16;
    char* db = ds + (int64_t)(t0 * TT + ig * 4) * 4 + (int64_t)(tq * TT) * sdq;
#pragma unroll
    for (int pass = 0; pass < 4; ++pass) {
      const int j = threadIdx.x / 16 + 16 * pass;
      const int swz = ((j / VX) * SWM) & 31;
      float4 f = *(const float4*)&sm[j][(ig * 4) ^ swz];
      if (NIN >= 2 && ymode == 2) {
        const int64_t sy0 = p.str[Y][0];
        const char* yb = ys + (int64_t)(t0 * TT + ig * 4) * sy0 + (int64_t)(tq * TT + j) * syq;
        float y[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) y[u] = to_f<TY>(__ldg((const TY*)(yb + u * sy0)));
        if (XI == 1) {
          f.x = fop<OP>(f.x, y[0]); f.y = fop<OP>(f.y, y[1]);
          f.z = fop<OP>(f.z, y[2]); f.w = fop<OP>(f.w, y[3]);
        } else {
          f.x = fop<OP>(y[0], f.x); f.y = fop<OP>(y[1], f.y);
          f.z = fop<OP>(y[2], f.z); f.w = fop<OP>(y[3], f.w);
        }
      }
      __stcs((float4*)(db + j * sdq), f);
    }
    __syncthreads();
  }
}

// k_tile_tma: the transposing float kernel fed by TMA (SURVEY cfg2, the
// headline; the default for 1-, 2- and 4-byte X; 1-byte X uses 64-B
// swizzled boxes and two warps per 16-B chunk).  The X operand is a 2-D
// tensor map over its memory order (reversed plan axes are handled by
// mirrored tile coordinates and index flips); each 64 x 64 X tile arrives
// by TMA (one box per 128 B of a tile row, 128-B swizzle) in an XS-stage
// shared-memory ring, one mbarrier per stage, thread 0 issuing XS tiles
// ahead.  There is no float staging tile: lane l of a warp owns output row
// i0 + l, reads the 16-B chunk of X row i0 + l holding VX adjacent output
// columns (the swizzle spreads the 8 rows of a 128-B bank window over all
// banks, so the 32-row column read is conflict free), converts, combines
// with Y and stores each column as ONE 128-B line per warp instruction
// (st.global.cs).  Measured against the register-staged k_tile_f32 and
// 30+ other transposing shapes in scripts/ubench_cfg2_tma.cu /
// ubench_tile_rot.cu: the fastest steady-state cfg2 kernel found.
// Y: 0 imm, 1 broadcast along axis 0, 2 unit stride along axis 0;
// NIN == 1: cast-copy of X.
constexpr int XS = 6;

__device__ __forceinline__ void tma_mbar_wait(uint32_t bar, uint32_t parity) {
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

template <int OP, int NIN, int XI, typename TX, typename TY>
__global__ void __launch_bounds__(256, 4) k_tile_tma(const __grid_constant__ CUtensorMap xmap,
                                                  EwParams p, int q, int nt0, int ntq, int ymode,
                                                  int rev0, int revq) {
  constexpr int SX = sizeof(TX);
  static_assert(SX == 1 || SX == 2 || SX == 4, "1-, 2- or 4-byte X");
  constexpr int VX = 16 / SX;           // X elements per 16-B chunk
  constexpr int ROWB = SX == 1 ? 64 : 128;  // bytes per box row (64- / 128-B swizzle)
  constexpr int BQ = ROWB / SX;         // box width (elements along q)
  constexpr int NB = TT / BQ;           // boxes per tile
  constexpr int BOX = TT * ROWB;        // bytes per box
  constexpr int STAGE = NB * BOX;       // = TT * TT * SX
  constexpr int NCH = TT / VX;          // 16-B chunks per tile row (4, 8 or 16)
  constexpr int CPB = ROWB / 16;        // chunks per box row
  // warps per chunk (1-byte X: 4 chunks, so two warps share one, one row
  // group each) and row groups per warp
  constexpr int WPC = NCH >= 8 ? 1 : 8 / NCH;
  constexpr int RGW = 2 / WPC;
  constexpr int Y = 3 - XI;
  extern __shared__ uint8_t tsm_raw[];
  uint8_t* xring = (uint8_t*)(((uintptr_t)tsm_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = (uint64_t*)(xring + XS * STAGE);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwork = nt0 * ntq;
  const char* ys = NIN >= 2 ? p.base[Y] : nullptr;
  char* ds = p.base[0];
  const int64_t sdq = p.str[0][q];
  const int64_t syq = NIN >= 2 ? p.str[Y][q] : 0;
  const int64_t sy0 = NIN >= 2 ? p.str[Y][0] : 0;
  float yimm = 0.0f;
  if (NIN >= 2 && ymode == 0) yimm = to_f<TY>(from_bits<TY>(p.imm[Y].lo));
  // byte step between the VX plan columns of a chunk (memory order)
  const int64_t dstep = revq ? -sdq : sdq, ystep = revq ? -syq : syq;
  auto issue = [&](int w, int s) {
    const int t0 = w % nt0, tq = w / nt0;
    const int mq = revq ? (ntq - 1 - tq) * TT : tq * TT;
    const int m0 = rev0 ? (nt0 - 1 - t0) * TT : t0 * TT;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(STAGE)
                 : "memory");
#pragma unroll
    for (int k = 0; k < NB; ++k)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
          "[%0], [%1, {%2, %3}], [%4];" ::"r"(
              (uint32_t)__cvta_generic_to_shared(xring + s * STAGE + k * BOX)),
          "l"((uint64_t)&xmap), "r"(mq + k * BQ), "r"(m0), "r"(b)
          : "memory");
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < XS; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
          (uint32_t)__cvta_generic_to_shared(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&xmap) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int w = blockIdx.x;
    for (int s = 0; s < XS && w < nwork; ++s, w += gridDim.x) issue(w, s);
  }
  // per-thread constants: warp w owns chunks w, w + 8, ... (CPW of them) of
  // every tile, for both 32-row groups (lane = output row i and i + 32, so
  // each column address serves two stores, the second at +128 B):
  // shared-memory offsets of the lane's 16-B chunk rows, and the byte offset
  // of each chunk's first plan column from the tile origin
  constexpr int CPW = NCH >= 8 ? NCH / 8 : 1;
  constexpr int WSTEP = 8 / WPC;                             // warps per pass over the chunks
  const int g0w = (warp / WSTEP) * RGW;                      // first row group of this warp
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(xring);
  uint32_t soff[CPW][RGW];
  int64_t dofs[CPW], yofs[CPW];
#pragma unroll
  for (int u = 0; u < CPW; ++u) {
    const int ch = warp % WSTEP + WSTEP * u;                 // chunk (memory order)
#pragma unroll
    for (int k = 0; k < RGW; ++k) {
      const int i = 32 * (g0w + k) + lane;                   // plan row (output fast axis)
      const int rm = rev0 ? TT - 1 - i : i;                  // memory row in the tile
      const int c = ch % CPB;
      const int pos = ROWB == 128 ? (c ^ (rm & 7)) : (c ^ ((rm >> 1) & 3));  // TMA swizzle
      soff[u][k] = (uint32_t)((ch / CPB) * BOX + rm * ROWB + (pos << 4));
    }
    const int jm0 = ch * VX;                                 // memory column of the chunk
    const int jl = revq ? TT - 1 - jm0 : jm0;                // its plan column in the tile
    dofs[u] = (int64_t)(32 * g0w + lane) * 4 + jl * sdq;
    yofs[u] = jl * syq + (ymode == 2 ? (int64_t)(32 * g0w + lane) * sy0 : 0);
  }
  // ymode 1 with a float row of unit stride (either sign) along q: each
  // chunk's VX row values are one aligned 16-32 B run, read as float4s
  // (chunks cover plan columns 8m .. 8m+7 (VX = 8) or 4m .. 4m+3 (VX = 4))
  bool yvec = false, yrev = false;
  if constexpr (NIN >= 2 && std::is_same<TY, float>::value) {
    yrev = revq != (syq < 0);
    yvec = ymode == 1 && (syq == 4 || syq == -4) &&
           (syq > 0 ? (uintptr_t)ys % 16 == 0 : ((uintptr_t)ys + 4) % 16 == 0);
  }
  int it = 0;
  // tile coordinates advanced incrementally (no per-tile division)
  int t0 = (int)blockIdx.x % nt0, tq = (int)blockIdx.x / nt0;
  const int g0 = (int)gridDim.x % nt0, gq = (int)gridDim.x / nt0;
  for (int w = blockIdx.x; w < nwork; w += gridDim.x, ++it) {
    const int s = it % XS;
    tma_mbar_wait(sbase + XS * STAGE + s * 8, (it / XS) & 1);
    char* dtile = ds + (int64_t)t0 * TT * 4 + (int64_t)tq * TT * sdq;
    const char* ytile = nullptr;
    if (NIN >= 2) ytile = ys + (int64_t)tq * TT * syq + (ymode == 2 ? (int64_t)t0 * TT * sy0 : 0);
#pragma unroll
    for (int u = 0; u < CPW; ++u) {
      uint4 raw[RGW];
#pragma unroll
      for (int g = 0; g < RGW; ++g)
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(raw[g].x), "=r"(raw[g].y), "=r"(raw[g].z), "=r"(raw[g].w)
                     : "r"(sbase + s * STAGE + soff[u][g]));
      char* dp = dtile + dofs[u];
      float yv[RGW][VX];
      if (NIN >= 2) {
        if (ymode == 0) {
#pragma unroll
          for (int k = 0; k < VX; ++k)
#pragma unroll
            for (int g = 0; g < RGW; ++g) yv[g][k] = yimm;
        } else if (yvec) {
          const float* yp = (const float*)(ytile + yofs[u]) - (yrev ? VX - 1 : 0);
          float t[VX];
#pragma unroll
          for (int h = 0; h < VX / 4; ++h) {
            const float4 f = __ldg((const float4*)yp + h);
            t[4 * h] = f.x; t[4 * h + 1] = f.y; t[4 * h + 2] = f.z; t[4 * h + 3] = f.w;
          }
#pragma unroll
          for (int k = 0; k < VX; ++k)
#pragma unroll
            for (int g = 0; g < RGW; ++g) yv[g][k] = t[yrev ? VX - 1 - k : k];
        } else {
          const char* yp = ytile + yofs[u];
#pragma unroll
          for (int g = 0; g < RGW; ++g) {
            const char* ypg = yp + (ymode == 2 ? g * 32 * sy0 : 0);
#pragma unroll
            for (int k = 0; k < VX; ++k) yv[g][k] = to_f<TY>(__ldg((const TY*)(ypg + k * ystep)));
          }
        }
      }
#pragma unroll
      for (int k = 0; k < VX; ++k) {
        float* col = (float*)(dp + k * dstep);
#pragma unroll
        for (int g = 0; g < RGW; ++g) {
          const float x = to_f<TX>(((const TX*)&raw[g])[k]);
          float v = x;
          if (NIN >= 2) v = XI == 1 ? fop<OP>(x, yv[g][k]) : fop<OP>(yv[g][k], x);
          __stcs(col + 32 * g, v);
        }
      }
    }
    __syncthreads();  // stage s consumed by every warp
    if (threadIdx.x == 0) {
      const int wn = w + XS * gridDim.x;
      if (wn < nwork) issue(wn, s);
    }
    t0 += g0;
    tq += gq;
    if (t0 >= nt0) {
      t0 -= nt0;
      ++tq;
    }
  }
}

template <int SX>
constexpr size_t tile_tma_smem() {
  return (size_t)XS * TT * TT * SX + XS * 8 + 1024;
}

// TMA launch of the cfg2 pattern: 2-D plan, X unit-stride (+-) along q,
// 16-B multiple row stride, element size <= 4.  Returns false when the
// layout is not eligible or the map cannot be encoded (caller falls back).
template <auto K, typename TX>
bool launch_tile_tma(EwParams& p, Stream* st, int xi, int q, int64_t nt0, int64_t ntq, int ymode) {
  constexpr int SX = sizeof(TX);
  if ((SX != 1 && SX != 2 && SX != 4) || p.ndim != 2) return false;
  const int64_t sq = p.str[xi][q], s0 = p.str[xi][0];
  if ((sq != SX && sq != -SX) || s0 == 0 || (s0 < 0 ? -s0 : s0) % 16) return false;
  const int64_t eq = p.ext[q], e0 = p.ext[0];
  const char* lo = p.base[xi] + (sq < 0 ? (eq - 1) * sq : 0) + (s0 < 0 ? (e0 - 1) * s0 : 0);
  if ((uintptr_t)lo % 16) return false;
  // encoded maps are reused across launches over the same X layout (a
  // small per-thread cache: the host cost of an op is part of its e2e time)
  struct MapCache {
    const char* lo;
    int64_t eq, e0, s0, sx;
    CUtensorMap map;
  };
  static thread_local MapCache cache[8];
  static thread_local unsigned next = 0;
  const int64_t s0a = s0 < 0 ? -s0 : s0;
  const CUtensorMap* mp = nullptr;
  for (auto& c : cache)
    if (c.lo == lo && c.eq == eq && c.e0 == e0 && c.s0 == s0a && c.sx == SX) mp = &c.map;
  if (!mp) {
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)tensor_map_encoder();
    if (!enc) return false;
    MapCache& c = cache[next++ % 8];
    cuuint64_t dims[2] = {(cuuint64_t)eq, (cuuint64_t)e0};
    cuuint64_t strides[1] = {(cuuint64_t)s0a};
    cuuint32_t box[2] = {(cuuint32_t)((SX == 1 ? 64 : 128) / SX), TT};
    cuuint32_t estr[2] = {1, 1};
    const CUtensorMapDataType ty = SX == 1   ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                   : SX == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                             : CU_TENSOR_MAP_DATA_TYPE_UINT32;
    c.lo = nullptr;
    if (enc(&c.map, ty, 2, const_cast<char*>(lo), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE,
            SX == 1 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
    c.lo = lo;
    c.eq = eq;
    c.e0 = e0;
    c.s0 = s0a;
    c.sx = SX;
    mp = &c.map;
  }
  const CUtensorMap& map = *mp;
  constexpr size_t smem = tile_tma_smem<SX>();
  static int bps = 0;
  if (!bps) {
    if (cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return false;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, K, 256, smem) != cudaSuccess || n < 1)
      n = 1;
    bps = n;
  }
  const int64_t slots = (int64_t)sm_count(st->device) * bps;
  const int grid = (int)std::min<int64_t>(nt0 * ntq, slots);
  K<<<grid, 256, smem, st->s>>>(map, p, q, (int)nt0, (int)ntq, ymode, s0 < 0 ? 1 : 0,
                                sq < 0 ? 1 : 0);
  return true;
}

// The TMA-fed tile kernel is the default for 1-, 2- and 4-byte X (TPG_TILE_TMA=0
// selects the register-staged k_tile_f32 instead, for A/B runs).
inline bool tile_tma_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TPG_TILE_TMA");
    v = (e && e[0] == '0') ? 1 : 0;
  }
  return v == 1;
}

// resident blocks per SM of kernel K at 256 threads (queried once per K)
template <auto K>
int blocks_per_sm() {
  static int cached = 0;
  if (!cached) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, K, 256, 0) != cudaSuccess || n < 1) n = 4;
    cached = n;
  }
  return cached;
}

// persistent launch of k_tile_f32: grid.x sized to the resident slots,
// grid.y = index over the plan's remaining axes
template <auto K>
void launch_tile_f32(EwParams& p, Stream* st, int q, int64_t nt0, int64_t ntq, int64_t nrest,
                     int ymode) {
  const int64_t slots =
      std::max<int64_t>(1, (int64_t)sm_count(st->device) * blocks_per_sm<K>() / nrest);
  const dim3 grid((unsigned)std::min<int64_t>(nt0 * ntq, slots), (unsigned)nrest);
  K<<<grid, 256, 0, st->s>>>(p, q, (int)nt0, (int)ntq, ymode);
}

// contig: 1-D unit-stride views, compile-time element sizes; 8 elements per
// thread per operand moved with the widest aligned vector accesses.
constexpr int CV = 8;

template <int S>
__device__ __forceinline__ void load_vec(const char* ptr, R16 (&o)[CV]) {
  constexpr int B = S * CV;
  if constexpr (B >= 16) {
    uint32_t w[B / 4];
#pragma unroll
    for (int i = 0; i < B / 16; ++i) {
      uint4 v = __ldcs((const uint4*)ptr + i);  // streaming: read once
      w[4 * i] = v.x; w[4 * i + 1] = v.y; w[4 * i + 2] = v.z; w[4 * i + 3] = v.w;
    }
#pragma unroll
    for (int j = 0; j < CV; ++j) {
      if constexpr (S == 16) {
        o[j].lo = w[4 * j] | ((uint64_t)w[4 * j + 1] << 32);
        o[j].hi = w[4 * j + 2] | ((uint64_t)w[4 * j + 3] << 32);
      } else if constexpr (S == 8) {
        o[j].lo = w[2 * j] | ((uint64_t)w[2 * j + 1] << 32);
        o[j].hi = 0;
      } else if constexpr (S == 4) {
        o[j].lo = w[j];
        o[j].hi = 0;
      } else {  // S == 2
        o[j].lo = (w[j / 2] >> (16 * (j % 2))) & 0xffffu;
        o[j].hi = 0;
      }
    }
  } else {  // S == 1: 8 bytes
    uint2 v = __ldcs((const uint2*)ptr);
#pragma unroll
    for (int j = 0; j < CV; ++j) {
      o[j].lo = ((j < 4 ? v.x : v.y) >> (8 * (j % 4))) & 0xffu;
      o[j].hi = 0;
    }
  }
}

template <int S>
__device__ __forceinline__ void store_vec(char* ptr, const R16 (&o)[CV]) {
  constexpr int B = S * CV;
  if constexpr (B >= 16) {
    uint32_t w[B / 4];
#pragma unroll
    for (int j = 0; j < CV; ++j) {
      if constexpr (S == 16) {
        w[4 * j] = (uint32_t)o[j].lo; w[4 * j + 1] = (uint32_t)(o[j].lo >> 32);
        w[4 * j + 2] = (uint32_t)o[j].hi; w[4 * j + 3] = (uint32_t)(o[j].hi >> 32);
      } else if constexpr (S == 8) {
        w[2 * j] = (uint32_t)o[j].lo; w[2 * j + 1] = (uint32_t)(o[j].lo >> 32);
      } else if constexpr (S == 4) {
        w[j] = (uint32_t)o[j].lo;
      } else {  // S == 2
        if (j % 2 == 0) w[j / 2] = (uint32_t)o[j].lo & 0xffffu;
        else w[j / 2] |= ((uint32_t)o[j].lo & 0xffffu) << 16;
      }
    }
#pragma unroll
    for (int i = 0; i < B / 16; ++i)
      __stcs((uint4*)ptr + i, make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]));
  } else {
    uint32_t x = 0, y = 0;
#pragma unroll
    for (int j = 0; j < CV; ++j) {
      uint32_t b = (uint32_t)o[j].lo & 0xffu;
      if (j < 4) x |= b << (8 * j); else y |= b << (8 * (j - 4));
    }
    __stcs((uint2*)ptr, make_uint2(x, y));
  }
}

template <class F, int NIN, int SD, int SA, int SB>
__global__ void __launch_bounds__(256) k_contig(EwParams p, int64_t n) {
  uint32_t st = 0;
  const int64_t nchunk = n / CV;
  const int64_t tid = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * 256;
  const bool bca = NIN >= 1 && (p.isimm[1] || p.str[1][0] == 0);
  const bool bcb = NIN >= 2 && (p.isimm[2] || p.str[2][0] == 0);
  R16 sa{0, 0}, sb{0, 0};
  if (NIN >= 1 && bca) sa = ld_op<F, 1>(p, 0);
  if (NIN >= 2 && bcb) sb = ld_op<F, 2>(p, 0);
  for (int64_t c = tid; c < nchunk; c += nthreads) {
    R16 a[CV], b[CV], o[CV];
    if (NIN >= 1) {
      if (bca) {
#pragma unroll
        for (int j = 0; j < CV; ++j) a[j] = sa;
      } else {
        load_vec<SA>(p.base[1] + c * (CV * SA), a);
      }
    }
    if (NIN >= 2) {
      if (bcb) {
#pragma unroll
        for (int j = 0; j < CV; ++j) b[j] = sb;
      } else {
        load_vec<SB>(p.base[2] + c * (CV * SB), b);
      }
    }
#pragma unroll
    for (int j = 0; j < CV; ++j)
      o[j] = F::apply(p, NIN >= 1 ? a[j] : sa, NIN >= 2 ? b[j] : sb, c * CV + j, st);
    if (!p.dry) store_vec<SD>(p.base[0] + c * (CV * SD), o);
  }
  // tail
  for (int64_t i = nchunk * CV + tid; i < n; i += nthreads) {
    R16 a{0, 0}, b{0, 0};
    if (NIN >= 1) a = bca ? sa : load_raw(F::dta(p), p.base[1] + i * SA, true);
    if (NIN >= 2) b = bcb ? sb : load_raw(F::dtb(p), p.base[2] + i * SB, true);
    R16 o = F::apply(p, a, b, i, st);
    if (!p.dry) store_raw(F::dtd(p), p.base[0] + i * SD, o, true);
  }
  if (st) atomicOr(p.flags, st);
}

// ------------------------------------------------------------ host side
struct Choice {
  int kind;  // 0 contig, 1 tile, 2 rows, 3 flat
  int x, q;
};

inline int64_t plan_total(const EwParams& p) {
  int64_t t = 1;
  for (int k = 0; k < p.ndim; ++k) t *= p.ext[k];
  return t;
}

inline Choice choose_traversal(const EwParams& p, bool typed, int oc) {
  const int nin = p.nin;
  if (typed && p.ndim == 1) {
    bool ok = true;
    for (int v = 0; v <= nin; ++v) {
      if (v > 0 && (p.isimm[v] || p.str[v][0] == 0)) continue;
      const int s = dt_size(p.dt[v]);
      const int al = std::min(16, s * CV);
      if (p.str[v][0] != s || ((uintptr_t)p.base[v] % al) != 0) ok = false;
    }
    if (ok) return Choice{0, 0, 0};
  }
  if (oc == OC_BINARY || oc == OC_UNARY || oc == OC_COPY || oc == OC_RAW) {
    for (int x = 1; x <= nin; ++x) {
      if (p.isimm[x]) continue;
      const int s = dt_size(p.dt[x]);
      if (s > 8) continue;
      const int64_t s0 = p.str[x][0] < 0 ? -p.str[x][0] : p.str[x][0];
      if (s0 <= 2 * s || p.ext[0] < 16) continue;
      int best = -1;
      int64_t bs = 0;
      for (int k = 1; k < p.ndim; ++k) {
        if (p.ext[k] < 16) continue;
        const int64_t sk = p.str[x][k] < 0 ? -p.str[x][k] : p.str[x][k];
        if (sk == 0) continue;
        if (best < 0 || sk < bs) { best = k; bs = sk; }
      }
      if (best > 0 && bs <= 2 * s && bs < s0) return Choice{1, x, best};
    }
  }
  if (p.ext[0] >= 128 || p.ndim <= 1) return Choice{2, 0, 0};
  return Choice{3, 0, 0};
}

inline int grid_for(int64_t work, int dev, int per_sm) {
  int64_t cap = (int64_t)sm_count(dev) * per_sm;
  int64_t g = work < cap ? work : cap;
  return (int)(g < 1 ? 1 : g);
}

// Launch one (op class, op, kind, dtypes) configuration.  Typed (Tier A)
// instantiations compile contig/tile/rows; the flat traversal (short axis
// 0, rare) always goes through the Tier B kernel of the same class/kind.
template <int OC, int NIN, int OP, int KIND, int DTD, int DTA, int DTB>
int launch_ew(EwParams& p, Stream* st) {
  typedef Ew<OC, NIN, OP, KIND, DTD, DTA, DTB> F;
  constexpr bool typed = F::typed;
  const int64_t total = plan_total(p);
  if (total == 0) return TPG_OK;
  Choice c = choose_traversal(p, typed, OC);
  const int dev = st->device;
  if (c.kind == 0) {
    if constexpr (typed) {
      constexpr int SD = dt_size(DTD);
      constexpr int SA = DTA >= 0 ? dt_size(DTA) : 1;
      constexpr int SB = DTB >= 0 ? dt_size(DTB) : 1;
      const int64_t n = p.ext[0];
      // grid: one CV-element chunk per thread (no grid-stride loop) when a
      // thread moves >= 48 B, else a persistent grid of 8 waves of resident
      // blocks (occupancy calculator).  Measured on cfg5 2^30 (r01d,
      // profiles/r01d_contig_grid.md): cast f64-BE -> f32 5.9 -> 7.0 TB/s,
      // scalar multiply / add 5.7 -> 6.2 TB/s one chunk per thread; int16-BE
      // -> half (16 B in, 16 B out per thread) is best persistent
      constexpr int TB = (SD + (NIN >= 1 ? SA : 0) + (NIN >= 2 ? SB : 0)) * CV;
      const int64_t chunks = (n / CV + 255) / 256;
      int g;
      if (TB >= 48) {
        g = (int)std::max<int64_t>(1, std::min<int64_t>(chunks, 1 << 30));
      } else {
        static int occ = 0;
        if (!occ) {
          if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_contig<F, NIN, SD, SA, SB>, 256, 0) !=
                  cudaSuccess || occ < 1)
            occ = 1;
        }
        g = grid_for(chunks, dev, occ * 8);
      }
      k_contig<F, NIN, SD, SA, SB><<<g, 256, 0, st->s>>>(p, n);
    }
  } else if (c.kind == 1) {
    if constexpr (NIN >= 1) {
      const int64_t nt0 = (p.ext[0] + TT - 1) / TT, ntq = (p.ext[c.q] + TT - 1) / TT;
      const int64_t nrest = total / (p.ext[0] * p.ext[c.q]);
      // one 64x64 tile per block where possible: more independent tiles
      // in flight per SM than a persistent loop (measured, scripts/ubench.cu)
      const int g = grid_for(nt0 * ntq * nrest, dev, 32);
      if constexpr (typed) {
        constexpr int SD = dt_size(DTD);
        constexpr int SA = DTA >= 0 ? dt_size(DTA) : 1;
        constexpr int SB = DTB >= 0 ? dt_size(DTB) : 1;
        const int x = c.x, y = 3 - x, qa = c.q;
        const int sx = x == 1 ? SA : SB;
        bool fast = p.ext[0] % TT == 0 && p.ext[qa] % TT == 0 && p.str[0][0] == SD &&
                    (uintptr_t)p.base[0] % 16 == 0 && p.str[0][qa] % 16 == 0 &&
                    p.str[x][qa] == sx && (uintptr_t)p.base[x] % 16 == 0 && p.str[x][0] % 16 == 0 &&
                    SD <= 8 && sx <= 8;
        for (int k = 1; k < p.ndim && fast; ++k)
          if (k != qa && (p.str[0][k] % 16 || p.str[x][k] % 16)) fast = false;
        int ymode = 0;
        if (NIN >= 2 && fast) {
          const int sy = y == 1 ? SA : SB;
          if (p.isimm[y]) ymode = 0;
          else if (p.str[y][0] == 0) ymode = 1;
          else if (p.str[y][0] == sy) ymode = 2;
          else fast = false;
          if (ymode > 0 && ((uintptr_t)p.base[y] % sy)) fast = false;
        }
        const bool plain = !p.swap[0] && !p.swap[1] && !p.swap[2] && !p.track && !p.dry;
        if constexpr (DTD == TPG_FLOAT && f32_exact(DTA) && (NIN < 2 || f32_exact(DTB)) &&
                      ((OC == OC_BINARY && KIND == K_FLT) || OC == OC_COPY)) {
          if (fast && plain && nrest <= 65535 && nt0 * ntq < (1 << 30)) {
            typedef typename Native<DTA>::T TA;
            typedef typename Native<(NIN >= 2 ? DTB : DTA)>::T TB;
            if (nrest == 1 && !tile_tma_disabled()) {
              bool ok = false;
              constexpr bool ta_ok = sizeof(TA) <= 4 && sizeof(TA) != 3;
              constexpr bool tb_ok = sizeof(TB) <= 4 && sizeof(TB) != 3;
              if constexpr (ta_ok) {
                if (NIN == 1)
                  ok = launch_tile_tma<k_tile_tma<0, 1, 1, TA, TA>, TA>(p, st, 1, qa, nt0, ntq, 0);
                else if (x == 1)
                  ok = launch_tile_tma<k_tile_tma<OP, 2, 1, TA, TB>, TA>(p, st, 1, qa, nt0, ntq, ymode);
              }
              if constexpr (tb_ok && NIN >= 2) {
                if (x == 2)
                  ok = launch_tile_tma<k_tile_tma<OP, 2, 2, TB, TA>, TB>(p, st, 2, qa, nt0, ntq, ymode);
              }
              if (ok) {
                TPG_LAUNCH_CHECK("tile_tma launch");
                return TPG_OK;
              }
            }
            if (NIN == 1)
              launch_tile_f32<k_tile_f32<0, 1, 1, TA, TA>>(p, st, qa, nt0, ntq, nrest, 0);
            else if (x == 1)
              launch_tile_f32<k_tile_f32<OP, 2, 1, TA, TB>>(p, st, qa, nt0, ntq, nrest, ymode);
            else
              launch_tile_f32<k_tile_f32<OP, 2, 2, TB, TA>>(p, st, qa, nt0, ntq, nrest, ymode);
            TPG_LAUNCH_CHECK("tile_f32 launch");
            return TPG_OK;
          }
        }
        if (fast) {
          if constexpr (SD <= 8 && SA <= 8 && SB <= 8) {
            if (x == 1) k_tile_fast<F, NIN, 1, SD, SA, SB><<<g, 256, 0, st->s>>>(p, qa, nt0, ntq, nrest, ymode);
            else if constexpr (NIN >= 2) k_tile_fast<F, NIN, 2, SD, SB, SA><<<g, 256, 0, st->s>>>(p, qa, nt0, ntq, nrest, ymode);
            TPG_LAUNCH_CHECK("tile_fast launch");
            return TPG_OK;
          }
        }
      }
      if (c.x == 1) {
        k_tile<F, NIN, 1><<<g, 256, 0, st->s>>>(p, c.q, nt0, ntq, nrest);
      } else {
        if constexpr (NIN >= 2) k_tile<F, NIN, 2><<<g, 256, 0, st->s>>>(p, c.q, nt0, ntq, nrest);
      }
    }
  } else if (c.kind == 2) {
    constexpr int U = 4;
    const int64_t rows = total / p.ext[0];
    const int64_t ntile = (p.ext[0] + 256 * U - 1) / (256 * U);
    const int g = grid_for(rows * ntile, dev, 16);
    k_rows<F, NIN, U><<<g, 256, 0, st->s>>>(p, rows, ntile);
  } else {
    typedef Ew<OC, NIN, -1, KIND, -1, -1, -1> G;
    if (OP >= 0) p.op = OP;  // generic kernels read op from params
    const int g = grid_for((total + 255) / 256, dev, 16);
    k_flat<G, NIN><<<g, 256, 0, st->s>>>(p, total);
  }
  TPG_LAUNCH_CHECK("elementwise launch");
  return TPG_OK;
}

// entry points implemented in the tpg_ewise_*.cu units
int ew_dispatch_fast(int oc, int op, int kind, EwParams& p, Stream* st, bool* done);
int ew_dispatch_generic_binary(int kind, EwParams& p, Stream* st);
int ew_dispatch_generic_unary(int kind, EwParams& p, Stream* st);
int ew_dispatch_generic_copy(int kind, EwParams& p, Stream* st);
int ew_dispatch_misc(int oc, EwParams& p, Stream* st);

}  // namespace tpg
