// tpg_reduce.cuh — axis and full reductions (shared by tpg_reduce_*.cu).
//
// Replaces kernels.reduce_strided (pkg/src/tidepool/kernels.py:305-320)
// driven by ops.reduce (ops.py:437-513) with the accumulators of
// ops._reduction_acc (ops.py:522-556), kernels.make_sum_acc (169-198) and
// make_product_acc (201-206).  The outer plan walks (dest, src base); the
// inner plan walks the reduced source axes.
//
// Semantics kept from the reference:
//   sum      floats/complex: compensated (the reference uses Neumaier in
//            double; here each partial is a double-double TwoSum accumulator,
//            at least as accurate), ints: exact then wrapped (mod 2^64 is
//            exact after the final wrap).
//   product  plain double / complex / wrapped-int product.
//   min/max  `v if acc is None or v < acc`: the result is NaN iff the first
//            element in plan order is NaN, otherwise the extreme over the
//            non-NaN elements, ties keep the earliest element.
//   any/all  `v != 0` (NaN is truthy).
//   norm     (sum |v|^p)^(1/p) in double.
// Work split: each output's inner range is cut into C chunks; a block (row
// mode: inner axis coalesced) or a thread (column mode: outputs coalesced)
// produces one partial per (output, chunk); a finalize pass combines the C
// partials of each output in a fixed order, so results are deterministic.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>

#include "tpg_common.cuh"
#include "tpg_internal.h"

namespace tpg {

struct Acc {
  double a, b, c, d;  // float / complex payload (double-double pairs)
  int64_t i;          // index of the selected element (min/max), -1 = none
  int64_t v;          // integer payload
};

struct RedParams {
  int ndo, ndi;
  int64_t eo[TPG_MAX_DIMS];
  int64_t so_d[TPG_MAX_DIMS], so_s[TPG_MAX_DIMS];
  int64_t ei[TPG_MAX_DIMS];
  int64_t si[TPG_MAX_DIMS];
  char* dbase;
  const char* sbase;
  int ddt, sdt, dswap, sswap, daligned, saligned;
  int track;
  double p;
  uint32_t* flags;
  int64_t O, N, C, chunk;
  Acc* ws;
  // fused peer-memory finish of a full sum (tpg_reduce_sum_p2p): mailboxes
  // of every rank, or nullptr
  P2pSlot** p2p;
  int p2p_rank, p2p_world;
  unsigned long long p2p_epoch;
  int64_t p2p_index_base;  // min / max: global plan index of this rank's element 0
};

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
__device__ __forceinline__ void dd_merge(double& hi, double& lo, double hi2, double lo2) {
  double s, e;
  two_sum(hi, hi2, s, e);
  hi = s;
  lo = __dadd_rn(lo, __dadd_rn(lo2, e));
}

template <int OP, int KIND>
__device__ __forceinline__ Acc acc_init() {
  Acc x;
  x.a = x.b = x.c = x.d = 0.0;
  x.i = -1;
  x.v = 0;
  if (OP == TPG_RPRODUCT) {
    x.a = 1.0;
    x.v = 1;
  }
  if (OP == TPG_RALL) x.v = 1;
  return x;
}

__device__ __forceinline__ bool cpx_nonzero(double2 z) { return z.x != 0.0 || z.y != 0.0; }

// fold one element (plan index idx) into acc
template <int OP, int KIND>
__device__ __forceinline__ void acc_feed(Acc& x, const RedParams& p, int sdt, R16 r, int64_t idx) {
  if (p.sswap) r = swap_raw(sdt, r);
  if (OP == TPG_RSUM) {
    if (KIND == K_INT || KIND == K_UINT) x.v = (int64_t)((uint64_t)x.v + (uint64_t)dec_int(sdt, r));
    else if (KIND == K_FLT) dd_add(x.a, x.b, dec_flt(sdt, r));
    else {
      double2 z = dec_cpx(sdt, r);
      dd_add(x.a, x.b, z.x);
      dd_add(x.c, x.d, z.y);
    }
  } else if (OP == TPG_RPRODUCT) {
    if (KIND == K_INT || KIND == K_UINT) x.v = (int64_t)((uint64_t)x.v * (uint64_t)dec_int(sdt, r));
    else if (KIND == K_FLT) x.a = __dmul_rn(x.a, dec_flt(sdt, r));
    else {
      double2 z = dec_cpx(sdt, r);
      const double re = __dsub_rn(__dmul_rn(x.a, z.x), __dmul_rn(x.c, z.y));
      const double im = __dadd_rn(__dmul_rn(x.a, z.y), __dmul_rn(x.c, z.x));
      x.a = re;
      x.c = im;
    }
  } else if (OP == TPG_RMIN || OP == TPG_RMAX) {
    const bool mn = OP == TPG_RMIN;
    if (KIND == K_INT || KIND == K_UINT) {
      const int64_t v = dec_int(sdt, r);
      bool take;
      if (x.i < 0) take = true;
      else if (KIND == K_UINT) take = mn ? (uint64_t)v < (uint64_t)x.v : (uint64_t)v > (uint64_t)x.v;
      else take = mn ? v < x.v : v > x.v;
      if (take) { x.v = v; x.i = idx; }
    } else if (KIND == K_FLT) {
      const double v = dec_flt(sdt, r);
      if (isnan(v)) {
        // first element NaN sticks; p < 0 selects the NaN-skipping variant
        // used for per-shard partials (sharded.py)
        if (idx == 0 && p.p >= 0.0) { x.b = 1.0; x.d = v; }
        return;
      }
      if (x.i < 0 || (mn ? v < x.a : v > x.a)) { x.a = v; x.i = idx; }
    } else {
      const double2 z = dec_cpx(sdt, r);
      if (isnan(z.x)) {
        if (idx == 0) { x.b = 1.0; x.d = z.x; x.v = (int64_t)__double_as_longlong(z.y); }
        return;
      }
      const double2 cur = make_double2(x.a, x.c);
      if (x.i < 0 || (mn ? cpx_lt(z, cur) : cpx_gt(z, cur))) { x.a = z.x; x.c = z.y; x.i = idx; }
    }
  } else if (OP == TPG_RANY || OP == TPG_RALL) {
    bool nz;
    if (KIND == K_CPX) nz = cpx_nonzero(dec_cpx(sdt, r));
    else if (KIND == K_FLT) nz = dec_flt(sdt, r) != 0.0;
    else nz = dec_int(sdt, r) != 0;
    if (OP == TPG_RANY) x.v |= nz;
    else x.v &= nz;
  } else {  // norm
    double m;
    if (KIND == K_CPX) {
      double2 z = dec_cpx(sdt, r);
      m = hypot(z.x, z.y);
    } else if (KIND == K_FLT) {
      m = fabs(dec_flt(sdt, r));
    } else {
      const int64_t v = dec_int(sdt, r);
      if (KIND == K_UINT) m = __ull2double_rn((uint64_t)v);
      else m = v < 0 ? __ull2double_rn(0ull - (uint64_t)v) : __ll2double_rn(v);
    }
    const double t = p.p == 2.0 ? __dmul_rn(m, m) : pow(m, p.p);
    dd_add(x.a, x.b, t);
  }
}

// combine x (earlier chunk) with y (later chunk)
template <int OP, int KIND>
__device__ __forceinline__ Acc acc_comb(Acc x, const Acc& y) {
  if (OP == TPG_RSUM || OP == TPG_RNORM) {
    if (KIND == K_INT || KIND == K_UINT) {
      if (OP == TPG_RSUM) x.v = (int64_t)((uint64_t)x.v + (uint64_t)y.v);
      else dd_merge(x.a, x.b, y.a, y.b);
    } else {
      dd_merge(x.a, x.b, y.a, y.b);
      if (KIND == K_CPX && OP == TPG_RSUM) dd_merge(x.c, x.d, y.c, y.d);
    }
  } else if (OP == TPG_RPRODUCT) {
    if (KIND == K_INT || KIND == K_UINT) x.v = (int64_t)((uint64_t)x.v * (uint64_t)y.v);
    else if (KIND == K_FLT) x.a = __dmul_rn(x.a, y.a);
    else {
      const double re = __dsub_rn(__dmul_rn(x.a, y.a), __dmul_rn(x.c, y.c));
      const double im = __dadd_rn(__dmul_rn(x.a, y.c), __dmul_rn(x.c, y.a));
      x.a = re;
      x.c = im;
    }
  } else if (OP == TPG_RMIN || OP == TPG_RMAX) {
    const bool mn = OP == TPG_RMIN;
    if (y.b != 0.0) { x.b = y.b; x.d = y.d; if (KIND == K_CPX) x.v = y.v; }
    if (y.i >= 0) {
      bool take;
      if (x.i < 0) {
        take = true;
      } else if (KIND == K_INT) {
        take = mn ? (y.v < x.v || (y.v == x.v && y.i < x.i)) : (y.v > x.v || (y.v == x.v && y.i < x.i));
      } else if (KIND == K_UINT) {
        const uint64_t a = (uint64_t)x.v, b = (uint64_t)y.v;
        take = mn ? (b < a || (b == a && y.i < x.i)) : (b > a || (b == a && y.i < x.i));
      } else if (KIND == K_FLT) {
        take = mn ? (y.a < x.a || (y.a == x.a && y.i < x.i)) : (y.a > x.a || (y.a == x.a && y.i < x.i));
      } else {
        const double2 a = make_double2(x.a, x.c), b = make_double2(y.a, y.c);
        const bool better = mn ? cpx_lt(b, a) : cpx_gt(b, a);
        const bool worse = mn ? cpx_lt(a, b) : cpx_gt(a, b);
        take = better || (!worse && y.i < x.i);
      }
      if (take) {
        const double sb = x.b, sd = x.d;
        const int64_t sv = x.v;
        x.a = y.a; x.c = y.c; x.i = y.i;
        if (KIND == K_INT || KIND == K_UINT) x.v = y.v;
        x.b = sb; x.d = sd;
        if (KIND == K_CPX) x.v = sv;
      }
    }
  } else if (OP == TPG_RANY) {
    x.v |= y.v;
  } else {  // all
    x.v &= y.v;
  }
  return x;
}

template <int OP, int KIND>
__device__ __forceinline__ void acc_store(const RedParams& p, const Acc& x, int64_t doff,
                                          uint32_t& st) {
  uint32_t* fl = p.track ? &st : nullptr;
  R16 o;
  if (OP == TPG_RANY || OP == TPG_RALL) {
    o = enc_from_int(p.ddt, x.v, false, fl);
  } else if (OP == TPG_RNORM) {
    const double s = __dadd_rn(x.a, x.b);
    const double r = p.p == 2.0 ? sqrt(s) : pow(s, 1.0 / p.p);
    o = enc_from_flt(p.ddt, r, fl);
  } else if (OP == TPG_RSUM) {
    if (KIND == K_INT) o = enc_from_int(p.ddt, x.v, false, fl);
    else if (KIND == K_UINT) o = enc_from_int(p.ddt, x.v, true, fl);
    else if (KIND == K_FLT) o = enc_from_flt(p.ddt, __dadd_rn(x.a, x.b), fl);
    else o = enc_from_cpx(p.ddt, __dadd_rn(x.a, x.b), __dadd_rn(x.c, x.d), fl);
  } else if (OP == TPG_RPRODUCT) {
    if (KIND == K_INT) o = enc_from_int(p.ddt, x.v, false, fl);
    else if (KIND == K_UINT) o = enc_from_int(p.ddt, x.v, true, fl);
    else if (KIND == K_FLT) o = enc_from_flt(p.ddt, x.a, fl);
    else o = enc_from_cpx(p.ddt, x.a, x.c, fl);
  } else {  // min / max
    if (KIND == K_INT) o = enc_from_int(p.ddt, x.v, false, fl);
    else if (KIND == K_UINT) o = enc_from_int(p.ddt, x.v, true, fl);
    else if (KIND == K_FLT)
      o = enc_from_flt(p.ddt, x.b != 0.0 ? x.d : (x.i < 0 ? __longlong_as_double(0x7ff8000000000000ll) : x.a), fl);
    else if (x.b != 0.0) o = enc_from_cpx(p.ddt, x.d, __longlong_as_double(x.v), fl);
    else o = enc_from_cpx(p.ddt, x.a, x.c, fl);
  }
  if (p.dswap) o = swap_raw(p.ddt, o);
  store_raw(p.ddt, p.dbase + doff, o, p.daligned);
}

__device__ __forceinline__ void outer_offsets(const RedParams& p, int64_t o, int64_t& doff,
                                              int64_t& soff) {
  doff = 0;
  soff = 0;
  for (int k = 0; k < p.ndo; ++k) {
    const int64_t e = p.eo[k];
    const int64_t c = o % e;
    o /= e;
    doff += c * p.so_d[k];
    soff += c * p.so_s[k];
  }
}

__device__ __forceinline__ int64_t inner_offset(const RedParams& p, int64_t j) {
  if (p.ndi == 1) return j * p.si[0];
  int64_t off = 0;
  for (int k = 0; k < p.ndi; ++k) {
    const int64_t e = p.ei[k];
    const int64_t c = j % e;
    j /= e;
    off += c * p.si[k];
  }
  return off;
}

template <int OP, int KIND>
__device__ __forceinline__ Acc warp_comb(Acc x) {
  // lanes hold consecutive sub-ranges in lane order; combine in order.
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    Acc y;
    y.a = __shfl_down_sync(0xffffffffu, x.a, s);
    y.b = __shfl_down_sync(0xffffffffu, x.b, s);
    y.c = __shfl_down_sync(0xffffffffu, x.c, s);
    y.d = __shfl_down_sync(0xffffffffu, x.d, s);
    y.i = __shfl_down_sync(0xffffffffu, x.i, s);
    y.v = __shfl_down_sync(0xffffffffu, x.v, s);
    const int lane = threadIdx.x & 31;
    if ((lane & (2 * s - 1)) == 0 && lane + s < 32) x = acc_comb<OP, KIND>(x, y);
  }
  return x;
}

// Source dtype SDT is a template parameter for the hot dtypes (f64, f32) so
// decoding is resolved at compile time; SDT = -1 reads it from the params.
template <int SDT>
__device__ __forceinline__ int sdt_of(const RedParams& p) { return SDT >= 0 ? SDT : p.sdt; }

// row mode: one block per (output, chunk); threads stride the chunk with U
// independent accumulators each (latency hiding, U loads in flight).
template <int OP, int KIND, int SDT>
__global__ void __launch_bounds__(256) k_red_rows(RedParams p) {
  constexpr int U = 8;
  __shared__ Acc sh[8];
  uint32_t st = 0;
  const int sdt = sdt_of<SDT>(p);
  const int64_t nwork = p.O * p.C;
  for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int64_t o = w / p.C, c = w - o * p.C;
    int64_t doff, soff;
    outer_offsets(p, o, doff, soff);
    const int64_t j0 = c * p.chunk;
    const int64_t j1 = min(p.N, j0 + p.chunk);
    Acc x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = acc_init<OP, KIND>();
    if (p.ndi == 1) {
      const int64_t s0 = p.si[0];
      const char* base = p.sbase + soff;
      for (int64_t jb = j0 + threadIdx.x; jb < j1; jb += 256 * U) {
        R16 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t j = jb + u * 256;
          if (j < j1) r[u] = load_raw(sdt, base + j * s0, p.saligned);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t j = jb + u * 256;
          if (j < j1) acc_feed<OP, KIND>(x[u], p, sdt, r[u], j);
        }
      }
    } else {
      for (int64_t jb = j0 + threadIdx.x; jb < j1; jb += 256 * U) {
        R16 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t j = jb + u * 256;
          if (j < j1) r[u] = load_raw(sdt, p.sbase + soff + inner_offset(p, j), p.saligned);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t j = jb + u * 256;
          if (j < j1) acc_feed<OP, KIND>(x[u], p, sdt, r[u], j);
        }
      }
    }
#pragma unroll
    for (int u = 1; u < U; ++u) x[0] = acc_comb<OP, KIND>(x[0], x[u]);
    Acc t = warp_comb<OP, KIND>(x[0]);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh[warp] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
      Acc a = sh[0];
      for (int k = 1; k < 8; ++k) a = acc_comb<OP, KIND>(a, sh[k]);
      if (p.C == 1) acc_store<OP, KIND>(p, a, doff, st);
      else p.ws[o * p.C + c] = a;
    }
    __syncthreads();
  }
  if (st) atomicOr(p.flags, st);
}

// column mode: one thread per (output, chunk); outputs along outer axis 0
// are adjacent in memory so a warp's loads coalesce.  Two accumulators
// alternate to break the dependency chain; U loads are in flight.
template <int OP, int KIND, int SDT>
__global__ void __launch_bounds__(256) k_red_cols(RedParams p, int64_t nob) {
  constexpr int U = 8;
  uint32_t st = 0;
  const int sdt = sdt_of<SDT>(p);
  const int64_t nwork = nob * p.C;
  for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int64_t ob = w % nob, c = w / nob;
    const int64_t o = ob * 256 + threadIdx.x;
    if (o >= p.O) continue;
    int64_t doff, soff;
    outer_offsets(p, o, doff, soff);
    const int64_t j0 = c * p.chunk;
    const int64_t j1 = min(p.N, j0 + p.chunk);
    Acc x[2];
    x[0] = x[1] = acc_init<OP, KIND>();
    const bool flat = p.ndi == 1;
    const int64_t s0 = p.si[0];
    for (int64_t jb = j0; jb < j1; jb += U) {
      R16 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (jb + u < j1)
          r[u] = load_raw(sdt, p.sbase + soff + (flat ? (jb + u) * s0 : inner_offset(p, jb + u)),
                          p.saligned);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (jb + u < j1) acc_feed<OP, KIND>(x[u & 1], p, sdt, r[u], jb + u);
    }
    x[0] = acc_comb<OP, KIND>(x[0], x[1]);
    if (p.C == 1) acc_store<OP, KIND>(p, x[0], doff, st);
    else p.ws[o * p.C + c] = x[0];
  }
  if (st) atomicOr(p.flags, st);
}

// finalize for few partials per output (C <= 32): one warp per output, lane
// c holds partial c, combined by the fixed warp tree.
template <int OP, int KIND>
__global__ void __launch_bounds__(256) k_red_final_warp(RedParams p) {
  uint32_t st = 0;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * 8;
  for (int64_t o = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); o < p.O; o += nw) {
    Acc x = lane < p.C ? p.ws[o * p.C + lane] : acc_init<OP, KIND>();
    x = warp_comb<OP, KIND>(x);
    if (lane == 0) {
      int64_t doff, soff;
      outer_offsets(p, o, doff, soff);
      acc_store<OP, KIND>(p, x, doff, st);
    }
  }
  if (st) atomicOr(p.flags, st);
}

// finalize: one block per output; all partials are loaded up front
// (coalesced, independent), then combined in a fixed tree order.
template <int OP, int KIND>
__global__ void __launch_bounds__(256) k_red_final(RedParams p) {
  __shared__ Acc sh[8];
  uint32_t st = 0;
  for (int64_t o = blockIdx.x; o < p.O; o += gridDim.x) {
    Acc x = acc_init<OP, KIND>();
    constexpr int PF = 8;
    for (int64_t c0 = threadIdx.x; c0 < p.C; c0 += 256 * PF) {
      Acc y[PF];
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        const int64_t c = c0 + u * 256;
        y[u] = c < p.C ? p.ws[o * p.C + c] : acc_init<OP, KIND>();
      }
#pragma unroll
      for (int u = 0; u < PF; ++u) x = acc_comb<OP, KIND>(x, y[u]);
    }
    x = warp_comb<OP, KIND>(x);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh[warp] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      Acc a = sh[0];
      for (int k = 1; k < 8; ++k) a = acc_comb<OP, KIND>(a, sh[k]);
      int64_t doff, soff;
      outer_offsets(p, o, doff, soff);
      acc_store<OP, KIND>(p, a, doff, st);
    }
    __syncthreads();
  }
  if (st) atomicOr(p.flags, st);
}

// sequential: one thread per output walks the inner plan in order, exactly
// like reduce_strided; used where the combine order is observable beyond
// rounding (complex products: inf/NaN propagation depends on the order).
template <int OP, int KIND>
__global__ void __launch_bounds__(128) k_red_seq(RedParams p) {
  uint32_t st = 0;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < p.O;
       o += (int64_t)gridDim.x * blockDim.x) {
    int64_t doff, soff;
    outer_offsets(p, o, doff, soff);
    Acc x = acc_init<OP, KIND>();
    for (int64_t j = 0; j < p.N; ++j)
      acc_feed<OP, KIND>(x, p, p.sdt, load_raw(p.sdt, p.sbase + soff + inner_offset(p, j), p.saligned), j);
    acc_store<OP, KIND>(p, x, doff, st);
  }
  if (st) atomicOr(p.flags, st);
}

// ---------------------------------------------------------------------------
// Float fast path (SURVEY cfg3: f64/f32 sum, norm, min, max).  Same
// semantics as the Acc machinery (it produces an Acc at the end), but the
// per-element state is just the double-double pair or (best, index), with
// NA independent accumulators per thread and U loads in flight.
template <int OP, bool GENP = true>  // GENP = false: norm order 2 only
struct FAcc {
  double hi, lo;  // sum / norm: double-double; min/max: hi = best value
  int64_t idx;    // min/max: index of best (-1 none)
  double nanv;    // min/max: first element (when NaN)
  bool fnan;
  __device__ __forceinline__ void init() {
    hi = lo = 0.0;
    idx = -1;
    nanv = 0.0;
    fnan = false;
  }
  __device__ __forceinline__ void feed(double v, int64_t j, double pp) {
    if (OP == TPG_RSUM) {
      dd_add(hi, lo, v);
    } else if (OP == TPG_RNORM) {
      const double m = fabs(v);
      dd_add(hi, lo, (!GENP || pp == 2.0) ? __dmul_rn(m, m) : pow(m, pp));
    } else {
      if (isnan(v)) {
        if (j == 0 && pp >= 0.0) { fnan = true; nanv = v; }
      } else if (idx < 0 || (OP == TPG_RMIN ? v < hi : v > hi)) {
        hi = v;
        idx = j;
      }
    }
  }
  __device__ __forceinline__ Acc to_acc() const {
    Acc x = acc_init<OP, K_FLT>();
    if (OP == TPG_RSUM || OP == TPG_RNORM) {
      x.a = hi;
      x.b = lo;
    } else {
      x.a = hi;
      x.i = idx;
      if (fnan) { x.b = 1.0; x.d = nanv; }
    }
    return x;
  }
};

// Streaming loads as volatile asm so a batch of them is issued back to back
// (ptxas otherwise pairs each load with its consumer, leaving one in flight).
template <typename T>
__device__ __forceinline__ double ld_real(const char* ptr);
template <>
__device__ __forceinline__ double ld_real<double>(const char* ptr) {
  double v;
  asm volatile("ld.global.cs.f64 %0, [%1];" : "=d"(v) : "l"(ptr));
  return v;
}
template <>
__device__ __forceinline__ double ld_real<float>(const char* ptr) {
  float v;
  asm volatile("ld.global.cs.f32 %0, [%1];" : "=f"(v) : "l"(ptr));
  return (double)v;
}

template <int OP, typename T>
__global__ void __launch_bounds__(256, 4) k_red_rows_flt(RedParams p) {
  constexpr int U = 4, NA = 4;  // 2 x U loads in flight (double-buffered)
  __shared__ Acc sh[8];
  uint32_t st = 0;
  const int64_t nwork = p.O * p.C;
  for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int64_t o = w / p.C, c = w - o * p.C;
    int64_t doff, soff;
    outer_offsets(p, o, doff, soff);
    const int64_t j0 = c * p.chunk;
    const int64_t j1 = min(p.N, j0 + p.chunk);
    FAcc<OP> x[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) x[a].init();
    const int64_t s0 = p.si[0];
    const char* base = p.sbase + soff;
    // full iterations: U unconditional loads issued back to back (all in
    // flight), then consumed; a predicated form lets the compiler pair each
    // load with its use and serialise them
    int64_t jb = j0 + threadIdx.x;
    // Full batches of U loads per thread, software-pipelined: batch k+1 is
    // loaded while batch k is folded in, so U loads stay in flight whatever
    // order ptxas schedules the arithmetic in.
    const int64_t avail = j1 - jb;
    const int64_t nfull = avail > 256 * (U - 1) ? (avail - 256 * (U - 1) - 1) / (256 * U) + 1 : 0;
    const char* ptr = base + jb * s0;
    const int64_t step = 256 * s0;
    if (nfull > 0) {
      double v[U], nv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld_real<T>(ptr + u * step);
      for (int64_t k = 0; k < nfull; ++k) {
        if (k + 1 < nfull) {
#pragma unroll
          for (int u = 0; u < U; ++u) nv[u] = ld_real<T>(ptr + (U + u) * step);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) x[u % NA].feed(v[u], jb + u * 256, p.p);
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = nv[u];
        jb += 256 * U;
        ptr += U * step;
      }
    }
    for (; jb < j1; jb += 256, ptr += step) x[0].feed(ld_real<T>(ptr), jb, p.p);
    Acc t = x[0].to_acc();
#pragma unroll
    for (int a = 1; a < NA; ++a) t = acc_comb<OP, K_FLT>(t, x[a].to_acc());
    t = warp_comb<OP, K_FLT>(t);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh[warp] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
      Acc a = sh[0];
      for (int k = 1; k < 8; ++k) a = acc_comb<OP, K_FLT>(a, sh[k]);
      if (p.C == 1) acc_store<OP, K_FLT>(p, a, doff, st);
      else p.ws[o * p.C + c] = a;
    }
    __syncthreads();
  }
  if (st) atomicOr(p.flags, st);
}

template <int OP, typename T>
__global__ void __launch_bounds__(256, 4) k_red_cols_flt(RedParams p, int64_t nob) {
  constexpr int U = 4, NA = 2;  // 2 x U loads in flight (double-buffered)
  uint32_t st = 0;
  const int64_t nwork = nob * p.C;
  for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int64_t ob = w % nob, c = w / nob;
    const int64_t o = ob * 256 + threadIdx.x;
    if (o >= p.O) continue;
    int64_t doff, soff;
    outer_offsets(p, o, doff, soff);
    const int64_t j0 = c * p.chunk;
    const int64_t j1 = min(p.N, j0 + p.chunk);
    FAcc<OP> x[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) x[a].init();
    const int64_t s0 = p.si[0];
    const char* base = p.sbase + soff;
    int64_t jb = j0;
    const char* ptr = base + j0 * s0;
    const int64_t nfull = (j1 - j0) / U;
    if (nfull > 0) {
      double v[U], nv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld_real<T>(ptr + u * s0);
      for (int64_t k = 0; k < nfull; ++k) {
        if (k + 1 < nfull) {
#pragma unroll
          for (int u = 0; u < U; ++u) nv[u] = ld_real<T>(ptr + (U + u) * s0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) x[u % NA].feed(v[u], jb + u, p.p);
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = nv[u];
        jb += U;
        ptr += U * s0;
      }
    }
    for (; jb < j1; ++jb, ptr += s0) x[0].feed(ld_real<T>(ptr), jb, p.p);
    Acc t = acc_comb<OP, K_FLT>(x[0].to_acc(), x[1].to_acc());
    if (p.C == 1) acc_store<OP, K_FLT>(p, t, doff, st);
    else p.ws[o * p.C + c] = t;
  }
  if (st) atomicOr(p.flags, st);
}

// ---------------------------------------------------------------------------
// Vectorised single-pass float reductions (SURVEY cfg3: f64 / f32 sum, norm,
// min, max).  16-byte loads (2 x f64 / 4 x f32) with a software pipeline
// that keeps 2 x U vectors in flight per thread, and no separate finalize
// launch: the worker that completes the last chunk of an output (arrival
// counter + threadfence) combines that output's partials in chunk order,
// so the result does not depend on which worker arrives last.  Counters come
// from the stream (stream_counters) and are left zero again.
//
// Partials are 16 bytes (Part): sum / norm keep the double-double pair;
// min / max keep (value, index) with index -1 = no element and -2 = "the
// first element of the range is NaN" (value = that NaN), which makes the
// result NaN whatever the other chunks hold (ops.py:527-544).
template <typename T>
struct Vec16;
template <>
struct Vec16<double> {
  double x[2];
  static constexpr int n = 2;
};
template <>
struct Vec16<float> {
  float x[4];
  static constexpr int n = 4;
};

template <typename T>
__device__ __forceinline__ Vec16<T> ld_vec(const char* ptr);
template <>
__device__ __forceinline__ Vec16<double> ld_vec<double>(const char* ptr) {
  Vec16<double> v;
  asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(v.x[0]), "=d"(v.x[1]) : "l"(ptr));
  return v;
}
template <>
__device__ __forceinline__ Vec16<float> ld_vec<float>(const char* ptr) {
  Vec16<float> v;
  asm volatile("ld.global.cs.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x[0]), "=f"(v.x[1]), "=f"(v.x[2]), "=f"(v.x[3])
               : "l"(ptr));
  return v;
}

// Per-thread accumulator of the vector kernels.  min/max are branch-free
// and index elements relative to the chunk start (32-bit); the reference's
// "first element NaN" rule is applied separately by the one thread that
// owns element 0 (first_nan), so the hot loop never tests for it.
// IDX = false (an accumulator fed strictly in element order, e.g. the
// column kernel): min/max is one fmin/fmax per element with no index;
// equal extremes are bit-identical except +-0, so when the extreme is zero
// the caller rescans its range for the first zero (its sign is the
// reference's answer); "no element yet" is hi = NaN.
template <int OP, bool IDX = true>
struct VAcc {
  double hi, lo;
  int idx;  // min/max: chunk-relative index of the best element, -1 = none
  bool fnan;
  double nanv;
  __device__ __forceinline__ void init() {
    hi = (IDX || OP == TPG_RSUM || OP == TPG_RNORM) ? 0.0 : __longlong_as_double(0x7ff8000000000000ll);
    lo = 0.0;
    idx = -1;
    fnan = false;
    nanv = 0.0;
  }
  __device__ __forceinline__ void feed(double v, int jr) {
    if (OP == TPG_RSUM) {
      dd_add(hi, lo, v);
    } else if (OP == TPG_RNORM) {
      const double m = fabs(v);
      dd_add(hi, lo, __dmul_rn(m, m));
    } else if (IDX) {
      const bool better = OP == TPG_RMIN ? v < hi : v > hi;  // false for NaN
      const bool take = (v == v) && (idx < 0 || better);
      hi = take ? v : hi;
      idx = take ? jr : idx;
    } else {
      // one DMNMX: NaN operands are ignored (hi NaN = empty), so this is the
      // extreme over the non-NaN elements; the only case where "first of
      // equal elements" is observable is a +-0 extreme, which the caller
      // resolves by rescanning (zero_first)
      hi = OP == TPG_RMIN ? fmin(hi, v) : fmax(hi, v);
    }
  }
  __device__ __forceinline__ void first_nan(double v) {
    if ((OP == TPG_RMIN || OP == TPG_RMAX) && v != v) {
      fnan = true;
      nanv = v;
    }
  }
};

struct __align__(16) Part {
  double hi, lo;
};

template <int OP, bool IDX>
__device__ __forceinline__ Part to_part(const VAcc<OP, IDX>& a, int64_t jbase) {
  Part r;
  if (OP == TPG_RSUM || OP == TPG_RNORM) {
    r.hi = a.hi;
    r.lo = a.lo;
  } else if (a.fnan) {
    r.hi = a.nanv;
    r.lo = __longlong_as_double(-2ll);
  } else if (IDX) {
    r.hi = a.hi;
    r.lo = __longlong_as_double(a.idx < 0 ? -1ll : jbase + a.idx);
  } else {
    // in-order accumulator: any index inside the chunk orders it correctly
    // against the other chunks' partials
    r.hi = a.hi;
    r.lo = __longlong_as_double(a.hi == a.hi ? jbase : -1ll);
  }
  return r;
}
__device__ __forceinline__ Part part_ident() {
  Part r;
  r.hi = 0.0;
  r.lo = 0.0;  // for min/max the caller uses index -1 (see part_none)
  return r;
}
template <int OP>
__device__ __forceinline__ Part part_none() {
  Part r;
  r.hi = 0.0;
  r.lo = (OP == TPG_RSUM || OP == TPG_RNORM) ? 0.0 : __longlong_as_double(-1ll);
  return r;
}
// x covers earlier elements than y
template <int OP>
__device__ __forceinline__ Part part_comb(Part x, const Part& y) {
  if (OP == TPG_RSUM || OP == TPG_RNORM) {
    dd_merge(x.hi, x.lo, y.hi, y.lo);
    return x;
  }
  const long long ix = __double_as_longlong(x.lo), iy = __double_as_longlong(y.lo);
  if (ix == -2) return x;
  if (iy == -2) return y;
  if (iy < 0) return x;
  if (ix < 0) return y;
  const bool take = OP == TPG_RMIN ? (y.hi < x.hi || (y.hi == x.hi && iy < ix))
                                   : (y.hi > x.hi || (y.hi == x.hi && iy < ix));
  return take ? y : x;
}
template <int OP>
__device__ __forceinline__ Acc part_acc(const Part& x) {
  Acc a = acc_init<OP, K_FLT>();
  if (OP == TPG_RSUM || OP == TPG_RNORM) {
    a.a = x.hi;
    a.b = x.lo;
  } else {
    const long long ix = __double_as_longlong(x.lo);
    if (ix == -2) {
      a.b = 1.0;
      a.d = x.hi;
    } else {
      a.a = x.hi;
      a.i = ix;
    }
  }
  return a;
}
__device__ __forceinline__ Part ld_part(const Part* p) {
  const double2 v = __ldcg((const double2*)p);
  Part r;
  r.hi = v.x;
  r.lo = v.y;
  return r;
}
__device__ __forceinline__ void st_part(Part* p, const Part& v) {
  __stcg((double2*)p, make_double2(v.hi, v.lo));
}
// lane-order combine (lanes hold consecutive ranges); result in lane 0
template <int OP>
__device__ __forceinline__ Part warp_part(Part x) {
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    Part y;
    y.hi = __shfl_down_sync(0xffffffffu, x.hi, s);
    y.lo = __shfl_down_sync(0xffffffffu, x.lo, s);
    const int lane = threadIdx.x & 31;
    if ((lane & (2 * s - 1)) == 0 && lane + s < 32) x = part_comb<OP>(x, y);
  }
  return x;
}
// thread-order combine over the block; result in thread 0
template <int OP, int NT>
__device__ __forceinline__ Part block_part(Part t, Part* sh) {
  t = warp_part<OP>(t);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[warp] = t;
  __syncthreads();
  Part a = sh[0];
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 1; k < NT / 32; ++k) a = part_comb<OP>(a, sh[k]);
  return a;
}

// Stream one unit-stride range [j0, j1) of T (base = element 0 of the
// plan's inner range) through NL lanes (lane index li): scalar head up to
// 16-byte alignment, pipelined 16-byte body, scalar tail.  Folds into x[NA]
// (a lane's feeds reach each accumulator in increasing element order).
template <int OP, typename T, int NL, int NA, int U>
__device__ __forceinline__ void stream_range(VAcc<OP> (&x)[NA], const char* base, int64_t j0,
                                             int64_t j1, int li, double pp) {
  constexpr int VE = Vec16<T>::n;
  const uintptr_t a0 = (uintptr_t)(base + j0 * (int64_t)sizeof(T));
  int64_t ja = j0 + (int64_t)(((16 - (a0 & 15)) & 15) / sizeof(T));
  if (ja > j1) ja = j1;
  if (j0 == 0 && li == 0 && pp >= 0.0) x[0].first_nan(ld_real<T>(base));
  if (j0 + li < ja) x[0].feed(ld_real<T>(base + (j0 + li) * (int64_t)sizeof(T)), li);
  const int64_t nv = (j1 - ja) / VE;
  const char* vb = base + ja * (int64_t)sizeof(T);
  const int64_t nfull = nv / (NL * U);
  int64_t vi = li;
  // three rotating batches: two batches of U vectors in flight while one
  // is folded in (no register copies waiting on loads)
  Vec16<T> bA[U], bB[U], bC[U];
  auto ld = [&](Vec16<T>(&b)[U], int64_t k) {
#pragma unroll
    for (int u = 0; u < U; ++u) b[u] = ld_vec<T>(vb + (li + (k * U + u) * NL) * 16);
  };
  auto fold = [&](const Vec16<T>(&b)[U], int64_t k) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = ja + (li + (k * U + u) * NL) * VE;
#pragma unroll
      for (int e = 0; e < VE; ++e) x[u % NA].feed((double)b[u].x[e], (int)(j - j0) + e);
    }
  };
  if (nfull > 0) ld(bA, 0);
  if (nfull > 1) ld(bB, 1);
  int64_t k = 0;
  for (; k + 3 <= nfull; k += 3) {
    if (k + 2 < nfull) ld(bC, k + 2);
    fold(bA, k);
    if (k + 3 < nfull) ld(bA, k + 3);
    fold(bB, k + 1);
    if (k + 4 < nfull) ld(bB, k + 4);
    fold(bC, k + 2);
  }
  if (k < nfull) fold(bA, k);
  if (k + 1 < nfull) fold(bB, k + 1);
  vi = li + nfull * U * NL;
  for (; vi < nv; vi += NL) {
    const Vec16<T> v = ld_vec<T>(vb + vi * 16);
    const int64_t j = ja + vi * VE;
#pragma unroll
    for (int e = 0; e < VE; ++e) x[0].feed((double)v.x[e], (int)(j - j0) + e);
  }
  const int64_t jt = ja + nv * VE + li;
  if (jt < j1) x[0].feed(ld_real<T>(base + jt * (int64_t)sizeof(T)), (int)(jt - j0));
}

template <int OP, int NA>
__device__ __forceinline__ Part fold_accs(VAcc<OP> (&x)[NA], int64_t jbase) {
  Part t = to_part(x[0], jbase);
#pragma unroll
  for (int a = 1; a < NA; ++a) t = part_comb<OP>(t, to_part(x[a], jbase));
  return t;
}

// Row mode, warp granularity: one warp per (output, chunk) work item (many
// outputs, e.g. cfg3 axis 0).  Warps never synchronise with each other, so
// one warp's drain overlaps the others' streaming.
template <int OP, typename T>
__global__ void __launch_bounds__(256, 2) k_red_rows_wv(RedParams p, Part* ws, uint32_t* cnt) {
  constexpr int U = 4, NA = 2;
  uint32_t st = 0;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nwork = p.O * p.C;
  for (int64_t w = gw; w < nwork; w += nw) {
    const int64_t o = w / p.C, c = w - o * p.C;
    int64_t doff, soff;
    outer_offsets(p, o, doff, soff);
    const int64_t j0 = c * p.chunk;
    const int64_t j1 = min(p.N, j0 + p.chunk);
    VAcc<OP> x[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) x[a].init();
    stream_range<OP, T, 32, NA, U>(x, p.sbase + soff, j0, j1, lane, p.p);
    const Part r = warp_part<OP>(fold_accs<OP, NA>(x, j0));
    if (p.C == 1) {
      if (lane == 0) acc_store<OP, K_FLT>(p, part_acc<OP>(r), doff, st);
      continue;
    }
    uint32_t last = 0;
    if (lane == 0) {
      st_part(&ws[o * p.C + c], r);
      __threadfence();
      last = atomicAdd(&cnt[o], 1u) == (uint32_t)(p.C - 1);
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      __threadfence();
      // lane l combines chunks [l*per, (l+1)*per), then lane order
      const int64_t per = (p.C + 31) / 32;
      Part y = part_none<OP>();
      for (int64_t cc = lane * per; cc < min(p.C, (lane + 1) * per); ++cc)
        y = part_comb<OP>(y, ld_part(&ws[o * p.C + cc]));
      y = warp_part<OP>(y);
      if (lane == 0) {
        acc_store<OP, K_FLT>(p, part_acc<OP>(y), doff, st);
        cnt[o] = 0;
      }
    }
  }
  if (st) atomicOr(p.flags, st);
}

// The cross-rank finish of a full sum inside the reduction kernel (called by
// the one thread that holds the rank's final double-double partial): store
// (hi, lo) into every rank's mailbox slot [parity][my rank] over NVLink,
// publish the epoch (system-scope release), wait for every rank's slot in
// this rank's mailbox (acquire, bounded), merge them IN RANK ORDER in
// double-double.  Bit 31 of the status word marks a peer that never came.
template <int OP>
__device__ __forceinline__ Part p2p_exchange(const RedParams& p, Part mine) {
  const unsigned long long ep = p.p2p_epoch;
  const int par = (int)(ep & 1);
  if (OP == TPG_RMIN || OP == TPG_RMAX) {
    // local plan indices -> global ones, so ties keep the earliest element
    const long long ix = __double_as_longlong(mine.lo);
    if (ix >= 0) mine.lo = __longlong_as_double(ix + p.p2p_index_base);
  }
  for (int q = 0; q < p.p2p_world; ++q) {
    P2pSlot* dst = p.p2p[q] + par * P2P_MAX_RANKS + p.p2p_rank;
    ((volatile uint64_t*)dst->payload)[0] = (uint64_t)__double_as_longlong(mine.hi);
    ((volatile uint64_t*)dst->payload)[1] = (uint64_t)__double_as_longlong(mine.lo);
  }
  __threadfence_system();
  for (int q = 0; q < p.p2p_world; ++q) {
    P2pSlot* dst = p.p2p[q] + par * P2P_MAX_RANKS + p.p2p_rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&dst->epoch), "l"(ep) : "memory");
  }
  const P2pSlot* box = p.p2p[p.p2p_rank] + par * P2P_MAX_RANKS;
  Part acc;
  for (int q = 0; q < p.p2p_world; ++q) {
    const long long t0 = clock64();
    unsigned long long e;
    do {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(e) : "l"(&box[q].epoch) : "memory");
      if (e >= ep) break;
      if (clock64() - t0 > (1ll << 33)) {
        atomicOr(p.flags, 0x80000000u);
        break;
      }
      __nanosleep(64);
    } while (true);
    Part y;
    y.hi = __longlong_as_double((long long)((const volatile uint64_t*)box[q].payload)[0]);
    y.lo = __longlong_as_double((long long)((const volatile uint64_t*)box[q].payload)[1]);
    // rank order: acc covers the earlier elements
    acc = q == 0 ? y : part_comb<OP>(acc, y);
  }
  return acc;
}

// Row mode, block granularity: one block per (output, chunk) (few outputs,
// e.g. full reductions).
template <int OP, typename T>
__global__ void __launch_bounds__(256, 2) k_red_rows_v(RedParams p, Part* ws, uint32_t* cnt) {
  constexpr int U = 4, NA = 2, NT = 256;
  __shared__ Part sh[NT / 32];
  __shared__ int is_last;
  uint32_t st = 0;
  const int tid = threadIdx.x;
  const int64_t nwork = p.O * p.C;
  for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int64_t o = w / p.C, c = w - o * p.C;
    int64_t doff, soff;
    outer_offsets(p, o, doff, soff);
    const int64_t j0 = c * p.chunk;
    const int64_t j1 = min(p.N, j0 + p.chunk);
    VAcc<OP> x[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) x[a].init();
    stream_range<OP, T, NT, NA, U>(x, p.sbase + soff, j0, j1, tid, p.p);
    const Part r = block_part<OP, NT>(fold_accs<OP, NA>(x, j0), sh);
    if (p.C == 1) {
      if (tid == 0) {
        Part f = r;
        if (p.p2p) f = p2p_exchange<OP>(p, f);
        acc_store<OP, K_FLT>(p, part_acc<OP>(f), doff, st);
      }
      continue;
    }
    if (tid == 0) {
      st_part(&ws[o * p.C + c], r);
      __threadfence();
      is_last = atomicAdd(&cnt[o], 1u) == (uint32_t)(p.C - 1);
    }
    __syncthreads();
    if (is_last) {
      __threadfence();
      const int64_t per = (p.C + NT - 1) / NT;
      Part y = part_none<OP>();
      for (int64_t cc = tid * per; cc < min(p.C, (tid + 1) * per); ++cc)
        y = part_comb<OP>(y, ld_part(&ws[o * p.C + cc]));
      Part z = block_part<OP, NT>(y, sh);
      if (tid == 0) {
        if (p.p2p) z = p2p_exchange<OP>(p, z);
        acc_store<OP, K_FLT>(p, part_acc<OP>(z), doff, st);
        cnt[o] = 0;
      }
    }
  }
  if (st) atomicOr(p.flags, st);
}

// Column mode: outputs adjacent in the source (outer axis 0 unit-stride),
// reduced axis strided (cfg3 axis 1).  Each thread owns VE adjacent outputs
// and reads one 16-byte vector per row; a block covers NT*VE outputs x one
// row chunk.  Partials are chunk-major (ws[c * O + o]) so the finalizing
// block reads them coalesced, 8 chunks in flight per thread.
template <int OP, typename T, int NT>
__global__ void __launch_bounds__(NT, 512 / NT) k_red_cols_v(RedParams p, int64_t nob, Part* ws,
                                                             uint32_t* cnt) {
  constexpr int VE = Vec16<T>::n, U = 4;
  __shared__ int is_last;
  uint32_t st = 0;
  const int tid = threadIdx.x;
  const int64_t nwork = nob * p.C;
  for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int64_t ob = w % nob, c = w / nob;
    const int64_t o = (ob * NT + tid) * VE;
    const bool act = o < p.O;
    int64_t doff = 0, soff = 0;
    if (act) outer_offsets(p, o, doff, soff);
    const int64_t j0 = c * p.chunk;
    const int64_t j1 = min(p.N, j0 + p.chunk);
    if (act) {
      // one in-order accumulator per output: min/max need no element index
      constexpr int NACC = 1;
      VAcc<OP, false> x[VE][NACC];
#pragma unroll
      for (int e = 0; e < VE; ++e)
#pragma unroll
        for (int a = 0; a < NACC; ++a) x[e][a].init();
      const int64_t s0 = p.si[0];
      const char* ptr = p.sbase + soff + j0 * s0;
      if (j0 == 0 && p.p >= 0.0) {
        const Vec16<T> f = ld_vec<T>(ptr);
#pragma unroll
        for (int e = 0; e < VE; ++e) x[e][0].first_nan((double)f.x[e]);
      }
      int64_t jb = j0;
      // three rotating batches of U row vectors: two batches (2*U*16 B)
      // stay in flight while one is folded in, and no register copies
      // wait on loads
      const int64_t nfull = (j1 - j0) / U;
      Vec16<T> bA[U], bB[U], bC[U];
      auto ld = [&](Vec16<T>(&b)[U], int64_t k) {
#pragma unroll
        for (int u = 0; u < U; ++u) b[u] = ld_vec<T>(ptr + (k * U + u) * s0);
      };
      // min/max fold into plain doubles (fmin/fmax: NaN operands ignored,
      // NaN = empty), which keeps the compiler from copying batch registers
      // whose loads are still in flight
      constexpr bool MM = OP == TPG_RMIN || OP == TPG_RMAX;
      double mm[VE];
#pragma unroll
      for (int e = 0; e < VE; ++e) mm[e] = x[e][0].hi;
      auto fold = [&](const Vec16<T>(&b)[U], int64_t k) {
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int e = 0; e < VE; ++e) {
            if constexpr (MM)
              mm[e] = OP == TPG_RMIN ? fmin(mm[e], (double)b[u].x[e]) : fmax(mm[e], (double)b[u].x[e]);
            else
              x[e][0].feed((double)b[u].x[e], (int)(k * U + u));
          }
      };
      if (nfull > 0) ld(bA, 0);
      if (nfull > 1) ld(bB, 1);
      int64_t k = 0;
      for (; k + 3 <= nfull; k += 3) {
        if (k + 2 < nfull) ld(bC, k + 2);
        fold(bA, k);
        if (k + 3 < nfull) ld(bA, k + 3);
        fold(bB, k + 1);
        if (k + 4 < nfull) ld(bB, k + 4);
        fold(bC, k + 2);
      }
      if (k < nfull) fold(bA, k);
      if (k + 1 < nfull) fold(bB, k + 1);
      if constexpr (MM) {
#pragma unroll
        for (int e = 0; e < VE; ++e) x[e][0].hi = mm[e];
      }
      jb = j0 + nfull * U;
      ptr += nfull * U * s0;
      for (; jb < j1; ++jb, ptr += s0) {
        const Vec16<T> v = ld_vec<T>(ptr);
#pragma unroll
        for (int e = 0; e < VE; ++e) x[e][0].feed((double)v.x[e], (int)(jb - j0));
      }
      if (OP == TPG_RMIN || OP == TPG_RMAX) {
        // a +-0 extreme: the sign is that of the first zero in the range
#pragma unroll
        for (int e = 0; e < VE; ++e) {
          if (x[e][0].hi != 0.0) continue;
          const char* q = p.sbase + soff + j0 * s0 + e * (int64_t)sizeof(T);
          for (int64_t j = j0; j < j1; ++j, q += s0) {
            const double v = (double)*(const T*)q;
            if (v == 0.0) {
              x[e][0].hi = v;
              break;
            }
          }
        }
      }
#pragma unroll
      for (int e = 0; e < VE; ++e) {
        const Part t = to_part(x[e][0], j0);
        if (p.C == 1) acc_store<OP, K_FLT>(p, part_acc<OP>(t), doff + e * p.so_d[0], st);
        else st_part(&ws[c * p.O + o + e], t);
      }
    }
    if (p.C == 1) continue;
    __threadfence();
    __syncthreads();
    if (tid == 0) is_last = atomicAdd(&cnt[ob], 1u) == (uint32_t)(p.C - 1);
    __syncthreads();
    if (is_last) {
      __threadfence();
      if (act) {
        // all VE outputs at once, FB chunks per batch: 8 partial loads in
        // flight per thread (chunk order per output is kept)
        constexpr int FB = 8 / VE;
        Part y[VE];
#pragma unroll
        for (int e = 0; e < VE; ++e) y[e] = part_none<OP>();
        for (int64_t c0 = 0; c0 < p.C; c0 += FB) {
          Part q[FB][VE];
#pragma unroll
          for (int u = 0; u < FB; ++u)
#pragma unroll
            for (int e = 0; e < VE; ++e)
              q[u][e] = c0 + u < p.C ? ld_part(&ws[(c0 + u) * p.O + o + e]) : part_none<OP>();
#pragma unroll
          for (int u = 0; u < FB; ++u)
#pragma unroll
            for (int e = 0; e < VE; ++e) y[e] = part_comb<OP>(y[e], q[u][e]);
        }
#pragma unroll
        for (int e = 0; e < VE; ++e) acc_store<OP, K_FLT>(p, part_acc<OP>(y[e]), doff + e * p.so_d[0], st);
      }
      if (tid == 0) cnt[ob] = 0;
    }
    __syncthreads();
  }
  if (st) atomicOr(p.flags, st);
}

// eligibility of the vector kernels (else the scalar float kernels run)
template <typename T>
bool rows_vec_ok(const RedParams& p) {
  return p.ndi == 1 && p.si[0] == (int64_t)sizeof(T);
}
template <typename T>
bool cols_vec_ok(const RedParams& p) {
  constexpr int VE = Vec16<T>::n;
  if (p.ndi != 1 || p.ndo < 1 || p.so_s[0] != (int64_t)sizeof(T) || p.eo[0] % VE) return false;
  if ((uintptr_t)p.sbase % 16 || p.si[0] % 16) return false;
  for (int k = 1; k < p.ndo; ++k)
    if (p.eo[k] > 1 && p.so_s[k] % 16) return false;
  return true;
}

// Work split + launch of the vector kernels; done = false when the layout
// is not eligible (the caller then runs the scalar kernels).
template <int OP, typename T>
int launch_vec(RedParams& p, Stream* st, bool col, bool& done) {
  done = false;
  if (OP == TPG_RNORM && p.p != 2.0) return TPG_OK;
  const int64_t sms = sm_count(st->device);
  Part* ws = nullptr;
  uint32_t* cnt = nullptr;
  auto scratch = [&](int64_t nparts, int64_t ncnt) -> int {
    if (p.C <= 1) return TPG_OK;
    cnt = stream_counters(st, ncnt);
    if (!cnt) return arg_fail("reduce: counter allocation failed");
    TPG_CUDA_CHECK(cudaMallocAsync((void**)&ws, sizeof(Part) * nparts, st->s));
    return TPG_OK;
  };
  if (col) {
    if (!cols_vec_ok<T>(p)) return TPG_OK;
    constexpr int VE = Vec16<T>::n;
    constexpr int NT = 64;  // 64 x 16 B = 1 KiB of a row per block (measured best)
    const int64_t nob = (p.O + NT * VE - 1) / (NT * VE);
    // one wave of resident blocks: the last-arriver finalize of each output
    // block reads C partials per output after the streaming ends, so C is
    // kept as small as filling the machine allows, rounded down to whole
    // finalize batches of 8 / VE chunks (cfg3 axis 1: C = 16; C = 64 cost
    // 20 us of finalize tail on max, 10 us on sum; C = 18 3 us more than 16)
    const int64_t slots = sms * (512 / NT);
    int64_t C = slots / nob;
    if (C > 8 / VE) C -= C % (8 / VE);
    if (C > p.N / 32) C = p.N / 32;
    if (C > 64) C = 64;
    if (C < 1) C = 1;
    p.chunk = (p.N + C - 1) / C;
    p.C = (p.N + p.chunk - 1) / p.chunk;
    if (int rc = scratch(p.O * p.C, nob)) return rc;
    const int64_t work = nob * p.C;
    k_red_cols_v<OP, T, NT><<<(int)std::min<int64_t>(work, 1 << 30), NT, 0, st->s>>>(p, nob, ws, cnt);
  } else {
    if (!rows_vec_ok<T>(p)) return TPG_OK;
    const int64_t wslots = sms * 2 * 8;  // resident warps
    if (p.O >= wslots / 2) {
      // warp items: enough outputs to fill the machine; split each output
      // only as far as needed for about two warp items per slot
      int64_t C = (2 * wslots + p.O - 1) / p.O;
      const int64_t minchunk = 2048;
      if (C > (p.N + minchunk - 1) / minchunk) C = (p.N + minchunk - 1) / minchunk;
      if (C > 32) C = 32;
      if (C < 1) C = 1;
      p.chunk = (p.N + C - 1) / C;
      p.chunk = (p.chunk + 7) & ~(int64_t)7;
      p.C = (p.N + p.chunk - 1) / p.chunk;
      if (int rc = scratch(p.O * p.C, p.O)) return rc;
      const int64_t warps = std::min<int64_t>(p.O * p.C, wslots);
      k_red_rows_wv<OP, T><<<(int)((warps + 7) / 8), 256, 0, st->s>>>(p, ws, cnt);
    } else {
      const int64_t target = sms * 2 * 2;  // two waves of resident blocks
      int64_t C = (target + p.O - 1) / p.O;
      const int64_t minchunk = 16384;
      if (C > (p.N + minchunk - 1) / minchunk) C = (p.N + minchunk - 1) / minchunk;
      if (C < 1) C = 1;
      p.chunk = (p.N + C - 1) / C;
      p.chunk = (p.chunk + 7) & ~(int64_t)7;  // chunk starts stay 16-B aligned
      p.C = (p.N + p.chunk - 1) / p.chunk;
      if (int rc = scratch(p.O * p.C, p.O)) return rc;
      const int64_t work = p.O * p.C;
      k_red_rows_v<OP, T><<<(int)std::min<int64_t>(work, 1 << 30), 256, 0, st->s>>>(p, ws, cnt);
    }
  }
  TPG_LAUNCH_CHECK("reduce vec");
  if (ws) TPG_CUDA_CHECK(cudaFreeAsync(ws, st->s));
  done = true;
  return TPG_OK;
}

template <int OP, typename T>
void launch_flt(RedParams& p, Stream* st, bool col) {
  if (col) {
    const int64_t nob = (p.O + 255) / 256;
    const int64_t work = nob * p.C;
    const int g = (int)(work < (int64_t)1 << 30 ? work : (int64_t)1 << 30);
    k_red_cols_flt<OP, T><<<g, 256, 0, st->s>>>(p, nob);
  } else {
    const int64_t work = p.O * p.C;
    const int g = (int)(work < (int64_t)1 << 30 ? work : (int64_t)1 << 30);
    k_red_rows_flt<OP, T><<<g, 256, 0, st->s>>>(p);
  }
}

template <int OP, int KIND, int SDT>
void launch_main(RedParams& p, Stream* st, bool col) {
  if constexpr (KIND == K_FLT && SDT >= 0 &&
                (OP == TPG_RSUM || OP == TPG_RNORM || OP == TPG_RMIN || OP == TPG_RMAX)) {
    if (p.ndi == 1 && p.saligned) {
      if (SDT == TPG_DOUBLE) launch_flt<OP, double>(p, st, col);
      else launch_flt<OP, float>(p, st, col);
      return;
    }
  }
  if (col) {
    const int64_t nob = (p.O + 255) / 256;
    const int64_t work = nob * p.C;
    const int g = (int)(work < (int64_t)1 << 30 ? work : (int64_t)1 << 30);
    k_red_cols<OP, KIND, SDT><<<g, 256, 0, st->s>>>(p, nob);
  } else {
    const int64_t work = p.O * p.C;
    const int g = (int)(work < (int64_t)1 << 30 ? work : (int64_t)1 << 30);
    k_red_rows<OP, KIND, SDT><<<g, 256, 0, st->s>>>(p);
  }
}

template <int OP, int KIND>
int launch_red(RedParams& p, Stream* st, bool col) {
  const int dev = st->device;
  if (OP == TPG_RPRODUCT && KIND == K_CPX) {
    const int g = (int)std::min<int64_t>((p.O + 127) / 128, 65535);
    k_red_seq<OP, KIND><<<g, 128, 0, st->s>>>(p);
    TPG_LAUNCH_CHECK("reduce seq");
    return TPG_OK;
  }
  if constexpr (KIND == K_FLT && (OP == TPG_RSUM || OP == TPG_RNORM || OP == TPG_RMIN ||
                                  OP == TPG_RMAX)) {
    if (!p.sswap && p.saligned && (p.sdt == TPG_DOUBLE || p.sdt == TPG_FLOAT)) {
      bool done = false;
      const int rc = p.sdt == TPG_DOUBLE ? launch_vec<OP, double>(p, st, col, done)
                                         : launch_vec<OP, float>(p, st, col, done);
      if (rc != TPG_OK || done) return rc;
    }
  }
  const int64_t target = (int64_t)sm_count(dev) * 8;
  if (col) {
    const int64_t nob = (p.O + 255) / 256;
    int64_t C = (target + nob - 1) / nob;
    const int64_t minchunk = 64;
    if (C > (p.N + minchunk - 1) / minchunk) C = (p.N + minchunk - 1) / minchunk;
    if (C > 32) C = 32;  // partials of one output fit one warp in the finalize
    if (C < 1) C = 1;
    p.chunk = (p.N + C - 1) / C;
  } else {
    int64_t C = (target + p.O - 1) / p.O;
    const int64_t minchunk = 8192;
    if (C > (p.N + minchunk - 1) / minchunk) C = (p.N + minchunk - 1) / minchunk;
    if (C < 1) C = 1;
    p.chunk = (p.N + C - 1) / C;
  }
  p.C = (p.N + p.chunk - 1) / p.chunk;
  if (p.C < 1) p.C = 1;
  p.ws = nullptr;
  if (p.C > 1) TPG_CUDA_CHECK(cudaMallocAsync((void**)&p.ws, sizeof(Acc) * p.O * p.C, st->s));
  bool done = false;
  if constexpr (KIND == K_FLT) {
    if (!p.sswap && p.sdt == TPG_DOUBLE) { launch_main<OP, KIND, TPG_DOUBLE>(p, st, col); done = true; }
    else if (!p.sswap && p.sdt == TPG_FLOAT) { launch_main<OP, KIND, TPG_FLOAT>(p, st, col); done = true; }
  }
  if (!done) launch_main<OP, KIND, -1>(p, st, col);
  TPG_LAUNCH_CHECK("reduce launch");
  if (p.C > 1) {
    const int g = (int)(p.O < 65536 ? p.O : 65536);
    if (p.C <= 32) {
      const int gw = (int)std::min<int64_t>((p.O + 7) / 8, 65536);
      k_red_final_warp<OP, KIND><<<gw, 256, 0, st->s>>>(p);
    } else {
      k_red_final<OP, KIND><<<g, 256, 0, st->s>>>(p);
    }
    TPG_LAUNCH_CHECK("reduce finalize");
    TPG_CUDA_CHECK(cudaFreeAsync(p.ws, st->s));
  }
  return TPG_OK;
}

template <int OP>
int launch_kind(RedParams& p, Stream* st, bool col, int kind) {
  switch (kind) {
    case K_INT: return launch_red<OP, K_INT>(p, st, col);
    case K_UINT: return launch_red<OP, K_UINT>(p, st, col);
    case K_FLT: return launch_red<OP, K_FLT>(p, st, col);
    default: return launch_red<OP, K_CPX>(p, st, col);
  }
}

int reduce_sum_norm(int op, RedParams& p, Stream* st, bool col, int kind);
int reduce_minmax(int op, RedParams& p, Stream* st, bool col, int kind);
int reduce_other(int op, RedParams& p, Stream* st, bool col, int kind);

}  // namespace tpg
