// tpg_reduce.cu — axis and full reductions.
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
#include <cuda_runtime.h>

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
__device__ __forceinline__ void acc_feed(Acc& x, const RedParams& p, R16 r, int64_t idx) {
  if (p.sswap) r = swap_raw(p.sdt, r);
  if (OP == TPG_RSUM) {
    if (KIND == K_INT || KIND == K_UINT) x.v = (int64_t)((uint64_t)x.v + (uint64_t)dec_int(p.sdt, r));
    else if (KIND == K_FLT) dd_add(x.a, x.b, dec_flt(p.sdt, r));
    else {
      double2 z = dec_cpx(p.sdt, r);
      dd_add(x.a, x.b, z.x);
      dd_add(x.c, x.d, z.y);
    }
  } else if (OP == TPG_RPRODUCT) {
    if (KIND == K_INT || KIND == K_UINT) x.v = (int64_t)((uint64_t)x.v * (uint64_t)dec_int(p.sdt, r));
    else if (KIND == K_FLT) x.a = __dmul_rn(x.a, dec_flt(p.sdt, r));
    else {
      double2 z = dec_cpx(p.sdt, r);
      const double re = __dsub_rn(__dmul_rn(x.a, z.x), __dmul_rn(x.c, z.y));
      const double im = __dadd_rn(__dmul_rn(x.a, z.y), __dmul_rn(x.c, z.x));
      x.a = re;
      x.c = im;
    }
  } else if (OP == TPG_RMIN || OP == TPG_RMAX) {
    const bool mn = OP == TPG_RMIN;
    if (KIND == K_INT || KIND == K_UINT) {
      const int64_t v = dec_int(p.sdt, r);
      bool take;
      if (x.i < 0) take = true;
      else if (KIND == K_UINT) take = mn ? (uint64_t)v < (uint64_t)x.v : (uint64_t)v > (uint64_t)x.v;
      else take = mn ? v < x.v : v > x.v;
      if (take) { x.v = v; x.i = idx; }
    } else if (KIND == K_FLT) {
      const double v = dec_flt(p.sdt, r);
      if (isnan(v)) {
        // first element NaN sticks; p < 0 selects the NaN-skipping variant
        // used for per-shard partials (sharded.py)
        if (idx == 0 && p.p >= 0.0) { x.b = 1.0; x.d = v; }
        return;
      }
      if (x.i < 0 || (mn ? v < x.a : v > x.a)) { x.a = v; x.i = idx; }
    } else {
      const double2 z = dec_cpx(p.sdt, r);
      if (isnan(z.x)) {
        if (idx == 0) { x.b = 1.0; x.d = z.x; x.v = (int64_t)__double_as_longlong(z.y); }
        return;
      }
      const double2 cur = make_double2(x.a, x.c);
      if (x.i < 0 || (mn ? cpx_lt(z, cur) : cpx_gt(z, cur))) { x.a = z.x; x.c = z.y; x.i = idx; }
    }
  } else if (OP == TPG_RANY || OP == TPG_RALL) {
    bool nz;
    if (KIND == K_CPX) nz = cpx_nonzero(dec_cpx(p.sdt, r));
    else if (KIND == K_FLT) nz = dec_flt(p.sdt, r) != 0.0;
    else nz = dec_int(p.sdt, r) != 0;
    if (OP == TPG_RANY) x.v |= nz;
    else x.v &= nz;
  } else {  // norm
    double m;
    if (KIND == K_CPX) {
      double2 z = dec_cpx(p.sdt, r);
      m = hypot(z.x, z.y);
    } else if (KIND == K_FLT) {
      m = fabs(dec_flt(p.sdt, r));
    } else {
      const int64_t v = dec_int(p.sdt, r);
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

// row mode: one block per (output, chunk); threads stride the chunk.
template <int OP, int KIND>
__global__ void __launch_bounds__(256) k_red_rows(RedParams p) {
  __shared__ Acc sh[8];
  uint32_t st = 0;
  const int64_t nwork = p.O * p.C;
  for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int64_t o = w / p.C, c = w - o * p.C;
    int64_t doff, soff;
    outer_offsets(p, o, doff, soff);
    const int64_t j0 = c * p.chunk;
    const int64_t j1 = min(p.N, j0 + p.chunk);
    // each thread takes a contiguous sub-range in order so the combine
    // order follows plan order (ties / first-NaN rule / product order)
    const int64_t len = j1 - j0;
    const int64_t per = (len + 255) / 256;
    Acc x = acc_init<OP, KIND>();
    // strided (coalesced) pass: thread t handles j0 + t + 256*u
    constexpr int U = 4;
    for (int64_t jb = j0 + threadIdx.x; jb < j1; jb += 256 * U) {
      R16 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t j = jb + u * 256;
        if (j < j1) r[u] = load_raw(p.sdt, p.sbase + soff + inner_offset(p, j), p.saligned);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t j = jb + u * 256;
        if (j < j1) acc_feed<OP, KIND>(x, p, r[u], j);
      }
    }
    (void)per;
    x = warp_comb<OP, KIND>(x);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh[warp] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      Acc t = sh[0];
      for (int k = 1; k < 8; ++k) t = acc_comb<OP, KIND>(t, sh[k]);
      if (p.C == 1) acc_store<OP, KIND>(p, t, doff, st);
      else p.ws[o * p.C + c] = t;
    }
    __syncthreads();
  }
  if (st) atomicOr(p.flags, st);
}

// column mode: one thread per (output, chunk); outputs along outer axis 0
// are adjacent in memory so a warp's loads coalesce.
template <int OP, int KIND>
__global__ void __launch_bounds__(256) k_red_cols(RedParams p, int64_t nob) {
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
    Acc x = acc_init<OP, KIND>();
    constexpr int U = 8;
    for (int64_t jb = j0; jb < j1; jb += U) {
      R16 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (jb + u < j1) r[u] = load_raw(p.sdt, p.sbase + soff + inner_offset(p, jb + u), p.saligned);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (jb + u < j1) acc_feed<OP, KIND>(x, p, r[u], jb + u);
    }
    if (p.C == 1) acc_store<OP, KIND>(p, x, doff, st);
    else p.ws[o * p.C + c] = x;
  }
  if (st) atomicOr(p.flags, st);
}

// finalize: one warp per output combines its C partials in chunk order.
template <int OP, int KIND>
__global__ void __launch_bounds__(256) k_red_final(RedParams p) {
  uint32_t st = 0;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * 8;
  for (int64_t o = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); o < p.O; o += nw) {
    // lane l owns the contiguous partial range [l*per, (l+1)*per)
    const int64_t per = (p.C + 31) / 32;
    Acc x = acc_init<OP, KIND>();
    for (int64_t c = lane * per; c < min(p.C, (int64_t)(lane + 1) * per); ++c)
      x = acc_comb<OP, KIND>(x, p.ws[o * p.C + c]);
    x = warp_comb<OP, KIND>(x);
    if (lane == 0) {
      int64_t doff, soff;
      outer_offsets(p, o, doff, soff);
      acc_store<OP, KIND>(p, x, doff, st);
    }
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
      acc_feed<OP, KIND>(x, p, load_raw(p.sdt, p.sbase + soff + inner_offset(p, j), p.saligned), j);
    acc_store<OP, KIND>(p, x, doff, st);
  }
  if (st) atomicOr(p.flags, st);
}

template <int OP, int KIND>
static int launch_red(RedParams& p, Stream* st, bool col) {
  const int dev = st->device;
  if (OP == TPG_RPRODUCT && KIND == K_CPX) {
    const int g = (int)std::min<int64_t>((p.O + 127) / 128, 65535);
    k_red_seq<OP, KIND><<<g, 128, 0, st->s>>>(p);
    TPG_LAUNCH_CHECK("reduce seq");
    return TPG_OK;
  }
  const int64_t target = (int64_t)sm_count(dev) * 8;
  if (col) {
    const int64_t nob = (p.O + 255) / 256;
    int64_t C = (target + nob - 1) / nob;
    int64_t minchunk = 64;
    if (C > (p.N + minchunk - 1) / minchunk) C = (p.N + minchunk - 1) / minchunk;
    if (C < 1) C = 1;
    p.C = C;
    p.chunk = (p.N + C - 1) / C;
    p.C = (p.N + p.chunk - 1) / p.chunk;
    if (p.C < 1) p.C = 1;
  } else {
    int64_t C = (target + p.O - 1) / p.O;
    int64_t minchunk = 4096;
    if (C > (p.N + minchunk - 1) / minchunk) C = (p.N + minchunk - 1) / minchunk;
    if (C < 1) C = 1;
    p.C = C;
    p.chunk = (p.N + C - 1) / C;
    p.C = (p.N + p.chunk - 1) / p.chunk;
    if (p.C < 1) p.C = 1;
  }
  p.ws = nullptr;
  if (p.C > 1) TPG_CUDA_CHECK(cudaMallocAsync((void**)&p.ws, sizeof(Acc) * p.O * p.C, st->s));
  if (col) {
    const int64_t nob = (p.O + 255) / 256;
    int64_t work = nob * p.C;
    const int g = (int)(work < (int64_t)1 << 30 ? work : (int64_t)1 << 30);
    k_red_cols<OP, KIND><<<g, 256, 0, st->s>>>(p, nob);
  } else {
    int64_t work = p.O * p.C;
    const int g = (int)(work < (int64_t)1 << 30 ? work : (int64_t)1 << 30);
    k_red_rows<OP, KIND><<<g, 256, 0, st->s>>>(p);
  }
  TPG_LAUNCH_CHECK("reduce launch");
  if (p.C > 1) {
    int64_t blocks = (p.O + 7) / 8;
    const int g = (int)(blocks < 65536 ? blocks : 65536);
    k_red_final<OP, KIND><<<g, 256, 0, st->s>>>(p);
    TPG_LAUNCH_CHECK("reduce finalize");
    TPG_CUDA_CHECK(cudaFreeAsync(p.ws, st->s));
  }
  return TPG_OK;
}

template <int OP>
static int launch_kind(RedParams& p, Stream* st, bool col, int kind) {
  switch (kind) {
    case K_INT: return launch_red<OP, K_INT>(p, st, col);
    case K_UINT: return launch_red<OP, K_UINT>(p, st, col);
    case K_FLT: return launch_red<OP, K_FLT>(p, st, col);
    default: return launch_red<OP, K_CPX>(p, st, col);
  }
}

// empty inner range: write fin(init()) to every output (no element visited)
template <int OP, int KIND>
__global__ void k_red_empty(RedParams p) {
  uint32_t st = 0;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < p.O;
       o += (int64_t)gridDim.x * blockDim.x) {
    int64_t doff, soff;
    outer_offsets(p, o, doff, soff);
    acc_store<OP, KIND>(p, acc_init<OP, KIND>(), doff, st);
  }
}

}  // namespace tpg

using namespace tpg;

extern "C" int tpg_reduce(tpg_stream stream, int op, double pnorm, const tpg_plan* outer,
                          const tpg_plan* inner, const tpg_operand* d, const tpg_operand* a,
                          int compute, int mode) {
  (void)compute;
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  if (!outer || !inner || !d || !a || !d->base || !a->base) return arg_fail("reduce: null argument");
  if (op < TPG_RSUM || op > TPG_RNORM) return arg_fail("bad reduce op");
  if (outer->ndim < 0 || outer->ndim > TPG_MAX_DIMS || inner->ndim < 0 || inner->ndim > TPG_MAX_DIMS)
    return arg_fail("reduce: bad plan ndim");
  RedParams p;
  memset(&p, 0, sizeof(p));
  p.ndo = outer->ndim;
  p.O = 1;
  for (int k = 0; k < p.ndo; ++k) {
    p.eo[k] = outer->extent[k];
    p.so_d[k] = outer->stride[0][k];
    p.so_s[k] = outer->stride[1][k];
    p.O *= p.eo[k];
  }
  p.ndi = inner->ndim;
  p.N = 1;
  for (int k = 0; k < p.ndi; ++k) {
    p.ei[k] = inner->extent[k];
    p.si[k] = inner->stride[0][k];
    p.N *= p.ei[k];
  }
  if (p.ndi == 0) {
    p.ndi = 1;
    p.ei[0] = 1;
    p.si[0] = 0;
  }
  if (p.O == 0) return TPG_OK;
  p.dbase = (char*)d->base + d->offset;
  p.sbase = (const char*)a->base + a->offset;
  p.ddt = d->dtype;
  p.sdt = a->dtype;
  p.dswap = d->big_endian;
  p.sswap = a->big_endian;
  {
    int al = std::min(dt_size(p.ddt), 8);
    bool ok = ((uintptr_t)p.dbase % al) == 0;
    for (int k = 0; k < p.ndo; ++k)
      if (p.eo[k] > 1 && p.so_d[k] % al) ok = false;
    p.daligned = ok;
    al = std::min(dt_size(p.sdt), 8);
    ok = ((uintptr_t)p.sbase % al) == 0;
    for (int k = 0; k < p.ndo; ++k)
      if (p.eo[k] > 1 && p.so_s[k] % al) ok = false;
    for (int k = 0; k < p.ndi; ++k)
      if (p.ei[k] > 1 && p.si[k] % al) ok = false;
    p.saligned = ok;
  }
  p.track = mode == TPG_WARNING || mode == TPG_ERROR;
  p.p = pnorm;
  p.flags = device_flags(st->device);
  const int kind = dt_kind(p.sdt);
  if (p.N == 0) {
    if (op == TPG_RMIN || op == TPG_RMAX) return arg_fail("min/max of an empty range");
    const int g = (int)std::min<int64_t>((p.O + 255) / 256, 65535);
#define EMPTY(OPX)                                                         \
  case OPX:                                                                \
    switch (kind) {                                                        \
      case K_INT: k_red_empty<OPX, K_INT><<<g, 256, 0, st->s>>>(p); break;   \
      case K_UINT: k_red_empty<OPX, K_UINT><<<g, 256, 0, st->s>>>(p); break; \
      case K_FLT: k_red_empty<OPX, K_FLT><<<g, 256, 0, st->s>>>(p); break;   \
      default: k_red_empty<OPX, K_CPX><<<g, 256, 0, st->s>>>(p); break;      \
    }                                                                      \
    break;
    switch (op) {
      EMPTY(TPG_RSUM)
      EMPTY(TPG_RPRODUCT)
      EMPTY(TPG_RANY)
      EMPTY(TPG_RALL)
      default: EMPTY(TPG_RNORM)
    }
#undef EMPTY
    TPG_LAUNCH_CHECK("reduce empty");
    return TPG_OK;
  }
  // column mode when the innermost reduced stride is large and adjacent
  // outputs are adjacent in the source
  const int s = dt_size(p.sdt);
  const int64_t si0 = p.si[0] < 0 ? -p.si[0] : p.si[0];
  const int64_t so0 = p.ndo > 0 ? (p.so_s[0] < 0 ? -p.so_s[0] : p.so_s[0]) : 0;
  const bool col = p.ndo > 0 && p.O >= 32 && so0 <= 2 * s && si0 > 2 * s;
  switch (op) {
    case TPG_RSUM: return launch_kind<TPG_RSUM>(p, st, col, kind);
    case TPG_RPRODUCT: return launch_kind<TPG_RPRODUCT>(p, st, col, kind);
    case TPG_RMIN: return launch_kind<TPG_RMIN>(p, st, col, kind);
    case TPG_RMAX: return launch_kind<TPG_RMAX>(p, st, col, kind);
    case TPG_RANY: return launch_kind<TPG_RANY>(p, st, col, kind);
    case TPG_RALL: return launch_kind<TPG_RALL>(p, st, col, kind);
    default: return launch_kind<TPG_RNORM>(p, st, col, kind);
  }
}
