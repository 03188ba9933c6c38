/*
 * tp_oracle.c — TEST INFRASTRUCTURE ONLY.  A plain-C restatement of the
 * reference tidepool core loops (pkg/src/tidepool/kernels.py) and of the
 * scalar semantics they are driven with (dtypes.py, ops.py), used as the
 * CPU oracle that the CUDA path is checked against and as the CPU baseline
 * of bench.py.  Nothing in the product links or calls this file.
 *
 * It follows the reference loop structure deliberately (odometer walk over
 * an IterPlan, one element at a time, Python value semantics):
 *   binary   kernels.binary_elementwise      kernels.py:213-248
 *            + ops._prepare dtype convert    ops.py:121-142
 *            + binary_scalar_fn              kernels.py:50-81
 *   unary    kernels.unary_elementwise       kernels.py:275-302
 *            + unary_scalar_fn / UNARY_TABLE kernels.py:121-158
 *   copy     ops._run_copy (identity fn)     ops.py:668-687
 *   reduce   kernels.reduce_strided          kernels.py:305-320
 *            + ops._reduction_acc            ops.py:522-556
 *            + make_sum_acc (Neumaier)       kernels.py:169-198
 *   matmul   kernels.matmul                  kernels.py:323-340
 *   fill / arange / byteswap                 kernels.py:343-381
 *   store    ops._make_store -> cast_scalar  ops.py:145-152, dtypes.py:281-325
 * Python ints are unbounded; here they are __int128 (enough for every
 * single product/sum of 64-bit operands) and accumulations that could
 * exceed it are kept modulo 2^64, which is exact after the final wrap to a
 * <=64-bit dtype.  Transcendentals call glibc libm, which is what CPython's
 * math module calls.  Complex transcendentals use C99 <complex.h>
 * (CPython's cmath has its own algorithms: tolerance-level agreement only).
 *
 * Parity of this file against the reference itself is pinned by
 * tests/test_oracle_golden.py over the vectors in tests/golden/, which
 * tests/golden/make_golden.py captured from the reference's own cpu table.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/tidepool_gpu.h"
#ifdef _OPENMP
#include <omp.h>
#endif

typedef __int128 i128;

enum { VK_INT = 0, VK_FLT = 1, VK_CPX = 2 };

typedef struct {
  int k;
  i128 i;
  double re, im;
} Val;

static int dsize(int dt) {
  static const int s[16] = {1, 1, 1, 2, 2, 4, 4, 8, 8, 2, 4, 8, 4, 8, 16, 2};
  return s[dt];
}
static int is_cpx(int dt) { return dt >= TPG_CHALF && dt <= TPG_CDOUBLE; }
static int is_flt(int dt) { return (dt >= TPG_HALF && dt <= TPG_CDOUBLE) || dt == TPG_BF16; }
static int is_signed_int(int dt) {
  return dt == TPG_INT8 || dt == TPG_INT16 || dt == TPG_INT32 || dt == TPG_INT64;
}
static int real_of(int dt) {
  return dt == TPG_CHALF ? TPG_HALF : dt == TPG_CFLOAT ? TPG_FLOAT : dt == TPG_CDOUBLE ? TPG_DOUBLE : dt;
}

/* ---------------------------------------------------------------- halves */
static double half_to_double(uint16_t h) {
  int s = h >> 15, e = (h >> 10) & 0x1f, f = h & 0x3ff;
  double v;
  if (e == 0) v = ldexp((double)f, -24);
  else if (e == 31) v = f ? NAN : INFINITY;
  else v = ldexp((double)(f | 0x400), e - 25);
  return s ? -v : v;
}

/* struct.pack('<e', x): round-half-even, overflow -> +-inf (the reference
 * catches OverflowError and substitutes inf, dtypes.py:275-278). */
static uint16_t double_to_half(double x) {
  uint16_t sign = signbit(x) ? 0x8000 : 0;
  double a = fabs(x);
  if (isnan(x)) return sign | 0x7e00;
  if (isinf(a)) return sign | 0x7c00;
  if (a == 0.0) return sign;
  int e;
  double m = frexp(a, &e); /* a = m * 2^e, m in [0.5, 1) */
  /* normal half: exponent range e-1 in [-14, 15] */
  int exp_h = e - 1;
  double scaled;
  if (exp_h < -14) {
    scaled = ldexp(a, 24); /* subnormal units of 2^-24 */
    double r = nearbyint(scaled); /* default rounding mode: RNE */
    if (r >= 1024.0) return sign | 0x0400;
    return sign | (uint16_t)r;
  }
  scaled = ldexp(m, 11); /* in [1024, 2048) */
  double r = nearbyint(scaled);
  if (r >= 2048.0) {
    r = 1024.0;
    exp_h += 1;
  }
  if (exp_h > 15) return sign | 0x7c00;
  return sign | (uint16_t)(((exp_h + 15) << 10) | ((uint16_t)r - 1024));
}

static double bf16_to_double(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static uint16_t double_to_bf16(double x) {
  if (isnan(x)) return signbit(x) ? 0xffc0 : 0x7fc0;
  uint16_t sign = signbit(x) ? 0x8000 : 0;
  double a = fabs(x);
  if (a == 0.0) return sign;
  int e;
  double m = frexp(a, &e);
  int exp_b = e - 1;
  if (exp_b < -126) {
    double r = nearbyint(ldexp(a, 133));
    if (r >= 128.0) return sign | 0x0080;
    return sign | (uint16_t)r;
  }
  double r = nearbyint(ldexp(m, 8));
  if (r >= 256.0) {
    r = 128.0;
    exp_b += 1;
  }
  if (exp_b > 127) return sign | 0x7f80;
  return sign | (uint16_t)(((exp_b + 127) << 7) | ((uint16_t)r - 128));
}

/* ---------------------------------------------------------------- codec */
static void get_bytes(const uint8_t* p, int n, int be, uint8_t* out) {
  for (int i = 0; i < n; ++i) out[i] = be ? p[n - 1 - i] : p[i];
}
static void put_bytes(uint8_t* p, int n, int be, const uint8_t* in) {
  for (int i = 0; i < n; ++i) p[i] = be ? in[n - 1 - i] : in[i];
}

static double real_load(int rdt, const uint8_t* p, int be) {
  uint8_t b[8];
  switch (rdt) {
    case TPG_HALF: {
      uint16_t h;
      get_bytes(p, 2, be, b);
      memcpy(&h, b, 2);
      return half_to_double(h);
    }
    case TPG_BF16: {
      uint16_t h;
      get_bytes(p, 2, be, b);
      memcpy(&h, b, 2);
      return bf16_to_double(h);
    }
    case TPG_FLOAT: {
      float f;
      get_bytes(p, 4, be, b);
      memcpy(&f, b, 4);
      return f;
    }
    default: {
      double d;
      get_bytes(p, 8, be, b);
      memcpy(&d, b, 8);
      return d;
    }
  }
}

/* dtypes.codec unpack: Python value of one element */
static Val unpack(int dt, const uint8_t* p, int be) {
  Val v;
  memset(&v, 0, sizeof(v));
  if (is_cpx(dt)) {
    int r = real_of(dt), cs = dsize(dt) / 2;
    v.k = VK_CPX;
    v.re = real_load(r, p, be);
    v.im = real_load(r, p + cs, be);
    return v;
  }
  if (is_flt(dt)) {
    v.k = VK_FLT;
    v.re = real_load(dt, p, be);
    return v;
  }
  v.k = VK_INT;
  uint8_t b[8];
  int n = dsize(dt);
  get_bytes(p, n, be, b);
  switch (dt) {
    case TPG_BOOL: v.i = b[0] != 0; break;
    case TPG_INT8: { int8_t x; memcpy(&x, b, 1); v.i = x; } break;
    case TPG_UINT8: { uint8_t x; memcpy(&x, b, 1); v.i = x; } break;
    case TPG_INT16: { int16_t x; memcpy(&x, b, 2); v.i = x; } break;
    case TPG_UINT16: { uint16_t x; memcpy(&x, b, 2); v.i = x; } break;
    case TPG_INT32: { int32_t x; memcpy(&x, b, 4); v.i = x; } break;
    case TPG_UINT32: { uint32_t x; memcpy(&x, b, 4); v.i = x; } break;
    case TPG_INT64: { int64_t x; memcpy(&x, b, 8); v.i = x; } break;
    default: { uint64_t x; memcpy(&x, b, 8); v.i = x; } break;
  }
  return v;
}

static void real_store(int rdt, uint8_t* p, int be, double x) {
  uint8_t b[8];
  switch (rdt) {
    case TPG_HALF: {
      uint16_t h = double_to_half(x);
      memcpy(b, &h, 2);
      put_bytes(p, 2, be, b);
      break;
    }
    case TPG_BF16: {
      uint16_t h = double_to_bf16(x);
      memcpy(b, &h, 2);
      put_bytes(p, 2, be, b);
      break;
    }
    case TPG_FLOAT: {
      float f = (float)x; /* C cast: round-to-nearest-even, overflow -> inf */
      memcpy(b, &f, 4);
      put_bytes(p, 4, be, b);
      break;
    }
    default:
      memcpy(b, &x, 8);
      put_bytes(p, 8, be, b);
  }
}

static void int_range(int dt, i128* lo, i128* hi) {
  int bits = 8 * dsize(dt);
  if (is_signed_int(dt)) {
    *lo = -((i128)1 << (bits - 1));
    *hi = ((i128)1 << (bits - 1)) - 1;
  } else {
    *lo = 0;
    *hi = ((i128)1 << bits) - 1;
  }
}

/* dtypes._wrap_int */
static i128 wrap_int(i128 v, int dt) {
  int bits = 8 * dsize(dt);
  unsigned __int128 m = ((unsigned __int128)1 << bits) - 1;
  unsigned __int128 u = (unsigned __int128)v & m;
  if (is_signed_int(dt) && (u >> (bits - 1)) & 1) return (i128)u - ((i128)1 << bits);
  return (i128)u;
}

/* int(trunc(x)) for a finite double, exact; magnitudes >= 2^127 are
 * multiples of 2^75, i.e. 0 modulo 2^64, which is all a wrap needs. */
static i128 trunc_to_i128(double x, int* huge) {
  double t = trunc(x);
  *huge = fabs(t) >= 1.7014118346046923e38;
  if (*huge) return 0;
  return (i128)t;
}

/* dtypes.cast_scalar (standard/warning/error share the value; loss sets
 * TPG_FLAG_CAST_LOSS, which the caller maps to ctx.domain_loss). */
static void store(int dt, uint8_t* p, int be, Val v, uint32_t* st) {
  if (v.k == VK_CPX && !is_cpx(dt)) {
    if (v.im != 0.0) *st |= TPG_FLAG_CAST_LOSS;
    v.k = VK_FLT;
  }
  if (dt == TPG_BOOL) {
    int t = v.k == VK_INT ? v.i != 0 : v.re != 0.0;
    p[0] = (uint8_t)t;
    return;
  }
  if (is_cpx(dt)) {
    int r = real_of(dt), cs = dsize(dt) / 2;
    double re, im;
    if (v.k == VK_CPX) { re = v.re; im = v.im; }
    else if (v.k == VK_FLT) { re = v.re; im = 0.0; }
    else { re = (double)v.i; im = 0.0; }
    real_store(r, p, be, re);
    real_store(r, p + cs, be, im);
    return;
  }
  if (is_flt(dt)) {
    double x = v.k == VK_INT ? (double)v.i : v.re; /* float(int): RNE */
    real_store(dt, p, be, x);
    return;
  }
  i128 iv;
  if (v.k == VK_FLT) {
    if (isnan(v.re) || isinf(v.re)) {
      *st |= TPG_FLAG_CAST_LOSS;
      iv = 0;
    } else {
      int huge;
      iv = trunc_to_i128(v.re, &huge);
      if (huge) *st |= TPG_FLAG_CAST_LOSS;
      i128 lo, hi;
      int_range(dt, &lo, &hi);
      if (!huge && (iv < lo || iv > hi)) *st |= TPG_FLAG_CAST_LOSS;
    }
  } else {
    iv = v.i;
    i128 lo, hi;
    int_range(dt, &lo, &hi);
    if (iv < lo || iv > hi) *st |= TPG_FLAG_CAST_LOSS;
  }
  iv = wrap_int(iv, dt);
  uint8_t b[8];
  uint64_t u = (uint64_t)iv;
  memcpy(b, &u, 8); /* little-endian host: low bytes first */
  put_bytes(p, dsize(dt), be, b);
}

/* cast to the compute dtype (ops._prepare -> _dtype_convert): Python value
 * of cast_scalar(v, compute) */
static Val to_compute(Val v, int src_dt, int compute) {
  if (src_dt == compute) return v;
  uint8_t tmp[16];
  uint32_t st = 0;
  store(compute, tmp, 0, v, &st);
  return unpack(compute, tmp, 0);
}

static int compute_kind(int compute) {
  return is_cpx(compute) ? VK_CPX : is_flt(compute) ? VK_FLT : VK_INT;
}

/* ---------------------------------------------------------------- binary */
static Val mk_int(i128 i) { Val v; memset(&v, 0, sizeof v); v.k = VK_INT; v.i = i; return v; }
static Val mk_flt(double d) { Val v; memset(&v, 0, sizeof v); v.k = VK_FLT; v.re = d; return v; }
static Val mk_cpx(double re, double im) {
  Val v; memset(&v, 0, sizeof v); v.k = VK_CPX; v.re = re; v.im = im; return v;
}
static double as_f(Val v) { return v.k == VK_INT ? (double)v.i : v.re; }
static Val as_c(Val v) { return v.k == VK_CPX ? v : mk_cpx(as_f(v), 0.0); }

/* tuple comparison (a.real, a.imag) op (b.real, b.imag) */
static int tup_le(Val a, Val b) { return a.re != b.re ? a.re < b.re : a.im <= b.im; }
static int tup_ge(Val a, Val b) { return a.re != b.re ? a.re > b.re : a.im >= b.im; }
static int tup_lt(Val a, Val b) { return a.re != b.re ? a.re < b.re : a.im < b.im; }
static int tup_gt(Val a, Val b) { return a.re != b.re ? a.re > b.re : a.im > b.im; }

/* CPython _Py_c_quot */
static Val c_quot(Val a, Val b) {
  double abr = b.re < 0 ? -b.re : b.re, abi = b.im < 0 ? -b.im : b.im;
  if (abr >= abi) {
    if (abr == 0.0) return mk_cpx(0.0, 0.0);
    double ratio = b.im / b.re, denom = b.re + b.im * ratio;
    return mk_cpx((a.re + a.im * ratio) / denom, (a.im - a.re * ratio) / denom);
  } else if (abi >= abr) {
    double ratio = b.re / b.im, denom = b.re * ratio + b.im;
    return mk_cpx((a.re * ratio + a.im) / denom, (a.im * ratio - a.re) / denom);
  }
  return mk_cpx(NAN, NAN);
}

static Val bin_fn(int op, int kind, Val a, Val b, int mode, uint32_t* st) {
  (void)mode;
  if (kind == VK_INT) {
    i128 x = a.i, y = b.i;
    switch (op) {
      case TPG_ADD: return mk_int(x + y);
      case TPG_SUBTRACT: return mk_int(x - y);
      case TPG_MULTIPLY: return mk_int(x * y);
      case TPG_DIVIDE: {
        if (y == 0) {
          *st |= TPG_FLAG_INT_DIV0;
          return mk_int(0);
        }
        i128 ax = x < 0 ? -x : x, ay = y < 0 ? -y : y;
        i128 q = ax / ay;
        return mk_int(((x < 0) != (y < 0)) ? -q : q);
      }
      case TPG_MINIMUM: return x <= y ? a : b;
      default: return x >= y ? a : b;
    }
  }
  if (kind == VK_FLT) {
    double x = a.re, y = b.re;
    switch (op) {
      case TPG_ADD: return mk_flt(x + y);
      case TPG_SUBTRACT: return mk_flt(x - y);
      case TPG_MULTIPLY: return mk_flt(x * y);
      case TPG_DIVIDE:
        if (y == 0.0) {
          if (x == 0.0 || isnan(x)) return mk_flt(NAN);
          return mk_flt(copysign(INFINITY, x) * copysign(1.0, y));
        }
        return mk_flt(x / y);
      case TPG_MINIMUM: return x <= y ? a : b;
      default: return x >= y ? a : b;
    }
  }
  switch (op) {
    case TPG_ADD: return mk_cpx(a.re + b.re, a.im + b.im);
    case TPG_SUBTRACT: return mk_cpx(a.re - b.re, a.im - b.im);
    case TPG_MULTIPLY: {
      volatile double p1 = a.re * b.re, p2 = a.im * b.im, p3 = a.re * b.im, p4 = a.im * b.re;
      return mk_cpx(p1 - p2, p3 + p4);
    }
    case TPG_DIVIDE:
      if (b.re == 0.0 && b.im == 0.0) return mk_cpx(NAN, NAN);
      return c_quot(a, b);
    case TPG_MINIMUM: return tup_le(a, b) ? a : b;
    default: return tup_ge(a, b) ? a : b;
  }
}

/* ---------------------------------------------------------------- plans */
/* odometer walk of an IterPlan, IterPlan.offsets (tensors.py:545-567) */
typedef struct {
  int nd, nv;
  int64_t ext[TPG_MAX_DIMS];
  int64_t str[TPG_MAX_VIEWS][TPG_MAX_DIMS];
  int64_t idx[TPG_MAX_DIMS];
  int64_t off[TPG_MAX_VIEWS];
} Walk;

static int64_t walk_init(Walk* w, const tpg_plan* p, int nviews, const int64_t* bases) {
  memset(w, 0, sizeof(*w));
  w->nd = p->ndim;
  w->nv = nviews;
  int64_t total = 1;
  for (int k = 0; k < w->nd; ++k) {
    w->ext[k] = p->extent[k];
    total *= p->extent[k];
    for (int v = 0; v < nviews; ++v) w->str[v][k] = p->stride[v][k];
  }
  for (int v = 0; v < nviews; ++v) w->off[v] = bases[v];
  return total;
}

/* position the walk at linear index i (for parallel chunks) */
static void walk_seek(Walk* w, const int64_t* bases, int64_t i) {
  for (int v = 0; v < w->nv; ++v) w->off[v] = bases[v];
  for (int k = 0; k < w->nd; ++k) {
    w->idx[k] = i % w->ext[k];
    i /= w->ext[k];
    for (int v = 0; v < w->nv; ++v) w->off[v] += w->idx[k] * w->str[v][k];
  }
}

static void walk_next(Walk* w) {
  for (int k = 0; k < w->nd; ++k) {
    w->idx[k] += 1;
    for (int v = 0; v < w->nv; ++v) w->off[v] += w->str[v][k];
    if (w->idx[k] < w->ext[k]) return;
    w->idx[k] = 0;
    for (int v = 0; v < w->nv; ++v) w->off[v] -= w->str[v][k] * w->ext[k];
  }
}

static const uint8_t* obase(const tpg_operand* o) { return (const uint8_t*)o->base; }

static Val load_op(const tpg_operand* o, int64_t off) {
  if (o->base == NULL) return unpack(o->dtype, (const uint8_t*)o->imm, o->big_endian);
  return unpack(o->dtype, obase(o) + off, o->big_endian);
}

/* ---------------------------------------------------------------- entries */
int tpo_binary(int op, const tpg_plan* plan, const tpg_operand* d, const tpg_operand* a,
               const tpg_operand* b, int compute, int mode, uint32_t* status) {
  int64_t bases[3] = {d->offset, a->offset, b->offset};
  int kind = compute_kind(compute);
  uint32_t st = 0;
  Walk w0;
  int64_t total = walk_init(&w0, plan, 3, bases);
  if (total == 0) return 0;
#pragma omp parallel reduction(| : st)
  {
    int nt = 1, tid = 0;
#ifdef _OPENMP
    nt = omp_get_num_threads();
    tid = omp_get_thread_num();
#endif
    int64_t lo = total * tid / nt, hi = total * (tid + 1) / nt;
    Walk w = w0;
    walk_seek(&w, bases, lo);
    for (int64_t i = lo; i < hi; ++i) {
      Val va = to_compute(load_op(a, w.off[1]), a->dtype, compute);
      Val vb = to_compute(load_op(b, w.off[2]), b->dtype, compute);
      Val r = bin_fn(op, kind, va, vb, mode, &st);
      store(d->dtype, (uint8_t*)d->base + w.off[0], d->big_endian, r, &st);
      walk_next(&w);
    }
  }
  *status |= st;
  return 0;
}

static Val un_fn(int op, int kind, Val v, int force_complex, uint32_t* st) {
  if (kind == VK_CPX || force_complex) {
    double complex z = CMPLX(as_c(v).re, as_c(v).im), r;
    switch (op) {
      case TPG_NEGATE: return mk_cpx(-creal(z), -cimag(z));
      case TPG_ABSOLUTE: return mk_flt(hypot(creal(z), cimag(z)));
      case TPG_SQRT: r = csqrt(z); break;
      case TPG_EXP: r = cexp(z); break;
      case TPG_LOG:
        if (creal(z) == 0.0 && cimag(z) == 0.0) return mk_cpx(-INFINITY, 0.0);
        r = clog(z);
        break;
      case TPG_SIN: r = csin(z); break;
      case TPG_COS: r = ccos(z); break;
      case TPG_ASIN: r = casin(z); break;
      case TPG_ACOS: r = cacos(z); break;
      case TPG_CONJ: return mk_cpx(creal(z), -cimag(z));
      default: return v;
    }
    return mk_cpx(creal(r), cimag(r));
  }
  if (kind == VK_FLT) {
    double x = v.re;
    switch (op) {
      case TPG_NEGATE: return mk_flt(-x);
      case TPG_ABSOLUTE: return mk_flt(fabs(x));
      case TPG_SQRT:
        if (x < 0.0) { *st |= TPG_FLAG_DOMAIN; return mk_flt(NAN); }
        return mk_flt(isnan(x) ? NAN : sqrt(x));
      case TPG_EXP: return mk_flt(isnan(x) ? NAN : exp(x));
      case TPG_LOG:
        if (x < 0.0) { *st |= TPG_FLAG_DOMAIN; return mk_flt(NAN); }
        if (isnan(x)) return mk_flt(NAN);
        if (x == 0.0) return mk_flt(-INFINITY);
        return mk_flt(log(x));
      case TPG_SIN: return mk_flt(isnan(x) ? NAN : sin(x));
      case TPG_COS: return mk_flt(isnan(x) ? NAN : cos(x));
      case TPG_ASIN:
        if (fabs(x) > 1.0) { *st |= TPG_FLAG_DOMAIN; return mk_flt(NAN); }
        return mk_flt(isnan(x) ? NAN : asin(x));
      case TPG_ACOS:
        if (fabs(x) > 1.0) { *st |= TPG_FLAG_DOMAIN; return mk_flt(NAN); }
        return mk_flt(isnan(x) ? NAN : acos(x));
      default: return v;
    }
  }
  switch (op) {
    case TPG_NEGATE: return mk_int(-v.i);
    case TPG_ABSOLUTE: return mk_int(v.i < 0 ? -v.i : v.i);
    default: return v;
  }
}

int tpo_unary(int op, const tpg_plan* plan, const tpg_operand* d, const tpg_operand* a,
              int compute, int mode, int force_complex, uint32_t* status) {
  (void)mode;
  int64_t bases[2] = {d->offset, a->offset};
  uint32_t st = 0;
  Walk w0;
  int64_t total = walk_init(&w0, plan, 2, bases);
  if (total == 0) return 0;
  const int identity = op == TPG_IDENTITY;
  const int kind = compute_kind(compute);
#pragma omp parallel reduction(| : st)
  {
    int nt = 1, tid = 0;
#ifdef _OPENMP
    nt = omp_get_num_threads();
    tid = omp_get_thread_num();
#endif
    int64_t lo = total * tid / nt, hi = total * (tid + 1) / nt;
    Walk w = w0;
    walk_seek(&w, bases, lo);
    for (int64_t i = lo; i < hi; ++i) {
      Val v = load_op(a, w.off[1]);
      Val r;
      if (identity) r = v;
      else r = un_fn(op, kind, to_compute(v, a->dtype, compute), force_complex, &st);
      store(d->dtype, (uint8_t*)d->base + w.off[0], d->big_endian, r, &st);
      walk_next(&w);
    }
  }
  *status |= st;
  return 0;
}

/* ---------------------------------------------------------------- reduce */
static void neumaier(double* s, double* c, double v) {
  double t = *s + v;
  if (fabs(*s) >= fabs(v)) *c += (*s - t) + v;
  else *c += (v - t) + *s;
  *s = t;
}

typedef struct {
  double s, c, s2, c2; /* Neumaier pairs (re / im) */
  i128 iacc;
  uint64_t uacc;
  Val best;
  int have;
  int flag;
} RAcc;

static void racc_init(RAcc* r, int op) {
  memset(r, 0, sizeof(*r));
  if (op == TPG_RPRODUCT) {
    r->s = 1.0;
    r->uacc = 1;
  }
  if (op == TPG_RALL) r->flag = 1;
}

static void racc_step(RAcc* r, int op, int kind, Val v, double p) {
  switch (op) {
    case TPG_RSUM:
      if (kind == VK_INT) r->iacc += v.i;
      else if (kind == VK_FLT) neumaier(&r->s, &r->c, v.re);
      else {
        Val z = as_c(v);
        neumaier(&r->s, &r->c, z.re);
        neumaier(&r->s2, &r->c2, z.im);
      }
      break;
    case TPG_RPRODUCT:
      if (kind == VK_INT) r->uacc *= (uint64_t)v.i;
      else if (kind == VK_FLT) r->s *= v.re;
      else {
        Val z = as_c(v);
        volatile double p1 = r->s * z.re, p2 = r->s2 * z.im, p3 = r->s * z.im, p4 = r->s2 * z.re;
        double re = p1 - p2, im = p3 + p4;
        r->s = re;
        r->s2 = im;
      }
      break;
    case TPG_RMIN:
    case TPG_RMAX: {
      int mn = op == TPG_RMIN;
      int take;
      if (!r->have) take = 1;
      else if (kind == VK_INT) take = mn ? v.i < r->best.i : v.i > r->best.i;
      else if (kind == VK_FLT) take = mn ? v.re < r->best.re : v.re > r->best.re;
      else take = mn ? tup_lt(v, r->best) : tup_gt(v, r->best);
      if (take) {
        r->best = v;
        r->have = 1;
      }
      break;
    }
    case TPG_RANY:
    case TPG_RALL: {
      int nz = v.k == VK_INT ? v.i != 0 : (v.k == VK_FLT ? v.re != 0.0 : (v.re != 0.0 || v.im != 0.0));
      if (op == TPG_RANY) r->flag = r->flag || nz;
      else r->flag = r->flag && nz;
      break;
    }
    default: { /* norm: step(acc, abs(v) ** p) with a double Neumaier acc */
      double m;
      if (v.k == VK_CPX) m = hypot(v.re, v.im);
      else if (v.k == VK_FLT) m = fabs(v.re);
      else m = (double)(v.i < 0 ? -v.i : v.i);
      neumaier(&r->s, &r->c, pow(m, p));
    }
  }
}

static Val racc_fin(RAcc* r, int op, int kind, double p) {
  switch (op) {
    case TPG_RSUM:
      if (kind == VK_INT) return mk_int(r->iacc);
      if (kind == VK_FLT) return mk_flt(r->s + r->c);
      return mk_cpx(r->s + r->c, r->s2 + r->c2);
    case TPG_RPRODUCT:
      if (kind == VK_INT) return mk_int((i128)(int64_t)r->uacc);
      if (kind == VK_FLT) return mk_flt(r->s);
      return mk_cpx(r->s, r->s2);
    case TPG_RMIN:
    case TPG_RMAX: return r->best;
    case TPG_RANY:
    case TPG_RALL: return mk_int(r->flag);
    default: return mk_flt(pow(r->s + r->c, 1.0 / p));
  }
}

int tpo_reduce(int op, double p, const tpg_plan* outer, const tpg_plan* inner,
               const tpg_operand* d, const tpg_operand* a, int compute, int mode,
               uint32_t* status) {
  (void)mode;
  (void)compute;
  int64_t obases[2] = {d->offset, a->offset};
  Walk wo0;
  int64_t O = walk_init(&wo0, outer, 2, obases);
  int64_t N = 1;
  for (int k = 0; k < inner->ndim; ++k) N *= inner->extent[k];
  if (O == 0) return 0;
  if (N == 0 && (op == TPG_RMIN || op == TPG_RMAX)) return -1; /* reference: TypeError */
  /* the value kind of the source elements (the reference compute type for
   * sum/product/min/max is widen(src); any/all/norm take raw values) */
  int kind = is_cpx(a->dtype) ? VK_CPX : is_flt(a->dtype) ? VK_FLT : VK_INT;
  uint32_t st = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : st) if (O > 1)
  for (int64_t o = 0; o < O; ++o) {
    Walk wo = wo0;
    walk_seek(&wo, obases, o);
    RAcc acc;
    racc_init(&acc, op);
    int64_t ib[1] = {wo.off[1]};
    Walk wi;
    walk_init(&wi, inner, 1, ib);
    for (int64_t j = 0; j < N; ++j) {
      racc_step(&acc, op, kind, unpack(a->dtype, obase(a) + wi.off[0], a->big_endian), p);
      walk_next(&wi);
    }
    Val r = racc_fin(&acc, op, kind, p);
    store(d->dtype, (uint8_t*)d->base + wo.off[0], d->big_endian, r, &st);
  }
  *status |= st;
  return 0;
}

/* ---------------------------------------------------------------- matmul */
int tpo_matmul(const tpg_operand* d, const int64_t* ds, const tpg_operand* a,
               const int64_t* as, const tpg_operand* b, const int64_t* bs, int64_t m,
               int64_t n, int64_t k, int compute, int mode, uint32_t* status) {
  (void)mode;
  int kind = compute_kind(compute);
  uint32_t st = 0;
#pragma omp parallel for collapse(2) schedule(static) reduction(| : st)
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t i = 0; i < m; ++i) {
      double s = 0, c = 0, s2 = 0, c2 = 0;
      uint64_t iacc = 0;
      int64_t ao = a->offset + i * as[0], bo = b->offset + j * bs[1];
      for (int64_t q = 0; q < k; ++q) {
        Val x = to_compute(unpack(a->dtype, obase(a) + ao, a->big_endian), a->dtype, compute);
        Val y = to_compute(unpack(b->dtype, obase(b) + bo, b->big_endian), b->dtype, compute);
        if (kind == VK_INT) iacc += (uint64_t)x.i * (uint64_t)y.i;
        else if (kind == VK_FLT) neumaier(&s, &c, x.re * y.re);
        else {
          volatile double p1 = x.re * y.re, p2 = x.im * y.im, p3 = x.re * y.im, p4 = x.im * y.re;
          neumaier(&s, &c, p1 - p2);
          neumaier(&s2, &c2, p3 + p4);
        }
        ao += as[1];
        bo += bs[0];
      }
      Val r = kind == VK_INT ? mk_int((i128)(int64_t)iacc)
            : kind == VK_FLT ? mk_flt(s + c) : mk_cpx(s + c, s2 + c2);
      if (kind == VK_INT && compute == TPG_UINT64) r = mk_int((i128)iacc);
      store(d->dtype, (uint8_t*)d->base + d->offset + i * ds[0] + j * ds[1], d->big_endian, r,
            &st);
    }
  }
  *status |= st;
  return 0;
}

/* ---------------------------------------------------------------- misc */
int tpo_fill(const tpg_plan* plan, const tpg_operand* d, const void* value, int32_t size) {
  int64_t bases[1] = {d->offset};
  Walk w;
  int64_t total = walk_init(&w, plan, 1, bases);
  for (int64_t i = 0; i < total; ++i) {
    memcpy((uint8_t*)d->base + w.off[0], value, (size_t)size);
    walk_next(&w);
  }
  return 0;
}

int tpo_arange(const tpg_plan* plan, const tpg_operand* d) {
  int64_t bases[1] = {d->offset};
  Walk w;
  uint32_t st = 0;
  int64_t total = walk_init(&w, plan, 1, bases);
  for (int64_t i = 0; i < total; ++i) {
    store(d->dtype, (uint8_t*)d->base + w.off[0], d->big_endian, mk_int(i), &st);
    walk_next(&w);
  }
  return 0;
}

int tpo_byteswap(const tpg_plan* plan, const tpg_operand* d) {
  int64_t bases[1] = {d->offset};
  Walk w;
  int64_t total = walk_init(&w, plan, 1, bases);
  int n = dsize(d->dtype), cs = is_cpx(d->dtype) ? n / 2 : n;
  for (int64_t i = 0; i < total; ++i) {
    uint8_t* p = (uint8_t*)d->base + w.off[0];
    for (int c0 = 0; c0 < n; c0 += cs)
      for (int x = 0; x < cs / 2; ++x) {
        uint8_t t = p[c0 + x];
        p[c0 + x] = p[c0 + cs - 1 - x];
        p[c0 + cs - 1 - x] = t;
      }
    walk_next(&w);
  }
  return 0;
}

/* use n host threads (the reference arm runs with every core the process
   may use, even under torchrun's OMP_NUM_THREADS=1) */
int tpo_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#endif
  (void)n;
  return 0;
}

int tpo_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
