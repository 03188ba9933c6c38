// tpg_common.cuh — device-side element codec and scalar semantics.
//
// This is the CUDA statement of the reference's numeric contract
// (SURVEY.md Appendix A):
//   * element unpack/pack with per-view byte order: dtypes.codec
//     (pkg/src/tidepool/dtypes.py:357-391) and swap_element (397-401);
//   * the store conversion cast_scalar (dtypes.py:281-325) with _wrap_int
//     (262-267) and _narrow_float (270-278): float->int truncates then wraps
//     modulo 2^n exactly for any magnitude, NaN/inf -> 0, double->half and
//     double->float are single RNE roundings with overflow to +-inf,
//     int64/uint64 -> float go through double first;
//   * the scalar functions of kernels.py: binary_scalar_fn (50-81),
//     _trunc_div (31-33), _float_div (36-41), _complex_div (44-47), and the
//     unary table (121-158).
// Values live in one of four compute domains that mirror the Python value
// kinds the reference computes with: int (Python int, exact; kept modulo
// 2^64 which is exact after the final wrap), uint (uint64 operands), float
// (Python float = IEEE double) and complex (Python complex = 2 doubles).
#pragma once
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/tidepool_gpu.h"

namespace tpg {

enum Kind { K_INT = 0, K_UINT = 1, K_FLT = 2, K_CPX = 3 };

struct R16 {
  uint64_t lo, hi;
};

__host__ __device__ constexpr int dt_size(int dt) {
  return dt == TPG_BOOL || dt == TPG_INT8 || dt == TPG_UINT8 ? 1
       : dt == TPG_INT16 || dt == TPG_UINT16 || dt == TPG_HALF || dt == TPG_BF16 ? 2
       : dt == TPG_INT32 || dt == TPG_UINT32 || dt == TPG_FLOAT || dt == TPG_CHALF ? 4
       : dt == TPG_CDOUBLE ? 16 : 8;
}
__host__ __device__ constexpr bool dt_is_complex(int dt) {
  return dt == TPG_CHALF || dt == TPG_CFLOAT || dt == TPG_CDOUBLE;
}
__host__ __device__ constexpr bool dt_is_float(int dt) {
  return dt == TPG_HALF || dt == TPG_FLOAT || dt == TPG_DOUBLE || dt == TPG_BF16 ||
         dt_is_complex(dt);
}
__host__ __device__ constexpr int dt_kind(int dt) {
  return dt_is_complex(dt) ? K_CPX : dt_is_float(dt) ? K_FLT : dt == TPG_UINT64 ? K_UINT : K_INT;
}
// component size for byte swapping (swap_element works per complex component)
__host__ __device__ constexpr int dt_comp(int dt) {
  return dt_is_complex(dt) ? dt_size(dt) / 2 : dt_size(dt);
}

// ------------------------------------------------------------------ bytes
__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }
__device__ __forceinline__ uint16_t bswap16(uint16_t x) {
  return (uint16_t)__byte_perm((uint32_t)x, 0, 0x3201);
}
__device__ __forceinline__ uint64_t bswap64(uint64_t x) {
  uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  return ((uint64_t)bswap32(lo) << 32) | bswap32(hi);
}

// Reverse the byte order of one element per component (dtypes.swap_element).
__device__ __forceinline__ R16 swap_raw(int dt, R16 r) {
  switch (dt_comp(dt)) {
    case 1: return r;
    case 2: {
      if (dt_is_complex(dt)) {
        uint32_t v = (uint32_t)r.lo;
        r.lo = (uint64_t)__byte_perm(v, 0, 0x2301);
      } else {
        r.lo = bswap16((uint16_t)r.lo);
      }
      return r;
    }
    case 4: {
      if (dt_is_complex(dt)) {
        uint32_t re = (uint32_t)r.lo, im = (uint32_t)(r.lo >> 32);
        r.lo = ((uint64_t)bswap32(im) << 32) | bswap32(re);
      } else {
        r.lo = bswap32((uint32_t)r.lo);
      }
      return r;
    }
    default:
      r.lo = bswap64(r.lo);
      if (dt_is_complex(dt)) r.hi = bswap64(r.hi);
      return r;
  }
}

// Raw element load; `aligned` false falls back to byte loads (views whose
// offset or strides are not multiples of the element size are legal in the
// reference: tensors.py:84-99 accepts any byte strides).
__device__ __forceinline__ R16 load_raw(int dt, const char* p, bool aligned) {
  R16 r{0, 0};
  const int s = dt_size(dt);
  if (aligned) {
    switch (s) {
      case 1: r.lo = *(const uint8_t*)p; break;
      case 2: r.lo = *(const uint16_t*)p; break;
      case 4: r.lo = *(const uint32_t*)p; break;
      case 8: r.lo = *(const uint64_t*)p; break;
      default: {
        const uint64_t* q = (const uint64_t*)p;
        r.lo = q[0];
        r.hi = q[1];
      }
    }
  } else {
    for (int i = 0; i < s; ++i) {
      uint64_t b = (uint8_t)p[i];
      if (i < 8) r.lo |= b << (8 * i);
      else r.hi |= b << (8 * (i - 8));
    }
  }
  return r;
}

__device__ __forceinline__ void store_raw(int dt, char* p, R16 r, bool aligned) {
  const int s = dt_size(dt);
  if (aligned) {
    switch (s) {
      case 1: *(uint8_t*)p = (uint8_t)r.lo; break;
      case 2: *(uint16_t*)p = (uint16_t)r.lo; break;
      case 4: *(uint32_t*)p = (uint32_t)r.lo; break;
      case 8: *(uint64_t*)p = r.lo; break;
      default: {
        uint64_t* q = (uint64_t*)p;
        q[0] = r.lo;
        q[1] = r.hi;
      }
    }
  } else {
    for (int i = 0; i < s; ++i) p[i] = (char)((i < 8 ? r.lo >> (8 * i) : r.hi >> (8 * (i - 8))) & 0xff);
  }
}

// ------------------------------------------------------------------ decode
__device__ __forceinline__ double half_bits_to_double(uint16_t h) {
  return (double)__half2float(__ushort_as_half(h));
}
__device__ __forceinline__ double bf16_bits_to_double(uint16_t h) {
  return (double)__uint_as_float(((uint32_t)h) << 16);
}

// Python int value of an integer/bool element (struct '?bBhHiIqQ').
__device__ __forceinline__ int64_t dec_int(int dt, R16 r) {
  switch (dt) {
    case TPG_BOOL: return (r.lo & 0xff) != 0;
    case TPG_INT8: return (int8_t)r.lo;
    case TPG_UINT8: return (uint8_t)r.lo;
    case TPG_INT16: return (int16_t)r.lo;
    case TPG_UINT16: return (uint16_t)r.lo;
    case TPG_INT32: return (int32_t)r.lo;
    case TPG_UINT32: return (uint32_t)r.lo;
    default: return (int64_t)r.lo;  // INT64 / UINT64 bits
  }
}

// Python float value (for a real float element) or float(int) for ints:
// int -> float conversion is RNE to double (Python float(int)).
__device__ __forceinline__ double dec_flt(int dt, R16 r) {
  switch (dt) {
    case TPG_HALF: return half_bits_to_double((uint16_t)r.lo);
    case TPG_BF16: return bf16_bits_to_double((uint16_t)r.lo);
    case TPG_FLOAT: return (double)__uint_as_float((uint32_t)r.lo);
    case TPG_DOUBLE: return __longlong_as_double((long long)r.lo);
    case TPG_UINT64: return __ull2double_rn(r.lo);
    case TPG_INT64: return __ll2double_rn((long long)r.lo);
    case TPG_CHALF: return half_bits_to_double((uint16_t)r.lo);
    case TPG_CFLOAT: return (double)__uint_as_float((uint32_t)r.lo);
    case TPG_CDOUBLE: return __longlong_as_double((long long)r.lo);
    default: return (double)dec_int(dt, r);  // exact for <= 32-bit ints
  }
}

__device__ __forceinline__ double2 dec_cpx(int dt, R16 r) {
  switch (dt) {
    case TPG_CHALF:
      return make_double2(half_bits_to_double((uint16_t)r.lo),
                          half_bits_to_double((uint16_t)(r.lo >> 16)));
    case TPG_CFLOAT:
      return make_double2((double)__uint_as_float((uint32_t)r.lo),
                          (double)__uint_as_float((uint32_t)(r.lo >> 32)));
    case TPG_CDOUBLE:
      return make_double2(__longlong_as_double((long long)r.lo),
                          __longlong_as_double((long long)r.hi));
    default: return make_double2(dec_flt(dt, r), 0.0);
  }
}

// ------------------------------------------------------------------ encode
__device__ __forceinline__ uint16_t dbl_to_half_bits(double d) {
  unsigned short h;
  asm("cvt.rn.f16.f64 %0, %1;" : "=h"(h) : "d"(d));
  return h;
}
__device__ __forceinline__ uint16_t dbl_to_bf16_bits(double d) {
  // double -> bf16 in one RNE rounding: round to float with round-to-odd
  // first (exact for the final RNE step), then RNE to bf16.
  float f;
  asm("cvt.rz.f32.f64 %0, %1;" : "=f"(f) : "d"(d));
  uint32_t u = __float_as_uint(f);
  if ((double)f != d && !isnan(d) && !isinf(f)) u |= 1u;  // sticky bit
  if (isnan(d)) return 0x7fc0;
  unsigned short h;
  asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(h) : "f"(__uint_as_float(u)));
  return h;
}

// _narrow_float: RNE to the target real type, overflow -> +-inf.
__device__ __forceinline__ uint64_t narrow_bits(int real_dt, double d) {
  switch (real_dt) {
    case TPG_HALF: return dbl_to_half_bits(d);
    case TPG_BF16: return dbl_to_bf16_bits(d);
    case TPG_FLOAT: return __float_as_uint(__double2float_rn(d));
    default: return (uint64_t)__double_as_longlong(d);
  }
}

__device__ __forceinline__ int real_of(int dt) {
  return dt == TPG_CHALF ? TPG_HALF : dt == TPG_CFLOAT ? TPG_FLOAT : dt == TPG_CDOUBLE ? TPG_DOUBLE : dt;
}

__device__ __forceinline__ R16 enc_cpx_parts(int dt, double re, double im) {
  R16 r{0, 0};
  switch (dt) {
    case TPG_CHALF: r.lo = narrow_bits(TPG_HALF, re) | (narrow_bits(TPG_HALF, im) << 16); break;
    case TPG_CFLOAT: r.lo = narrow_bits(TPG_FLOAT, re) | (narrow_bits(TPG_FLOAT, im) << 32); break;
    default:
      r.lo = (uint64_t)__double_as_longlong(re);
      r.hi = (uint64_t)__double_as_longlong(im);
  }
  return r;
}

// integer range of a dtype (for the CastContext "out of range" diagnostic)
__device__ __forceinline__ bool int_in_range(int dt, int64_t v, bool uns) {
  if (uns) {
    uint64_t u = (uint64_t)v;
    switch (dt) {
      case TPG_INT8: return u <= 127u;
      case TPG_UINT8: return u <= 255u;
      case TPG_INT16: return u <= 32767u;
      case TPG_UINT16: return u <= 65535u;
      case TPG_INT32: return u <= 2147483647u;
      case TPG_UINT32: return u <= 4294967295u;
      case TPG_INT64: return u <= 9223372036854775807ull;
      default: return true;
    }
  }
  switch (dt) {
    case TPG_INT8: return v >= -128 && v <= 127;
    case TPG_UINT8: return v >= 0 && v <= 255;
    case TPG_INT16: return v >= -32768 && v <= 32767;
    case TPG_UINT16: return v >= 0 && v <= 65535;
    case TPG_INT32: return v >= -2147483648ll && v <= 2147483647ll;
    case TPG_UINT32: return v >= 0 && v <= 4294967295ll;
    case TPG_UINT64: return v >= 0;
    default: return true;
  }
}

// low bits of a two's-complement value for an integer dtype (_wrap_int)
__device__ __forceinline__ uint64_t wrap_bits(int dt, uint64_t v) {
  switch (dt_size(dt)) {
    case 1: return v & 0xffull;
    case 2: return v & 0xffffull;
    case 4: return v & 0xffffffffull;
    default: return v;
  }
}

// store from a Python int value (int64 domain, or uint64 when uns)
__device__ __forceinline__ R16 enc_from_int(int dt, int64_t v, bool uns, uint32_t* fl) {
  R16 r{0, 0};
  if (dt == TPG_BOOL) {
    r.lo = v != 0;
    return r;
  }
  if (dt_is_float(dt)) {
    double d = uns ? __ull2double_rn((uint64_t)v) : __ll2double_rn(v);
    if (dt_is_complex(dt)) return enc_cpx_parts(dt, d, 0.0);
    r.lo = narrow_bits(dt, d);
    return r;
  }
  if (fl && !int_in_range(dt, v, uns)) *fl |= TPG_FLAG_CAST_LOSS;
  r.lo = wrap_bits(dt, (uint64_t)v);
  return r;
}

// float -> integer: truncate toward zero, wrap modulo 2^n exactly for any
// magnitude (dtypes.py:317-325); NaN/inf -> 0 with a domain-loss diagnostic.
__device__ __forceinline__ uint64_t f2i_wrap(double d, int dt, uint32_t* fl) {
  if (isnan(d) || isinf(d)) {
    if (fl) *fl |= TPG_FLAG_CAST_LOSS;
    return 0;
  }
  const double t = trunc(d);
  if (fl) {
    bool ok;
    switch (dt) {
      case TPG_INT8: ok = t >= -128.0 && t <= 127.0; break;
      case TPG_UINT8: ok = t >= 0.0 && t <= 255.0; break;
      case TPG_INT16: ok = t >= -32768.0 && t <= 32767.0; break;
      case TPG_UINT16: ok = t >= 0.0 && t <= 65535.0; break;
      case TPG_INT32: ok = t >= -2147483648.0 && t <= 2147483647.0; break;
      case TPG_UINT32: ok = t >= 0.0 && t <= 4294967295.0; break;
      case TPG_INT64: ok = t >= -9223372036854775808.0 && t < 9223372036854775808.0; break;
      default: ok = t >= 0.0 && t < 18446744073709551616.0; break;
    }
    if (!ok) *fl |= TPG_FLAG_CAST_LOSS;
  }
  uint64_t bits;
  if (fabs(t) < 9223372036854775808.0) {
    bits = (uint64_t)(int64_t)t;
  } else {
    double r = fmod(t, 18446744073709551616.0);  // exact, |r| < 2^64
    if (r < 0.0) r += 18446744073709551616.0;     // exact (r is a multiple of 2^11)
    bits = r >= 9223372036854775808.0 ? (uint64_t)r : (uint64_t)(int64_t)r;
  }
  return wrap_bits(dt, bits);
}

// store from a Python float value
__device__ __forceinline__ R16 enc_from_flt(int dt, double d, uint32_t* fl) {
  R16 r{0, 0};
  if (dt == TPG_BOOL) {
    r.lo = d != 0.0;  // NaN -> True
    return r;
  }
  if (dt_is_complex(dt)) return enc_cpx_parts(dt, d, 0.0);
  if (dt_is_float(dt)) {
    r.lo = narrow_bits(dt, d);
    return r;
  }
  r.lo = f2i_wrap(d, dt, fl);
  return r;
}

// store from a Python complex value
__device__ __forceinline__ R16 enc_from_cpx(int dt, double re, double im, uint32_t* fl) {
  if (dt_is_complex(dt)) return enc_cpx_parts(dt, re, im);
  if (fl && im != 0.0) *fl |= TPG_FLAG_CAST_LOSS;  // discarding nonzero imag
  return enc_from_flt(dt, re, fl);
}

// ------------------------------------------------------------ binary ops
// kernels.binary_scalar_fn (kernels.py:50-81) in each compute domain.
__device__ __forceinline__ double float_div(double a, double b) {  // _float_div
  if (b == 0.0) {
    if (a == 0.0 || isnan(a)) return __longlong_as_double(0x7ff8000000000000ll);
    return copysign(INFINITY, a) * copysign(1.0, b);
  }
  return __ddiv_rn(a, b);
}

// CPython complex division (Objects/complexobject.c _Py_c_quot, Smith's
// algorithm); b == 0 is intercepted as NaN+NaNj by kernels._complex_div.
__device__ __forceinline__ double2 complex_div(double2 a, double2 b) {
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  if (b.x == 0.0 && b.y == 0.0) return make_double2(nan, nan);
  const double abr = fabs(b.x), abi = fabs(b.y);
  if (abr >= abi) {
    const double ratio = __ddiv_rn(b.y, b.x);
    const double denom = __dadd_rn(b.x, __dmul_rn(b.y, ratio));
    return make_double2(__ddiv_rn(__dadd_rn(a.x, __dmul_rn(a.y, ratio)), denom),
                        __ddiv_rn(__dsub_rn(a.y, __dmul_rn(a.x, ratio)), denom));
  } else if (abi >= abr) {
    const double ratio = __ddiv_rn(b.x, b.y);
    const double denom = __dadd_rn(__dmul_rn(b.x, ratio), b.y);
    return make_double2(__ddiv_rn(__dadd_rn(__dmul_rn(a.x, ratio), a.y), denom),
                        __ddiv_rn(__dsub_rn(__dmul_rn(a.y, ratio), a.x), denom));
  }
  return make_double2(nan, nan);
}

// Python tuple comparison (a.real, a.imag) <= (b.real, b.imag)
__device__ __forceinline__ bool cpx_le(double2 a, double2 b) {
  if (a.x != b.x) return a.x < b.x;  // NaN != NaN: falls to '<' (False)
  return a.y <= b.y;
}
__device__ __forceinline__ bool cpx_ge(double2 a, double2 b) {
  if (a.x != b.x) return a.x > b.x;
  return a.y >= b.y;
}
__device__ __forceinline__ bool cpx_lt(double2 a, double2 b) {
  if (a.x != b.x) return a.x < b.x;
  return a.y < b.y;
}
__device__ __forceinline__ bool cpx_gt(double2 a, double2 b) {
  if (a.x != b.x) return a.x > b.x;
  return a.y > b.y;
}

__device__ __forceinline__ double bin_flt(int op, double a, double b) {
  switch (op) {
    case TPG_ADD: return __dadd_rn(a, b);
    case TPG_SUBTRACT: return __dsub_rn(a, b);
    case TPG_MULTIPLY: return __dmul_rn(a, b);
    case TPG_DIVIDE: return float_div(a, b);
    case TPG_MINIMUM: return a <= b ? a : b;
    default: return a >= b ? a : b;
  }
}

__device__ __forceinline__ double2 bin_cpx(int op, double2 a, double2 b) {
  switch (op) {
    case TPG_ADD: return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
    case TPG_SUBTRACT: return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
    case TPG_MULTIPLY:
      return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                          __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
    case TPG_DIVIDE: return complex_div(a, b);
    case TPG_MINIMUM: return cpx_le(a, b) ? a : b;
    default: return cpx_ge(a, b) ? a : b;
  }
}

// integer domain: exact Python ints kept modulo 2^64 (exact after _wrap_int);
// min/max/divide compare true values, so uint64 operands use the U domain.
__device__ __forceinline__ int64_t bin_int(int op, int64_t a, int64_t b, uint32_t* status) {
  switch (op) {
    case TPG_ADD: return (int64_t)((uint64_t)a + (uint64_t)b);
    case TPG_SUBTRACT: return (int64_t)((uint64_t)a - (uint64_t)b);
    case TPG_MULTIPLY: return (int64_t)((uint64_t)a * (uint64_t)b);
    case TPG_DIVIDE:
      if (b == 0) {
        *status |= TPG_FLAG_INT_DIV0;
        return 0;
      }
      if (b == -1) return (int64_t)(0ull - (uint64_t)a);  // INT64_MIN / -1 wraps
      return a / b;                                        // C truncates toward zero
    case TPG_MINIMUM: return a <= b ? a : b;
    default: return a >= b ? a : b;
  }
}
__device__ __forceinline__ uint64_t bin_uint(int op, uint64_t a, uint64_t b, uint32_t* status) {
  switch (op) {
    case TPG_ADD: return a + b;
    case TPG_SUBTRACT: return a - b;
    case TPG_MULTIPLY: return a * b;
    case TPG_DIVIDE:
      if (b == 0) {
        *status |= TPG_FLAG_INT_DIV0;
        return 0;
      }
      return a / b;
    case TPG_MINIMUM: return a <= b ? a : b;
    default: return a >= b ? a : b;
  }
}

}  // namespace tpg
