// tpg_chain.cu — fused elementwise chains (cfg5's
// Z = add(multiply(Y, 1.5f), -2.0f)).
//
// A chain applies n binary steps `x = op_i(x, s_i)` (or `op_i(s_i, x)`) with
// by-value scalars s_i to one tensor in ONE pass over memory.  Every step
// has exactly the reference's per-op semantics (kernels.binary_elementwise
// via binary_scalar_fn, kernels.py:50-81, 213-248): operands decoded to the
// step's compute domain (widen_for_compute of the step's result dtype,
// dtypes.py:190-196), the op evaluated there, and the value rounded ONCE to
// the step's result dtype by the store conversion (cast_scalar,
// dtypes.py:281-325) — which is exactly what materialising each
// intermediate tensor would do, so the chain is bit-identical to running
// the ops one after another, while moving 8 instead of 16 B per element
// for a 2-step f32 chain.
#include "tpg_ewise.cuh"

namespace tpg {

constexpr int MAX_STEPS = 8;

struct ChainStep {
  int op, dt, kind, sfirst, sdt;
  R16 s;
};

struct ChainParams {
  EwParams ew;  // views: 0 dest, 1 source
  int n;
  ChainStep step[MAX_STEPS];
};

// all-float fast chain: f32 source / steps / dest, native byte order.
// The scalars are decoded once per thread into registers (FScal); NS
// steps are unrolled at compile time (NS = 0: runtime count, up to 8).
struct FScal {
  double w[MAX_STEPS];
  float wf[MAX_STEPS];
  int op[MAX_STEPS], sf[MAX_STEPS], ex[MAX_STEPS];
};
__device__ __forceinline__ FScal chain_scalars(const ChainParams& c) {
  FScal f;
#pragma unroll
  for (int i = 0; i < MAX_STEPS; ++i) {
    f.w[i] = i < c.n ? dec_flt(c.step[i].sdt, c.step[i].s) : 0.0;
    f.wf[i] = (float)f.w[i];
    f.ex[i] = (double)f.wf[i] == f.w[i];
    f.op[i] = c.step[i].op;
    f.sf[i] = c.step[i].sfirst;
  }
  return f;
}
__device__ __forceinline__ float rnd_f32(double r, uint32_t* fl) {
  return __uint_as_float((uint32_t)enc_from_flt(TPG_FLOAT, r, fl).lo);
}
// apply the chain to V values: the (warp-uniform) op switch runs once per
// step, each case is a tight loop over the V values.
// + - * with a scalar that is exactly a float run in float arithmetic: for
// float operands, rounding the exact result to double and then to float
// equals rounding it to float once (double has >= 2*24+2 significand bits,
// so the double rounding is innocuous for + - * /), which is what the
// reference's compute-in-double-then-narrow store does (ops.py:145-152,
// dtypes.py:270-278) -- and it keeps the f32<->f64 conversions (the
// 16/clk XU pipe, 67% busy on the double path) off the chain
template <int NS, int V>
__device__ __forceinline__ void chain_f32(const FScal& f, int n, float (&x)[V], uint32_t* fl) {
  constexpr int M = NS ? NS : MAX_STEPS;
#pragma unroll
  for (int i = 0; i < M; ++i) {
    if (NS == 0 && i >= n) break;
    const double w = f.w[i];
    const bool sf = f.sf[i];
    if (f.ex[i]) {
      const float wf = f.wf[i];
      const int op = f.op[i];
      if (op == TPG_ADD) {
#pragma unroll
        for (int e = 0; e < V; ++e) x[e] = __fadd_rn(x[e], wf);
        continue;
      }
      if (op == TPG_MULTIPLY) {
#pragma unroll
        for (int e = 0; e < V; ++e) x[e] = __fmul_rn(x[e], wf);
        continue;
      }
      if (op == TPG_SUBTRACT) {
#pragma unroll
        for (int e = 0; e < V; ++e) x[e] = sf ? __fsub_rn(wf, x[e]) : __fsub_rn(x[e], wf);
        continue;
      }
    }
    switch (f.op[i]) {
      case TPG_ADD:
#pragma unroll
        for (int e = 0; e < V; ++e) x[e] = rnd_f32(__dadd_rn((double)x[e], w), fl);
        break;
      case TPG_MULTIPLY:
#pragma unroll
        for (int e = 0; e < V; ++e) x[e] = rnd_f32(__dmul_rn((double)x[e], w), fl);
        break;
      case TPG_SUBTRACT:
#pragma unroll
        for (int e = 0; e < V; ++e)
          x[e] = rnd_f32(sf ? __dsub_rn(w, (double)x[e]) : __dsub_rn((double)x[e], w), fl);
        break;
      default:
#pragma unroll 1
        for (int e = 0; e < V; ++e) {
          const double v = (double)x[e];
          x[e] = rnd_f32(sf ? bin_flt(f.op[i], w, v) : bin_flt(f.op[i], v, w), fl);
        }
        break;
    }
  }
}

template <int KIND>
__device__ __forceinline__ R16 chain_step_gen(const EwDesc& e, R16 a, R16 b, uint32_t& st) {
  R16S r = ew_body_gen<OC_BINARY, KIND>(e, a, b, 0);
  st |= r.st;
  return r.r;
}

__device__ R16 chain_any(const ChainParams& c, R16 x, uint32_t& st) {
  int cur = c.ew.dt[1], sw = c.ew.swap[1];
#pragma unroll 1
  for (int i = 0; i < c.n; ++i) {
    const ChainStep& s = c.step[i];
    EwDesc e;
    e.dtd = s.dt;
    e.sd = (i == c.n - 1) ? c.ew.swap[0] : 0;
    e.op = s.op;
    e.track = c.ew.track;
    e.fc = 0;
    R16 a = x, b = s.s;
    e.dta = cur; e.sa = sw; e.dtb = s.sdt; e.sb = 0;
    if (s.sfirst) {
      a = s.s; b = x;
      e.dta = s.sdt; e.sa = 0; e.dtb = cur; e.sb = sw;
    }
    switch (s.kind) {
      case K_INT: x = chain_step_gen<K_INT>(e, a, b, st); break;
      case K_UINT: x = chain_step_gen<K_UINT>(e, a, b, st); break;
      case K_FLT: x = chain_step_gen<K_FLT>(e, a, b, st); break;
      default: x = chain_step_gen<K_CPX>(e, a, b, st); break;
    }
    cur = s.dt;
    sw = 0;
  }
  return x;
}

// contiguous f32 -> f32: 16-B loads/stores, 8 elements per thread per step
template <int NS>
__global__ void __launch_bounds__(256) k_chain_f32(ChainParams c, int64_t n) {
  uint32_t st = 0;
  uint32_t* fl = c.ew.track ? &st : nullptr;
  const FScal f = chain_scalars(c);
  const int ns = c.n;
  const float* __restrict__ src = (const float*)c.ew.base[1];
  float* __restrict__ dst = (float*)c.ew.base[0];
  const int64_t nv = n / 8;
  const int64_t tid = (int64_t)blockIdx.x * 256 + threadIdx.x, nt = (int64_t)gridDim.x * 256;
  for (int64_t v = tid; v < nv; v += nt) {
    float4 a = __ldcs((const float4*)src + 2 * v);
    float4 b = __ldcs((const float4*)src + 2 * v + 1);
    float x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    chain_f32<NS, 8>(f, ns, x, fl);
    a = make_float4(x[0], x[1], x[2], x[3]);
    b = make_float4(x[4], x[5], x[6], x[7]);
    if (!c.ew.dry) {
      __stcs((float4*)dst + 2 * v, a);
      __stcs((float4*)dst + 2 * v + 1, b);
    }
  }
  for (int64_t i = nv * 8 + tid; i < n; i += nt) {
    float x[1] = {src[i]};
    chain_f32<NS, 1>(f, ns, x, fl);
    if (!c.ew.dry) dst[i] = x[0];
  }
  if (st) atomicOr(c.ew.flags, st);
}

// any plan / dtype: per-element index decomposition
__global__ void __launch_bounds__(256) k_chain_any(ChainParams c, int64_t total) {
  uint32_t st = 0;
  const EwParams& p = c.ew;
  const int64_t nt = (int64_t)gridDim.x * 256;
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < total; i += nt) {
    int64_t r = i, d = 0, a = 0;
    for (int k = 0; k < p.ndim; ++k) {
      const int64_t e = p.ext[k];
      const int64_t q = r % e;
      r /= e;
      d += q * p.str[0][k];
      a += q * p.str[1][k];
    }
    const R16 x = load_raw(p.dt[1], p.base[1] + a, p.aligned[1]);
    const R16 o = chain_any(c, x, st);
    if (!p.dry) store_raw(p.dt[0], p.base[0] + d, o, p.aligned[0]);
  }
  if (st) atomicOr(p.flags, st);
}

}  // namespace tpg

using namespace tpg;

static int tpg_chain_impl(tpg_stream stream, const tpg_plan* plan, const tpg_operand* d,
                              const tpg_operand* a, int nsteps, const tpg_chain_step* steps,
                              int mode, int dry) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  if (!plan || !d || !a || !steps || !d->base || !a->base) return arg_fail("chain: null argument");
  if (nsteps < 1 || nsteps > MAX_STEPS) return arg_fail("chain: 1..8 steps");
  if (plan->ndim < 0 || plan->ndim > TPG_MAX_DIMS) return arg_fail("chain: bad plan");
  ChainParams c;
  memset(&c, 0, sizeof(c));
  EwParams& p = c.ew;
  p.nin = 1;
  p.ndim = plan->ndim ? plan->ndim : 1;
  int64_t total = 1;
  for (int k = 0; k < p.ndim; ++k) {
    p.ext[k] = plan->ndim ? plan->extent[k] : 1;
    if (p.ext[k] < 0) return arg_fail("chain: negative extent");
    total *= p.ext[k];
    for (int v = 0; v < 2; ++v) p.str[v][k] = plan->ndim ? plan->stride[v][k] : 0;
  }
  const tpg_operand* ops[2] = {d, a};
  for (int v = 0; v < 2; ++v) {
    if (ops[v]->dtype < 0 || ops[v]->dtype > TPG_BF16) return arg_fail("chain: bad dtype");
    p.dt[v] = ops[v]->dtype;
    p.swap[v] = ops[v]->big_endian ? 1 : 0;
    p.base[v] = (char*)ops[v]->base + ops[v]->offset;
    const int al = std::min(dt_size(p.dt[v]), 8);
    bool ok = ((uintptr_t)p.base[v] % al) == 0;
    for (int k = 0; k < p.ndim; ++k)
      if (p.ext[k] > 1 && p.str[v][k] % al) ok = false;
    p.aligned[v] = ok;
  }
  p.track = mode == TPG_WARNING || mode == TPG_ERROR;
  p.dry = dry;
  p.flags = device_flags(st->device);
  c.n = nsteps;
  bool all_f32 = p.dt[0] == TPG_FLOAT && p.dt[1] == TPG_FLOAT && !p.swap[0] && !p.swap[1];
  for (int i = 0; i < nsteps; ++i) {
    const tpg_chain_step& s = steps[i];
    if (s.op < TPG_ADD || s.op > TPG_MAXIMUM) return arg_fail("chain: bad op");
    if (s.dtype < 0 || s.dtype > TPG_BF16 || s.compute < 0 || s.compute > TPG_BF16 ||
        s.scalar_dtype < 0 || s.scalar_dtype > TPG_BF16)
      return arg_fail("chain: bad step dtype");
    c.step[i].op = s.op;
    c.step[i].dt = s.dtype;
    c.step[i].kind = dt_kind(s.compute);
    c.step[i].sfirst = s.scalar_first ? 1 : 0;
    c.step[i].sdt = s.scalar_dtype;
    memcpy(&c.step[i].s, s.scalar, 16);
    if (s.dtype != TPG_FLOAT || dt_kind(s.compute) != K_FLT || dt_is_complex(s.scalar_dtype))
      all_f32 = false;
  }
  if (steps[nsteps - 1].dtype != p.dt[0]) return arg_fail("chain: last step dtype != dest dtype");
  if (total == 0) return TPG_OK;
  const int64_t cap = (int64_t)sm_count(st->device) * 8;
  if (all_f32 && p.ndim == 1 && p.str[0][0] == 4 && p.str[1][0] == 4 &&
      (uintptr_t)p.base[0] % 16 == 0 && (uintptr_t)p.base[1] % 16 == 0) {
    const int64_t g = std::max<int64_t>(1, std::min<int64_t>((total / 8 + 255) / 256, cap));
    switch (nsteps) {
      case 1: k_chain_f32<1><<<(int)g, 256, 0, st->s>>>(c, total); break;
      case 2: k_chain_f32<2><<<(int)g, 256, 0, st->s>>>(c, total); break;
      case 3: k_chain_f32<3><<<(int)g, 256, 0, st->s>>>(c, total); break;
      default: k_chain_f32<0><<<(int)g, 256, 0, st->s>>>(c, total); break;
    }
  } else {
    const int64_t g = std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, cap));
    k_chain_any<<<(int)g, 256, 0, st->s>>>(c, total);
  }
  TPG_LAUNCH_CHECK("chain");
  return TPG_OK;
}

extern "C" {
int tpg_chain(tpg_stream stream, const tpg_plan* plan, const tpg_operand* d, const tpg_operand* a,
              int nsteps, const tpg_chain_step* steps, int mode) {
  return tpg_chain_impl(stream, plan, d, a, nsteps, steps, mode, 0);
}
int tpg_chain_check(tpg_stream stream, const tpg_plan* plan, const tpg_operand* d,
                    const tpg_operand* a, int nsteps, const tpg_chain_step* steps, int mode) {
  return tpg_chain_impl(stream, plan, d, a, nsteps, steps, mode, 1);
}
}
