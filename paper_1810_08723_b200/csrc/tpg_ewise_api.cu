// tpg_ewise_api.cu — C-ABI entries of the elementwise engine (binary,
// unary, copy, fill, arange, byteswap, gather, scatter, scatter_fill).
// See tpg_ewise.cuh for the engine and the reference citations.
#include <vector>

#include "tpg_ewise.cuh"

namespace tpg {

// ----------------------------------------------------------- param set-up
static bool valid_dt(int dt) { return dt >= 0 && dt <= TPG_BF16; }

static int setup(EwParams& p, const tpg_plan* plan, const tpg_operand* const* ops, int nin,
                 int mode, Stream* st) {
  memset(&p, 0, sizeof(p));
  if (!plan) return arg_fail("null plan");
  if (plan->ndim < 0 || plan->ndim > TPG_MAX_DIMS) return arg_fail("plan ndim out of range");
  p.nin = nin;
  if (plan->ndim == 0) {
    p.ndim = 1;
    p.ext[0] = 1;
  } else {
    p.ndim = plan->ndim;
    for (int k = 0; k < p.ndim; ++k) {
      if (plan->extent[k] < 0) return arg_fail("negative plan extent");
      p.ext[k] = plan->extent[k];
      for (int v = 0; v <= nin; ++v) p.str[v][k] = plan->stride[v][k];
    }
  }
  for (int v = 0; v <= nin; ++v) {
    const tpg_operand* o = ops[v];
    if (!o) return arg_fail("null operand");
    if (!valid_dt(o->dtype)) return arg_fail("bad dtype code");
    p.dt[v] = o->dtype;
    p.swap[v] = o->big_endian ? 1 : 0;
    if (o->base == nullptr) {
      if (v == 0) return arg_fail("destination needs storage");
      p.isimm[v] = 1;
      p.imm[v] = R16{o->imm[0], o->imm[1]};
      for (int k = 0; k < p.ndim; ++k) p.str[v][k] = 0;
      p.aligned[v] = 1;
    } else {
      p.base[v] = (char*)o->base + o->offset;
      int al = std::min(dt_size(o->dtype), 8);
      bool ok = ((uintptr_t)p.base[v] % al) == 0;
      for (int k = 0; k < p.ndim; ++k)
        if (p.ext[k] > 1 && (p.str[v][k] % al) != 0) ok = false;
      p.aligned[v] = ok;
    }
  }
  p.track = mode == TPG_WARNING || mode == TPG_ERROR;
  p.flags = device_flags(st->device);
  return TPG_OK;
}


static int run(int oc, int op, int kind, EwParams& p, Stream* st, bool allow_fast) {
  p.op = op;
  if (allow_fast) {
    bool done = false;
    int rc = ew_dispatch_fast(oc, op, kind, p, st, &done);
    if (done) return rc;
  }
  switch (oc) {
    case OC_BINARY: return ew_dispatch_generic_binary(kind, p, st);
    case OC_UNARY: return ew_dispatch_generic_unary(kind, p, st);
    case OC_COPY: return ew_dispatch_generic_copy(kind, p, st);
    default: return ew_dispatch_misc(oc, p, st);
  }
}

}  // namespace tpg

using namespace tpg;

static int kind_of(int compute) { return dt_kind(compute); }

extern "C" {

int tpg_binary(tpg_stream stream, int op, const tpg_plan* plan, const tpg_operand* d,
               const tpg_operand* a, const tpg_operand* b, int compute, int mode) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream (tpg_init not called?)");
  if (op < TPG_ADD || op > TPG_MAXIMUM) return arg_fail("bad binary op");
  if (!valid_dt(compute)) return arg_fail("bad compute dtype");
  EwParams p;
  const tpg_operand* ops[3] = {d, a, b};
  int rc = setup(p, plan, ops, 2, mode, st);
  if (rc) return rc;
  p.dry = 0;
  return run(OC_BINARY, op, kind_of(compute), p, st, true);
}

int tpg_unary(tpg_stream stream, int op, const tpg_plan* plan, const tpg_operand* d,
              const tpg_operand* a, int compute, int mode, int force_complex) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream (tpg_init not called?)");
  if (op < TPG_NEGATE || op > TPG_IDENTITY) return arg_fail("bad unary op");
  EwParams p;
  const tpg_operand* ops[3] = {d, a, nullptr};
  int rc = setup(p, plan, ops, 1, mode, st);
  if (rc) return rc;
  if (op == TPG_IDENTITY) return run(OC_COPY, 0, kind_of(a->dtype), p, st, true);
  if (!valid_dt(compute)) return arg_fail("bad compute dtype");
  p.force_complex = force_complex ? 1 : 0;
  return run(OC_UNARY, op, kind_of(compute), p, st, !force_complex);
}

int tpg_copy(tpg_stream stream, const tpg_plan* plan, const tpg_operand* d, const tpg_operand* a,
             int mode) {
  return tpg_unary(stream, TPG_IDENTITY, plan, d, a, a ? a->dtype : 0, mode, 0);
}

// dry-run variants used by the host for error-mode pre-checks: identical
// computation, no stores, flags only.
int tpg_binary_check(tpg_stream stream, int op, const tpg_plan* plan, const tpg_operand* d,
                     const tpg_operand* a, const tpg_operand* b, int compute, int mode) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  EwParams p;
  const tpg_operand* ops[3] = {d, a, b};
  int rc = setup(p, plan, ops, 2, mode, st);
  if (rc) return rc;
  p.dry = 1;
  return run(OC_BINARY, op, kind_of(compute), p, st, false);
}

int tpg_unary_check(tpg_stream stream, int op, const tpg_plan* plan, const tpg_operand* d,
                    const tpg_operand* a, int compute, int mode, int force_complex) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  EwParams p;
  const tpg_operand* ops[3] = {d, a, nullptr};
  int rc = setup(p, plan, ops, 1, mode, st);
  if (rc) return rc;
  p.dry = 1;
  p.force_complex = force_complex ? 1 : 0;
  if (op == TPG_IDENTITY) return run(OC_COPY, 0, kind_of(a->dtype), p, st, false);
  return run(OC_UNARY, op, kind_of(compute), p, st, false);
}

int tpg_fill(tpg_stream stream, const tpg_plan* plan, const tpg_operand* d, const void* value,
             int32_t size) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  if (!d || !value || size != dt_size(d->dtype)) return arg_fail("fill: value size mismatch");
  tpg_operand v{};
  v.base = nullptr;
  v.dtype = d->dtype;
  memcpy(v.imm, value, size);
  EwParams p;
  const tpg_operand* ops[3] = {d, &v, nullptr};
  int rc = setup(p, plan, ops, 1, TPG_STANDARD, st);
  if (rc) return rc;
  p.nin = 0;  // value comes from imm[1]
  p.swap[0] = 0;
  return run(OC_FILL, 0, K_INT, p, st, false);
}

int tpg_arange(tpg_stream stream, const tpg_plan* plan, const tpg_operand* d) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  EwParams p;
  const tpg_operand* ops[3] = {d, nullptr, nullptr};
  int rc = setup(p, plan, ops, 0, TPG_STANDARD, st);
  if (rc) return rc;
  return run(OC_ARANGE, 0, K_INT, p, st, false);
}

int tpg_byteswap(tpg_stream stream, const tpg_plan* plan, const tpg_operand* d) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  EwParams p;
  const tpg_operand* ops[3] = {d, d, nullptr};
  int rc = setup(p, plan, ops, 1, TPG_STANDARD, st);
  if (rc) return rc;
  for (int k = 0; k < p.ndim; ++k) p.str[1][k] = p.str[0][k];
  p.swap[0] = p.swap[1] = 0;
  return run(OC_BSWAP, 0, K_INT, p, st, false);
}

static int raw_dt(int size) {
  switch (size) {
    case 1: return TPG_UINT8;
    case 2: return TPG_UINT16;
    case 4: return TPG_UINT32;
    case 8: return TPG_UINT64;
    case 16: return TPG_CDOUBLE;
    default: return -1;
  }
}

int tpg_gather_plan(tpg_stream stream, const tpg_plan* plan, void* dst_base, int64_t dst_off,
                    const void* src_base, int64_t src_off, int32_t size) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  const int dt = raw_dt(size);
  if (dt < 0) return arg_fail("gather: bad element size");
  tpg_operand d{}, s{};
  d.base = dst_base; d.offset = dst_off; d.dtype = dt;
  s.base = (void*)src_base; s.offset = src_off; s.dtype = dt;
  EwParams p;
  const tpg_operand* ops[3] = {&d, &s, nullptr};
  int rc = setup(p, plan, ops, 1, TPG_STANDARD, st);
  if (rc) return rc;
  return run(OC_RAW, 0, K_INT, p, st, false);
}

}  // extern "C"

// ------------------------------------------------------- pair-list entries
namespace tpg {

__global__ void k_gather_pairs(char* dst, const char* src, const int64_t* pairs, int64_t n,
                               int size) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = pairs[2 * i], s = pairs[2 * i + 1];
    for (int b = 0; b < size; ++b) dst[d + b] = src[s + b];
  }
}

__global__ void k_scatter_pairs(EwParams p, const int64_t* pairs, int64_t n, int kind) {
  uint32_t st = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = pairs[2 * i], s = pairs[2 * i + 1];
    R16 r = load_raw(p.dt[1], p.base[1] + s, p.aligned[1]);
    R16 o;
    switch (kind) {
      case K_INT: o = Ew<OC_COPY, 1, 0, K_INT, -1, -1, -1>::apply(p, r, r, 0, st); break;
      case K_UINT: o = Ew<OC_COPY, 1, 0, K_UINT, -1, -1, -1>::apply(p, r, r, 0, st); break;
      case K_FLT: o = Ew<OC_COPY, 1, 0, K_FLT, -1, -1, -1>::apply(p, r, r, 0, st); break;
      default: o = Ew<OC_COPY, 1, 0, K_CPX, -1, -1, -1>::apply(p, r, r, 0, st); break;
    }
    store_raw(p.dt[0], p.base[0] + d, o, p.aligned[0]);
  }
  if (st) atomicOr(p.flags, st);
}

__global__ void k_scatter_fill(char* dst, const int64_t* offs, int64_t n, R16 v, int size) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = offs[i];
    for (int b = 0; b < size; ++b)
      dst[d + b] = (char)((b < 8 ? v.lo >> (8 * b) : v.hi >> (8 * (b - 8))) & 0xff);
  }
}

static int upload(Stream* st, const int64_t* host, int64_t count, int64_t** dev) {
  const size_t nbytes = (size_t)count * sizeof(int64_t);
  TPG_CUDA_CHECK(cudaMallocAsync((void**)dev, nbytes ? nbytes : 8, st->s));
  if (nbytes) TPG_CUDA_CHECK(cudaMemcpyAsync(*dev, host, nbytes, cudaMemcpyHostToDevice, st->s));
  return TPG_OK;
}

}  // namespace tpg

extern "C" {

int tpg_gather(tpg_stream stream, void* dst_base, const void* src_base, const int64_t* pairs,
               int64_t n, int32_t size) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  if (n <= 0) return TPG_OK;
  int64_t* dp = nullptr;
  int rc = upload(st, pairs, 2 * n, &dp);
  if (rc) return rc;
  const int g = grid_for((n + 255) / 256, st->device, 16);
  k_gather_pairs<<<g, 256, 0, st->s>>>((char*)dst_base, (const char*)src_base, dp, n, size);
  TPG_LAUNCH_CHECK("gather");
  TPG_CUDA_CHECK(cudaFreeAsync(dp, st->s));
  return TPG_OK;
}

int tpg_scatter(tpg_stream stream, const int64_t* pairs, int64_t n, const tpg_operand* d,
                const tpg_operand* s, int mode) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  if (n <= 0) return TPG_OK;
  // duplicates: the last pair for a destination wins (kernels.py:366-369
  // runs in order); keep only the last occurrence so the parallel scatter
  // is deterministic.
  std::vector<int64_t> idx((size_t)n);
  for (int64_t i = 0; i < n; ++i) idx[(size_t)i] = i;
  std::stable_sort(idx.begin(), idx.end(),
                   [&](int64_t x, int64_t y) { return pairs[2 * x] < pairs[2 * y]; });
  std::vector<int64_t> keep;
  keep.reserve((size_t)(2 * n));
  for (size_t i = 0; i < idx.size(); ++i) {
    if (i + 1 < idx.size() && pairs[2 * idx[i]] == pairs[2 * idx[i + 1]]) continue;
    keep.push_back(pairs[2 * idx[i]]);
    keep.push_back(pairs[2 * idx[i] + 1]);
  }
  const int64_t m = (int64_t)keep.size() / 2;
  EwParams p;
  tpg_plan plan{};
  plan.ndim = 0;
  const tpg_operand* ops[3] = {d, s, nullptr};
  int rc = setup(p, &plan, ops, 1, mode, st);
  if (rc) return rc;
  // pair offsets are relative to the storage base, not base+offset
  p.base[0] = (char*)d->base;
  p.base[1] = (char*)s->base;
  int64_t* dp = nullptr;
  rc = upload(st, keep.data(), 2 * m, &dp);
  if (rc) return rc;
  const int g = grid_for((m + 255) / 256, st->device, 16);
  k_scatter_pairs<<<g, 256, 0, st->s>>>(p, dp, m, dt_kind(s->dtype));
  TPG_LAUNCH_CHECK("scatter");
  // make sure the host vector outlives the async copy
  TPG_CUDA_CHECK(cudaStreamSynchronize(st->s));
  TPG_CUDA_CHECK(cudaFreeAsync(dp, st->s));
  return TPG_OK;
}

int tpg_scatter_fill(tpg_stream stream, const int64_t* offsets, int64_t n, void* d_base,
                     const void* value, int32_t size) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  if (n <= 0) return TPG_OK;
  if (size < 1 || size > 16) return arg_fail("scatter_fill: bad size");
  R16 v{0, 0};
  memcpy(&v, value, size);
  int64_t* dp = nullptr;
  int rc = upload(st, offsets, n, &dp);
  if (rc) return rc;
  const int g = grid_for((n + 255) / 256, st->device, 16);
  k_scatter_fill<<<g, 256, 0, st->s>>>((char*)d_base, dp, n, v, size);
  TPG_LAUNCH_CHECK("scatter_fill");
  TPG_CUDA_CHECK(cudaFreeAsync(dp, st->s));
  return TPG_OK;
}

}  // extern "C"
