// tpg_reduce.cu — reduction table entry (tpg_reduce) and the empty-range
// case; kernels in tpg_reduce.cuh, instantiated per op family in
// tpg_reduce_sum.cu / tpg_reduce_minmax.cu / tpg_reduce_other.cu.
#include "tpg_reduce.cuh"

namespace tpg {

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

// thread-local request for the fused peer-memory finish, consumed by the
// next reduce launch on this thread (tpg_reduce_sum_p2p)
static thread_local P2pSlot** tl_p2p = nullptr;
static thread_local int tl_p2p_rank = 0, tl_p2p_world = 0;
static thread_local unsigned long long tl_p2p_epoch = 0;
static thread_local int64_t tl_p2p_index_base = 0;

extern "C" int tpg_reduce(tpg_stream stream, int op, double pnorm, const tpg_plan* outer,
                          const tpg_plan* inner, const tpg_operand* d, const tpg_operand* a,
                          int compute, int mode) {
  (void)compute;
  P2pSlot** const want_p2p = tl_p2p;
  tl_p2p = nullptr;
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
  if (want_p2p) {
    // the fused finish lives in the block-granularity row kernel's final
    // block: require exactly the layout that selects it (full reduction of
    // a unit-stride, aligned, native-order f32 / f64 range)
    const int es = dt_size(p.sdt);
    if ((op != TPG_RSUM && op != TPG_RMIN && op != TPG_RMAX &&
         !(op == TPG_RNORM && pnorm == 2.0)) || p.O != 1 || p.ndi != 1 || p.si[0] != es || p.sswap || !p.saligned ||
        (p.sdt != TPG_DOUBLE && p.sdt != TPG_FLOAT) || p.N == 0) {
      set_error("reduce_sum_p2p: source layout not eligible for the fused finish");
      return TPG_E_UNSUPPORTED;
    }
    p.p2p = want_p2p;
    p.p2p_rank = tl_p2p_rank;
    p.p2p_world = tl_p2p_world;
    p.p2p_epoch = tl_p2p_epoch;
    p.p2p_index_base = tl_p2p_index_base;
  }
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
    case TPG_RSUM:
    case TPG_RNORM: return reduce_sum_norm(op, p, st, col, kind);
    case TPG_RMIN:
    case TPG_RMAX: return reduce_minmax(op, p, st, col, kind);
    default: return reduce_other(op, p, st, col, kind);
  }
}

// Full sum of a unit-stride f32 / f64 range with the cross-rank finish fused
// into the reduction kernel (its final block stores the rank's double-double
// partial into every peer's mailbox over NVLink, waits for the world's and
// merges them in rank order): ONE kernel for compute + collective.  The
// peers must be connected (tpg_p2p_connect); `epoch` as tpg_p2p_allreduce.
// Returns TPG_E_UNSUPPORTED (nothing launched) for other layouts.
static int reduce_p2p(tpg_stream stream, int op, const tpg_plan* outer, const tpg_plan* inner,
                      const tpg_operand* d, const tpg_operand* a, unsigned long long epoch,
                      double pnorm = 2.0, int64_t index_base = 0) {
  int rank = 0, world = 0;
  P2pSlot** boxes = p2p_boxes(&rank, &world);
  if (!boxes) return arg_fail("reduce_sum_p2p: peers not connected (tpg_p2p_connect)");
  tl_p2p = boxes;
  tl_p2p_rank = rank;
  tl_p2p_world = world;
  tl_p2p_epoch = epoch;
  tl_p2p_index_base = index_base;
  const int rc = tpg_reduce(stream, op, pnorm, outer, inner, d, a, TPG_DOUBLE, TPG_STANDARD);
  tl_p2p = nullptr;
  return rc;
}

extern "C" int tpg_reduce_sum_p2p(tpg_stream stream, const tpg_plan* outer,
                                  const tpg_plan* inner, const tpg_operand* d,
                                  const tpg_operand* a, unsigned long long epoch) {
  return reduce_p2p(stream, TPG_RSUM, outer, inner, d, a, epoch);
}

// the 2-norm with the same fused finish: ranks exchange sum |x|^2 in
// double-double, the root is taken once on the merged total
extern "C" int tpg_reduce_norm2_p2p(tpg_stream stream, const tpg_plan* outer,
                                    const tpg_plan* inner, const tpg_operand* d,
                                    const tpg_operand* a, unsigned long long epoch) {
  return reduce_p2p(stream, TPG_RNORM, outer, inner, d, a, epoch);
}

// min / max with the fused finish: the reference's rule (NaN iff the
// tensor's first element is NaN, ties keep the earliest) across ranks --
// the rank holding element 0 reduces with first-NaN tracking, the others
// NaN-skipping; partials carry global plan indices (`index_base` = global
// index of this rank's first element) and merge in rank order.
extern "C" int tpg_reduce_minmax_p2p(tpg_stream stream, int op, const tpg_plan* outer,
                                     const tpg_plan* inner, const tpg_operand* d,
                                     const tpg_operand* a, unsigned long long epoch,
                                     int64_t index_base) {
  if (op != TPG_RMIN && op != TPG_RMAX) return arg_fail("reduce_minmax_p2p: op must be min/max");
  return reduce_p2p(stream, op, outer, inner, d, a, epoch, index_base == 0 ? 1.0 : -1.0,
                    index_base);
}
