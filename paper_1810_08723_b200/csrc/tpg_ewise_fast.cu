// tpg_ewise_fast.cu — Tier A: compile-time-typed elementwise kernels for the
// hot (op, dtype) combinations of SURVEY.md §8d (cfg1/cfg2/cfg5) and the
// common same-dtype float ops.  Everything else runs through Tier B.
#include "tpg_ewise.cuh"

namespace tpg {

#define FAST(OC_, NIN_, OP_, K_, D_, A_, B_)                                          \
  if (oc == OC_ && op == OP_ && kind == K_ && p.dt[0] == D_ && (NIN_ < 1 || p.dt[1] == A_) && \
      (NIN_ < 2 || p.dt[2] == B_))                                                     \
    return launch_ew<OC_, NIN_, OP_, K_, D_, A_, B_>(p, st);

int ew_dispatch_fast(int oc, int op, int kind, EwParams& p, Stream* st, bool* done) {
  *done = true;
#define BIN_SAME(OPX)                                                   \
  FAST(OC_BINARY, 2, OPX, K_FLT, TPG_FLOAT, TPG_FLOAT, TPG_FLOAT)       \
  FAST(OC_BINARY, 2, OPX, K_FLT, TPG_DOUBLE, TPG_DOUBLE, TPG_DOUBLE)
  BIN_SAME(TPG_ADD)
  BIN_SAME(TPG_SUBTRACT)
  BIN_SAME(TPG_MULTIPLY)
  BIN_SAME(TPG_DIVIDE)
  BIN_SAME(TPG_MINIMUM)
  BIN_SAME(TPG_MAXIMUM)
#undef BIN_SAME
  FAST(OC_BINARY, 2, TPG_ADD, K_FLT, TPG_HALF, TPG_HALF, TPG_HALF)
  FAST(OC_BINARY, 2, TPG_MULTIPLY, K_FLT, TPG_HALF, TPG_HALF, TPG_HALF)
  FAST(OC_BINARY, 2, TPG_ADD, K_INT, TPG_INT32, TPG_INT32, TPG_INT32)
  FAST(OC_BINARY, 2, TPG_MULTIPLY, K_INT, TPG_INT32, TPG_INT32, TPG_INT32)
  FAST(OC_BINARY, 2, TPG_ADD, K_INT, TPG_INT64, TPG_INT64, TPG_INT64)
  // SURVEY cfg2: int16 view (fused cast-on-load) + float broadcast row
  FAST(OC_BINARY, 2, TPG_ADD, K_FLT, TPG_FLOAT, TPG_INT16, TPG_FLOAT)
  FAST(OC_BINARY, 2, TPG_ADD, K_FLT, TPG_FLOAT, TPG_FLOAT, TPG_INT16)
  // the same shape family from 8-bit data (e.g. uint8 images viewed
  // transposed): 1-byte TMA tiles
  FAST(OC_BINARY, 2, TPG_ADD, K_FLT, TPG_FLOAT, TPG_UINT8, TPG_FLOAT)
  // unary
  FAST(OC_UNARY, 1, TPG_NEGATE, K_FLT, TPG_FLOAT, TPG_FLOAT, -1)
  FAST(OC_UNARY, 1, TPG_NEGATE, K_FLT, TPG_DOUBLE, TPG_DOUBLE, -1)
  FAST(OC_UNARY, 1, TPG_ABSOLUTE, K_FLT, TPG_FLOAT, TPG_FLOAT, -1)
  FAST(OC_UNARY, 1, TPG_ABSOLUTE, K_FLT, TPG_DOUBLE, TPG_DOUBLE, -1)
  FAST(OC_UNARY, 1, TPG_SQRT, K_FLT, TPG_FLOAT, TPG_FLOAT, -1)
  FAST(OC_UNARY, 1, TPG_SQRT, K_FLT, TPG_DOUBLE, TPG_DOUBLE, -1)
  // copy / astype (kind = source value kind)
  FAST(OC_COPY, 1, 0, K_FLT, TPG_FLOAT, TPG_DOUBLE, -1)   // cfg5
  FAST(OC_COPY, 1, 0, K_FLT, TPG_DOUBLE, TPG_FLOAT, -1)
  FAST(OC_COPY, 1, 0, K_INT, TPG_FLOAT, TPG_INT16, -1)    // cfg2 through the table
  FAST(OC_COPY, 1, 0, K_INT, TPG_FLOAT, TPG_UINT8, -1)
  FAST(OC_COPY, 1, 0, K_INT, TPG_HALF, TPG_INT16, -1)     // cfg5
  FAST(OC_COPY, 1, 0, K_FLT, TPG_HALF, TPG_FLOAT, -1)
  FAST(OC_COPY, 1, 0, K_FLT, TPG_FLOAT, TPG_HALF, -1)
  FAST(OC_COPY, 1, 0, K_FLT, TPG_FLOAT, TPG_FLOAT, -1)
  FAST(OC_COPY, 1, 0, K_FLT, TPG_DOUBLE, TPG_DOUBLE, -1)
  FAST(OC_COPY, 1, 0, K_FLT, TPG_HALF, TPG_HALF, -1)
  FAST(OC_COPY, 1, 0, K_INT, TPG_INT16, TPG_INT16, -1)
  FAST(OC_COPY, 1, 0, K_INT, TPG_INT32, TPG_INT32, -1)
  FAST(OC_COPY, 1, 0, K_INT, TPG_INT64, TPG_INT64, -1)
  FAST(OC_COPY, 1, 0, K_INT, TPG_UINT8, TPG_UINT8, -1)
  *done = false;
  return TPG_OK;
}
#undef FAST

}  // namespace tpg
