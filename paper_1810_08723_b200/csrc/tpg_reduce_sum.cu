// tpg_reduce_sum.cu — instantiation of the reduction kernels for TPG_RSUM, TPG_RNORM.
#include "tpg_reduce.cuh"

namespace tpg {

int reduce_sum_norm(int op, RedParams& p, Stream* st, bool col, int kind) {
  if (op == TPG_RSUM) return launch_kind<TPG_RSUM>(p, st, col, kind);
  if (op == TPG_RNORM) return launch_kind<TPG_RNORM>(p, st, col, kind);
  return arg_fail("bad reduce op");
}

}  // namespace tpg
