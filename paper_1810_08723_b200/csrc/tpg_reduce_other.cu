// tpg_reduce_other.cu — instantiation of the reduction kernels for TPG_RPRODUCT, TPG_RANY, TPG_RALL.
#include "tpg_reduce.cuh"

namespace tpg {

int reduce_other(int op, RedParams& p, Stream* st, bool col, int kind) {
  if (op == TPG_RPRODUCT) return launch_kind<TPG_RPRODUCT>(p, st, col, kind);
  if (op == TPG_RANY) return launch_kind<TPG_RANY>(p, st, col, kind);
  if (op == TPG_RALL) return launch_kind<TPG_RALL>(p, st, col, kind);
  return arg_fail("bad reduce op");
}

}  // namespace tpg
