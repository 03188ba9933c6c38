// tpg_reduce_minmax.cu — instantiation of the reduction kernels for TPG_RMIN, TPG_RMAX.
#include "tpg_reduce.cuh"

namespace tpg {

int reduce_minmax(int op, RedParams& p, Stream* st, bool col, int kind) {
  if (op == TPG_RMIN) return launch_kind<TPG_RMIN>(p, st, col, kind);
  if (op == TPG_RMAX) return launch_kind<TPG_RMAX>(p, st, col, kind);
  return arg_fail("bad reduce op");
}

}  // namespace tpg
