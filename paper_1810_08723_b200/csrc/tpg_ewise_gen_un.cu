// tpg_ewise_gen_un.cu — Tier B (runtime dtype) unary elementwise kernels.
#include "tpg_ewise.cuh"

namespace tpg {

int ew_dispatch_generic_unary(int kind, EwParams& p, Stream* st) {
  switch (kind) {
    case K_INT: return launch_ew<OC_UNARY, 1, -1, K_INT, -1, -1, -1>(p, st);
    case K_UINT: return launch_ew<OC_UNARY, 1, -1, K_UINT, -1, -1, -1>(p, st);
    case K_FLT: return launch_ew<OC_UNARY, 1, -1, K_FLT, -1, -1, -1>(p, st);
    default: return launch_ew<OC_UNARY, 1, -1, K_CPX, -1, -1, -1>(p, st);
  }
}

}  // namespace tpg
