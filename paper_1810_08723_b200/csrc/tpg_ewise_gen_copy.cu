// tpg_ewise_gen_copy.cu — Tier B (runtime dtype) copy/astype kernels.
#include "tpg_ewise.cuh"

namespace tpg {

int ew_dispatch_generic_copy(int kind, EwParams& p, Stream* st) {
  switch (kind) {
    case K_INT: return launch_ew<OC_COPY, 1, -1, K_INT, -1, -1, -1>(p, st);
    case K_UINT: return launch_ew<OC_COPY, 1, -1, K_UINT, -1, -1, -1>(p, st);
    case K_FLT: return launch_ew<OC_COPY, 1, -1, K_FLT, -1, -1, -1>(p, st);
    default: return launch_ew<OC_COPY, 1, -1, K_CPX, -1, -1, -1>(p, st);
  }
}

int ew_dispatch_misc(int oc, EwParams& p, Stream* st) {
  switch (oc) {
    case OC_FILL: return launch_ew<OC_FILL, 0, 0, K_INT, -1, -1, -1>(p, st);
    case OC_ARANGE: return launch_ew<OC_ARANGE, 0, 0, K_INT, -1, -1, -1>(p, st);
    case OC_BSWAP: return launch_ew<OC_BSWAP, 1, 0, K_INT, -1, -1, -1>(p, st);
    default: return launch_ew<OC_RAW, 1, 0, K_INT, -1, -1, -1>(p, st);
  }
}

}  // namespace tpg
