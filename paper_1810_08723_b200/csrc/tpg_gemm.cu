// tpg_gemm.cu — matmul table entry: picks the tcgen05 tensor-core path
// (tpg_gemm_sm100.cu) when dtypes/layout/size allow, else the SIMT path.
// Reference: kernels.matmul (pkg/src/tidepool/kernels.py:323-340),
// ops.matmul (ops.py:577-640); batched gemm is an extension entry.
#include <cuda_runtime.h>

#include "tpg_common.cuh"
#include "tpg_internal.h"

namespace tpg {
int gemm_simt(Stream* st, int64_t batch, const tpg_operand* d, const int64_t* ds,
              const tpg_operand* a, const int64_t* as, const tpg_operand* b, const int64_t* bs,
              int64_t m, int64_t n, int64_t k, int compute, int mode);
// returns 1 when handled, 0 when the shape/layout is not eligible, <0 error
int gemm_sm100(Stream* st, int64_t batch, const tpg_operand* d, const int64_t* ds,
               const tpg_operand* a, const int64_t* as, const tpg_operand* b, const int64_t* bs,
               int64_t m, int64_t n, int64_t k, int compute, int mode);
}  // namespace tpg

using namespace tpg;

static int matmul_impl(tpg_stream stream, int64_t batch, const tpg_operand* d, const int64_t* ds,
                       const tpg_operand* a, const int64_t* as, const tpg_operand* b,
                       const int64_t* bs, int64_t m, int64_t n, int64_t k, int compute, int mode) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  if (!d || !a || !b || !d->base || !a->base || !b->base) return arg_fail("matmul: null operand");
  if (m < 0 || n < 0 || k < 0 || batch < 0) return arg_fail("matmul: negative size");
  if (m == 0 || n == 0 || batch == 0) return TPG_OK;
  int rc = gemm_sm100(st, batch, d, ds, a, as, b, bs, m, n, k, compute, mode);
  if (rc < 0) return rc;
  if (rc == 1) return TPG_OK;
  return gemm_simt(st, batch, d, ds, a, as, b, bs, m, n, k, compute, mode);
}

extern "C" {

int tpg_matmul(tpg_stream stream, const tpg_operand* d, const int64_t d_strides[2],
               const tpg_operand* a, const int64_t a_strides[2], const tpg_operand* b,
               const int64_t b_strides[2], int64_t m, int64_t n, int64_t k, int compute,
               int mode) {
  int64_t ds[3] = {d_strides[0], d_strides[1], 0};
  int64_t as[3] = {a_strides[0], a_strides[1], 0};
  int64_t bs[3] = {b_strides[0], b_strides[1], 0};
  return matmul_impl(stream, 1, d, ds, a, as, b, bs, m, n, k, compute, mode);
}

int tpg_matmul_batched(tpg_stream stream, int64_t batch, const tpg_operand* d,
                       const int64_t d_strides[3], const tpg_operand* a,
                       const int64_t a_strides[3], const tpg_operand* b,
                       const int64_t b_strides[3], int64_t m, int64_t n, int64_t k, int compute,
                       int mode) {
  int64_t ds[3] = {d_strides[0], d_strides[1], d_strides[2]};
  int64_t as[3] = {a_strides[0], a_strides[1], a_strides[2]};
  int64_t bs[3] = {b_strides[0], b_strides[1], b_strides[2]};
  return matmul_impl(stream, batch, d, ds, a, as, b, bs, m, n, k, compute, mode);
}

}  // extern "C"
