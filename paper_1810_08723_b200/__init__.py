"""B200-native gpu device module for the tidepool dense-tensor core
(arXiv 1810.08723, reference `tidepool`).

Importing the package registers module "core" and the ("core", "gpu")
function table (table.build_core_table, 31 entries backed by
libtidepool_gpu.so) in this package's dispatch registry, and exposes the
reference API names (add, reduce, matmul, cast, ...) over gpu tensors.
`paper_1810_08723_b200.tidepool_plugin.register()` attaches the same
kernels to an unmodified reference `tidepool` as its "gpu" device type.
"""

from . import dispatch as _dispatch
from . import dtypes, errors, plan, table, tensors
from .devices import GPU_TYPE, configure, gpu, list_devices
from .dispatch import lookup, override_op, register_device_impl, register_module, table_stats
from .dtypes import (cast_scalar, implicit_casting, promote, set_implicit_casting,
                     set_warning_handler, widen_for_compute)
from .errors import *  # noqa: F401,F403
from .ops import (absolute, add, arange, arccosine, arcsine, array_equal, byteswap, cast,
                  clear_status, conjugate, copy, cosine, divide, ensure, exponential, fill,
                  frobenius_norm, get_status, identity, inner, logarithm, matmul, matmul_batched, chain,
                  maximum, minimum, multiply, negate, ones, outer, reduce, sine, square_root,
                  subtract, zeros)
from . import profiling, transfer  # noqa: F401
from .transfer import download, pinned, upload, use_stream
from .otp1 import load_otp1, save_otp1, save_otp1_bytes
from .plan import IterPlan, build_plan, canonicalize
from .tensors import (MAX_DIMS, Scalar, Tensor, apply_index, broadcast_to, contiguous_clone,
                     diag_view, from_nested, from_numpy, imag_view, pair_overlap, permute_axes,
                     read_values, real_view, reshape, scalar_tensor, self_overlap, set_byteorder,
                     set_default_device, set_default_dtype, tensor, tensor_create,
                     tensor_from_nested, tensor_from_storage, to_numpy, transpose)

_dispatch.register_module("core")
_dispatch.register_device_impl("core", "gpu", table.build_core_table())
# extension entries beyond the reference's 31 keys (dispatch.add_op,
# reference dispatch.py:111-117)
_dispatch.add_op("core", "gpu", "ewise_chain", table.chain_entry)
_dispatch.add_op("core", "gpu", "matmul_batched", table.matmul_batched_entry)

bool = dtypes.BOOL  # noqa: A001
int8 = dtypes.INT8
uint8 = dtypes.UINT8
int16 = dtypes.INT16
uint16 = dtypes.UINT16
int32 = dtypes.INT32
uint32 = dtypes.UINT32
int64 = dtypes.INT64
uint64 = dtypes.UINT64
half = dtypes.HALF
float = dtypes.FLOAT  # noqa: A001
double = dtypes.DOUBLE
complex_half = dtypes.CHALF
complex_float = dtypes.CFLOAT
complex_double = dtypes.CDOUBLE
bfloat16 = dtypes.BFLOAT16
ALL_DTYPES = dtypes.ALL_DTYPES

__version__ = "0.1.0"
