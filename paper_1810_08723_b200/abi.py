"""ctypes mirror of include/tidepool_gpu.h (structs, enums, prototypes)."""

from __future__ import annotations

import ctypes as C

MAX_DIMS = 8
MAX_VIEWS = 3

# op codes (tidepool_gpu.h)
BINARY_CODE = {"add": 0, "subtract": 1, "multiply": 2, "divide": 3, "minimum": 4, "maximum": 5}
UNARY_CODE = {"negate": 0, "absolute": 1, "square_root": 2, "exponential": 3, "logarithm": 4,
              "sine": 5, "cosine": 6, "arcsine": 7, "arccosine": 8, "conjugate": 9,
              "identity": 10}
REDUCE_CODE = {"sum": 0, "product": 1, "minimum": 2, "maximum": 3, "any": 4, "all": 5,
               "norm": 6}
FLAG_DOMAIN = 1
FLAG_INT_DIV0 = 2
FLAG_CAST_LOSS = 4


class Plan(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("nviews", C.c_int32),
                ("extent", C.c_int64 * MAX_DIMS),
                ("stride", (C.c_int64 * MAX_DIMS) * MAX_VIEWS)]


class Operand(C.Structure):
    _fields_ = [("base", C.c_void_p), ("offset", C.c_int64), ("dtype", C.c_int32),
                ("big_endian", C.c_int32), ("imm", C.c_uint64 * 2)]


class ChainStep(C.Structure):
    _fields_ = [("op", C.c_int32), ("dtype", C.c_int32), ("compute", C.c_int32),
                ("scalar_first", C.c_int32), ("scalar_dtype", C.c_int32),
                ("reserved", C.c_int32), ("scalar", C.c_uint8 * 16)]


class DeviceProps(C.Structure):
    _fields_ = [("sm_count", C.c_int32), ("cc_major", C.c_int32), ("cc_minor", C.c_int32),
                ("total_mem", C.c_int64), ("free_mem", C.c_int64), ("l2_bytes", C.c_int32),
                ("name", C.c_char * 128)]


def make_plan(extents, strides_per_view) -> Plan:
    p = Plan()
    p.ndim = len(extents)
    p.nviews = len(strides_per_view)
    if p.ndim > MAX_DIMS:
        raise ValueError("plan has too many axes")
    for k, e in enumerate(extents):
        p.extent[k] = e
    for v, s in enumerate(strides_per_view):
        for k, x in enumerate(s):
            p.stride[v][k] = x
    return p


def make_operand(ptr, offset, dtype_code, big_endian, imm: bytes | None = None) -> Operand:
    o = Operand()
    o.base = ptr
    o.offset = offset
    o.dtype = dtype_code
    o.big_endian = 1 if big_endian else 0
    if imm is not None:
        raw = imm.ljust(16, b"\0")
        o.imm[0] = int.from_bytes(raw[:8], "little")
        o.imm[1] = int.from_bytes(raw[8:16], "little")
    return o


P = C.POINTER
_i32, _i64, _f64, _vp = C.c_int32, C.c_int64, C.c_double, C.c_void_p
_PLAN, _OP = P(Plan), P(Operand)

# name -> (restype, argtypes); the list every test checks the .so exports
PROTOTYPES = {
    "tpg_init": (_i32, []),
    "tpg_device_count": (_i32, [P(C.c_int)]),
    "tpg_device_props_get": (_i32, [C.c_int, P(DeviceProps)]),
    "tpg_last_error": (C.c_char_p, []),
    "tpg_version": (C.c_char_p, []),
    "tpg_malloc": (_i32, [C.c_int, C.c_size_t, P(_vp)]),
    "tpg_free": (_i32, [C.c_int, _vp, _vp]),
    "tpg_malloc_on": (_i32, [_vp, C.c_size_t, P(_vp)]),
    "tpg_host_alloc": (_i32, [C.c_size_t, P(_vp)]),
    "tpg_host_free": (_i32, [_vp]),
    "tpg_mem_stats": (_i32, [C.c_int, P(_i64), P(_i64), P(_i64)]),
    "tpg_empty_cache": (_i32, [C.c_int]),
    "tpg_default_stream": (_i32, [C.c_int, P(_vp)]),
    "tpg_stream_create": (_i32, [C.c_int, P(_vp)]),
    "tpg_stream_destroy": (_i32, [_vp]),
    "tpg_stream_sync": (_i32, [_vp]),
    "tpg_stream_wait": (_i32, [_vp, _vp]),
    "tpg_event_create": (_i32, [P(_vp)]),
    "tpg_event_destroy": (_i32, [_vp]),
    "tpg_event_record": (_i32, [_vp, _vp]),
    "tpg_event_sync": (_i32, [_vp]),
    "tpg_event_elapsed": (_i32, [_vp, _vp, P(C.c_float)]),
    "tpg_memcpy_h2d": (_i32, [_vp, _vp, C.c_size_t, _vp]),
    "tpg_memcpy_d2h": (_i32, [_vp, _vp, C.c_size_t, _vp]),
    "tpg_memcpy_d2d": (_i32, [_vp, _vp, C.c_size_t, _vp]),
    "tpg_memset": (_i32, [_vp, C.c_int, C.c_size_t, _vp]),
    "tpg_memcpy2d": (_i32, [_vp, C.c_size_t, _vp, C.c_size_t, C.c_size_t, C.c_size_t, _vp]),
    "tpg_flags_get": (_i32, [C.c_int, P(C.c_uint32)]),
    "tpg_flags_clear": (_i32, [C.c_int]),
    "tpg_flags_take": (_i32, [_vp, P(C.c_uint32)]),
    "tpg_malloc_managed": (_i32, [C.c_int, C.c_size_t, P(_vp)]),
    "tpg_free_managed": (_i32, [_vp]),
    "tpg_event_create_untimed": (_i32, [P(_vp)]),
    "tpg_event_query": (_i32, [_vp]),
    "tpg_mark_word_create": (_i32, [P(_vp)]),
    "tpg_mark_word_free": (_i32, [_vp]),
    "tpg_stream_mark": (_i32, [_vp, _vp, C.c_uint64]),
    "tpg_l2_flush": (_i32, [_vp, C.c_size_t, _vp]),
    "tpg_enable_peer_all": (_i32, [P(C.c_int)]),
    "tpg_graph_begin": (_i32, [_vp]),
    "tpg_graph_end": (_i32, [_vp, P(_vp)]),
    "tpg_graph_launch": (_i32, [_vp, _vp]),
    "tpg_graph_destroy": (_i32, [_vp]),
    "tpg_gate_arm": (_i32, [_vp]),
    "tpg_gate_release": (_i32, []),
    "tpg_binary": (_i32, [_vp, C.c_int, _PLAN, _OP, _OP, _OP, C.c_int, C.c_int]),
    "tpg_unary": (_i32, [_vp, C.c_int, _PLAN, _OP, _OP, C.c_int, C.c_int, C.c_int]),
    "tpg_copy": (_i32, [_vp, _PLAN, _OP, _OP, C.c_int]),
    "tpg_reduce": (_i32, [_vp, C.c_int, _f64, _PLAN, _PLAN, _OP, _OP, C.c_int, C.c_int]),
    "tpg_matmul": (_i32, [_vp, _OP, P(_i64), _OP, P(_i64), _OP, P(_i64), _i64, _i64, _i64,
                          C.c_int, C.c_int]),
    "tpg_matmul_batched": (_i32, [_vp, _i64, _OP, P(_i64), _OP, P(_i64), _OP, P(_i64), _i64,
                                  _i64, _i64, C.c_int, C.c_int]),
    "tpg_chain": (_i32, [_vp, _PLAN, _OP, _OP, C.c_int, C.POINTER(ChainStep), C.c_int]),
    "tpg_chain_check": (_i32, [_vp, _PLAN, _OP, _OP, C.c_int, C.POINTER(ChainStep), C.c_int]),
    "tpg_fill": (_i32, [_vp, _PLAN, _OP, _vp, _i32]),
    "tpg_arange": (_i32, [_vp, _PLAN, _OP]),
    "tpg_byteswap": (_i32, [_vp, _PLAN, _OP]),
    "tpg_gather": (_i32, [_vp, _vp, _vp, P(_i64), _i64, _i32]),
    "tpg_gather_plan": (_i32, [_vp, _PLAN, _vp, _i64, _vp, _i64, _i32]),
    "tpg_scatter": (_i32, [_vp, P(_i64), _i64, _OP, _OP, C.c_int]),
    "tpg_scatter_fill": (_i32, [_vp, P(_i64), _i64, _vp, _vp, _i32]),
    "tpg_nccl_get_unique_id": (_i32, [_vp]),
    "tpg_nccl_init": (_i32, [C.c_int, C.c_int, C.c_int, _vp]),
    "tpg_nccl_allreduce": (_i32, [_vp, _vp, _i64, C.c_int, C.c_int]),
    "tpg_nccl_destroy": (_i32, []),
    "tpg_nccl_info": (_i32, [P(C.c_int), P(C.c_int)]),
    "tpg_p2p_init": (_i32, [C.c_int, C.c_int, C.c_int, _vp]),
    "tpg_p2p_connect": (_i32, [_vp]),
    "tpg_p2p_allreduce": (_i32, [_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_ulonglong]),
    "tpg_p2p_destroy": (_i32, []),
    "tpg_reduce_sum_p2p": (_i32, [_vp, _PLAN, _PLAN, _OP, _OP, C.c_ulonglong]),
    "tpg_reduce_norm2_p2p": (_i32, [_vp, _PLAN, _PLAN, _OP, _OP, C.c_ulonglong]),
    "tpg_reduce_minmax_p2p": (_i32, [_vp, C.c_int, _PLAN, _PLAN, _OP, _OP, C.c_ulonglong,
                                     _i64]),
    "tpg_shard_pack": (_i32, [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, C.c_int, C.c_int]),
    "tpg_shard_unpack": (_i32, [_vp, C.c_int, C.c_int, _vp]),
}

# not in the public header (host-side error-mode pre-checks)
EXTRA_PROTOTYPES = {
    "tpg_binary_check": (_i32, [_vp, C.c_int, _PLAN, _OP, _OP, _OP, C.c_int, C.c_int]),
    "tpg_unary_check": (_i32, [_vp, C.c_int, _PLAN, _OP, _OP, C.c_int, C.c_int, C.c_int]),
}


def declare(lib, table=None):
    for name, (res, args) in (table or {**PROTOTYPES, **EXTRA_PROTOTYPES}).items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib
