// tpg_comm.cu — NCCL plumbing for the multi-GPU full-reduction finish
// (each rank reduces its shard to one partial, one
// ncclAllReduce over NVLink/NVSwitch combines them).  The reference has no
// collective (it is single-process, placement-only multi-device).
// libnccl is loaded lazily with dlopen so the library itself has no hard
// NCCL dependency (single-GPU users never touch it).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <string>

#include "tpg_internal.h"

namespace tpg {
typedef ncclResult_t (*fn_uid)(ncclUniqueId*);
typedef ncclResult_t (*fn_init)(ncclComm_t*, int, ncclUniqueId, int);
typedef ncclResult_t (*fn_ar)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t);
typedef ncclResult_t (*fn_destroy)(ncclComm_t);
typedef const char* (*fn_err)(ncclResult_t);

static void* g_lib = nullptr;
static fn_uid p_uid = nullptr;
static fn_init p_init = nullptr;
static fn_ar p_ar = nullptr;
static fn_destroy p_destroy = nullptr;
static fn_err p_err = nullptr;
static ncclComm_t g_comm = nullptr;

static int load_nccl() {
  if (g_lib) return TPG_OK;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* n : names) {
    g_lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (g_lib) break;
  }
  if (!g_lib) {
    set_error(std::string("cannot load libnccl: ") + dlerror());
    return TPG_E_NCCL;
  }
  p_uid = (fn_uid)dlsym(g_lib, "ncclGetUniqueId");
  p_init = (fn_init)dlsym(g_lib, "ncclCommInitRank");
  p_ar = (fn_ar)dlsym(g_lib, "ncclAllReduce");
  p_destroy = (fn_destroy)dlsym(g_lib, "ncclCommDestroy");
  p_err = (fn_err)dlsym(g_lib, "ncclGetErrorString");
  if (!p_uid || !p_init || !p_ar || !p_destroy) {
    set_error("libnccl is missing required symbols");
    return TPG_E_NCCL;
  }
  return TPG_OK;
}

static int nccl_fail(ncclResult_t r, const char* what) {
  set_error(std::string(what) + ": " + (p_err ? p_err(r) : "nccl error"));
  return TPG_E_NCCL;
}

static ncclDataType_t nccl_dt(int dt, bool* ok) {
  *ok = true;
  switch (dt) {
    case TPG_INT8: return ncclInt8;
    case TPG_UINT8: case TPG_BOOL: return ncclUint8;
    case TPG_INT32: return ncclInt32;
    case TPG_UINT32: return ncclUint32;
    case TPG_INT64: return ncclInt64;
    case TPG_UINT64: return ncclUint64;
    case TPG_HALF: return ncclFloat16;
    case TPG_FLOAT: return ncclFloat32;
    case TPG_DOUBLE: return ncclFloat64;
    case TPG_BF16: return ncclBfloat16;
    default: *ok = false; return ncclFloat64;
  }
}
// ---- sharded min/max finish: one MAX all-reduce over a 2-slot payload
// (SURVEY §8e).  slot 0 = order key of the rank's extreme over its non-NaN
// elements (lowest key when the rank holds none), slot 1 = 1 iff this rank
// holds the tensor's first element and it is NaN (the reference's
// first-element rule, ops.py:533-544).  Keys are order-preserving maps into
// the payload type, so MAX serves both ops: doubles (float sources) use
// v / -v; signed integers (int64 payload) v / ~v; unsigned (uint64 source)
// flip the sign bit first.  All exact.
__device__ __forceinline__ int64_t key_of_u64(uint64_t u) {
  return (int64_t)(u ^ 0x8000000000000000ull);
}

__global__ void k_shard_pack(int is_max, int kind, int has, void* payload, const void* first,
                             int first_dtype, int first_big) {
  double fnan = 0.0;
  if (first) {
    double v = 0.0;
    if (first_dtype == TPG_DOUBLE) {
      uint64_t b = *(const uint64_t*)first;
      if (first_big) b = __byte_perm((uint32_t)(b >> 32), 0, 0x0123) |
                         ((uint64_t)__byte_perm((uint32_t)b, 0, 0x0123) << 32);
      v = __longlong_as_double((long long)b);
    } else if (first_dtype == TPG_FLOAT) {
      uint32_t b = *(const uint32_t*)first;
      if (first_big) b = __byte_perm(b, 0, 0x0123);
      v = (double)__uint_as_float(b);
    } else if (first_dtype == TPG_HALF || first_dtype == TPG_BF16) {
      uint16_t b = *(const uint16_t*)first;
      if (first_big) b = (uint16_t)((b >> 8) | (b << 8));
      const uint32_t exp_mask = first_dtype == TPG_HALF ? 0x7c00u : 0x7f80u;
      const uint32_t man_mask = first_dtype == TPG_HALF ? 0x03ffu : 0x007fu;
      v = ((b & exp_mask) == exp_mask && (b & man_mask)) ? __longlong_as_double(0x7ff8000000000000ll)
                                                         : 0.0;
    }
    fnan = v != v ? 1.0 : 0.0;
  }
  if (kind == 0) {  // double payload
    double* p = (double*)payload;
    const double v = p[0];
    // a NaN partial means the rank holds no non-NaN value: lowest key
    p[0] = (has && v == v) ? (is_max ? v : -v) : -__longlong_as_double(0x7ff0000000000000ll);
    p[1] = fnan;
  } else {  // int64 payload (kind 1 signed, kind 2 unsigned source)
    int64_t* p = (int64_t*)payload;
    int64_t k = kind == 2 ? key_of_u64((uint64_t)p[0]) : p[0];
    p[0] = has ? (is_max ? k : ~k) : (int64_t)0x8000000000000000ull;
    p[1] = 0;
  }
}

// inverse map; the extreme goes back to slot 0 in the partial's type, slot 1
// keeps the NaN flag (the host copies slot 0, or a NaN, into the result)
__global__ void k_shard_unpack(int is_max, int kind, void* payload) {
  if (kind == 0) {
    double* p = (double*)payload;
    p[0] = p[1] != 0.0 ? __longlong_as_double(0x7ff8000000000000ll) : (is_max ? p[0] : -p[0]);
  } else {
    int64_t* p = (int64_t*)payload;
    const int64_t k = is_max ? p[0] : ~p[0];
    p[0] = kind == 2 ? (int64_t)((uint64_t)k ^ 0x8000000000000000ull) : k;
  }
}
}  // namespace tpg

using namespace tpg;

extern "C" {

int tpg_shard_pack(tpg_stream stream, int is_max, int kind, int has, void* payload,
                   const void* first, int first_dtype, int first_big_endian) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  if (kind < 0 || kind > 2) return arg_fail("shard pack: bad payload kind");
  k_shard_pack<<<1, 1, 0, st->s>>>(is_max, kind, has, payload, first, first_dtype,
                                   first_big_endian);
  TPG_LAUNCH_CHECK("shard pack");
  return TPG_OK;
}

int tpg_shard_unpack(tpg_stream stream, int is_max, int kind, void* payload) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  if (kind < 0 || kind > 2) return arg_fail("shard unpack: bad payload kind");
  k_shard_unpack<<<1, 1, 0, st->s>>>(is_max, kind, payload);
  TPG_LAUNCH_CHECK("shard unpack");
  return TPG_OK;
}

int tpg_nccl_info(int* nranks, int* rank) {
  if (!g_comm) return arg_fail("nccl communicator not initialised");
  typedef ncclResult_t (*fn_count)(const ncclComm_t, int*);
  fn_count p_count = (fn_count)dlsym(g_lib, "ncclCommCount");
  fn_count p_rank = (fn_count)dlsym(g_lib, "ncclCommUserRank");
  if (!p_count || !p_rank) return arg_fail("libnccl lacks ncclCommCount / ncclCommUserRank");
  ncclResult_t r = p_count(g_comm, nranks);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommCount");
  r = p_rank(g_comm, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommUserRank");
  return TPG_OK;
}

int tpg_nccl_get_unique_id(void* id128) {
  int rc = load_nccl();
  if (rc) return rc;
  ncclUniqueId id;
  ncclResult_t r = p_uid(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(id128, &id, sizeof(id));
  return TPG_OK;
}

int tpg_nccl_init(int device, int nranks, int rank, const void* id128) {
  int rc = load_nccl();
  if (rc) return rc;
  TPG_CUDA_CHECK(cudaSetDevice(device));
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclResult_t r = p_init(&g_comm, nranks, id, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  return TPG_OK;
}

int tpg_nccl_allreduce(tpg_stream stream, void* buf, int64_t count, int dtype, int op) {
  if (!g_comm) return arg_fail("nccl communicator not initialised");
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  bool ok;
  ncclDataType_t t = nccl_dt(dtype, &ok);
  if (!ok) return arg_fail("allreduce: unsupported dtype");
  if (op < 0 || op > 3) return arg_fail("allreduce: bad op");
  ncclResult_t r = p_ar(buf, buf, (size_t)count, t, (ncclRedOp_t)op, g_comm, st->s);
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
  return TPG_OK;
}

int tpg_nccl_destroy(void) {
  if (g_comm && p_destroy) p_destroy(g_comm);
  g_comm = nullptr;
  return TPG_OK;
}

}  // extern "C"
