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
}  // namespace tpg

using namespace tpg;

extern "C" {

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
