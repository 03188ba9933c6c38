// tpg_runtime.cu — devices, stream-ordered caching allocator, streams,
// events, transfers and the sticky status word.
//
// Reference counterparts: devices.Device / Stream (pkg/src/tidepool/
// devices.py:47-192), storage_alloc (storage.py:91-97) and the sticky
// status set ops._status (ops.py:27-38).  The reference frees buffers when
// the Python object dies (storage.py:59-67); on the GPU a free must not
// overtake in-flight kernels, so frees are stream-ordered (cudaFreeAsync
// into the device's memory pool, whose release threshold keeps freed
// blocks cached for reuse: a caching allocator with stream semantics).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <string>
#include <vector>

#include "tpg_internal.h"

namespace tpg {

static thread_local std::string g_err;
static std::mutex g_mu;
static bool g_inited = false;
static int g_ndev = 0;
static std::vector<Stream*> g_default;
static std::vector<int> g_sms;
static std::vector<uint32_t*> g_flags;

void set_error(const std::string& msg) { g_err = msg; }

int cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? TPG_E_ALLOC : TPG_E_CUDA;
}

int arg_fail(const std::string& msg) {
  set_error(msg);
  return TPG_E_ARG;
}

static int init_locked() {
  if (g_inited) return TPG_OK;
  cudaError_t e = cudaGetDeviceCount(&g_ndev);
  if (e != cudaSuccess) {
    g_ndev = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  g_default.assign(g_ndev, nullptr);
  g_sms.assign(g_ndev, 0);
  g_flags.assign(g_ndev, nullptr);
  for (int d = 0; d < g_ndev; ++d) {
    TPG_CUDA_CHECK(cudaSetDevice(d));
    cudaDeviceProp prop;
    TPG_CUDA_CHECK(cudaGetDeviceProperties(&prop, d));
    g_sms[d] = prop.multiProcessorCount;
    Stream* st = new Stream{d, nullptr};
    TPG_CUDA_CHECK(cudaStreamCreateWithFlags(&st->s, cudaStreamNonBlocking));
    g_default[d] = st;
    // keep freed blocks cached in the pool (no release back to the OS)
    cudaMemPool_t pool;
    TPG_CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, d));
    uint64_t thresh = UINT64_MAX;
    TPG_CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
    uint32_t* f = nullptr;
    TPG_CUDA_CHECK(cudaMalloc(&f, 64));
    TPG_CUDA_CHECK(cudaMemset(f, 0, 64));
    g_flags[d] = f;
  }
  if (g_ndev > 0) TPG_CUDA_CHECK(cudaSetDevice(0));
  g_inited = true;
  return TPG_OK;
}

Stream* resolve_stream(tpg_stream s) {
  Stream* st = (Stream*)s;
  if (st == nullptr) {
    int d = 0;
    cudaGetDevice(&d);
    if (d < 0 || d >= (int)g_default.size()) return nullptr;
    st = g_default[d];
  }
  // cudaSetDevice only on a change (a host-side per-launch cost otherwise)
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != st->device) cudaSetDevice(st->device);
  return st;
}

int sm_count(int device) {
  if (device < 0 || device >= (int)g_sms.size()) return 148;
  return g_sms[device];
}

uint32_t* device_flags(int device) {
  if (device < 0 || device >= (int)g_flags.size()) return nullptr;
  return g_flags[device];
}

void* tensor_map_encoder() {
  static void* fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = p;
  }
  return fn;
}

uint32_t* stream_counters(Stream* st, int64_t n) {
  if (n <= st->ncounters) return st->counters;
  int64_t cap = st->ncounters ? st->ncounters : 4096;
  while (cap < n) cap *= 2;
  if (st->counters && cudaFreeAsync(st->counters, st->s) != cudaSuccess) return nullptr;
  st->counters = nullptr;
  st->ncounters = 0;
  uint32_t* c = nullptr;
  if (cudaMallocAsync((void**)&c, cap * sizeof(uint32_t), st->s) != cudaSuccess) return nullptr;
  if (cudaMemsetAsync(c, 0, cap * sizeof(uint32_t), st->s) != cudaSuccess) return nullptr;
  st->counters = c;
  st->ncounters = cap;
  return c;
}

}  // namespace tpg

using namespace tpg;

extern "C" {

const char* tpg_last_error(void) { return g_err.c_str(); }

const char* tpg_version(void) { return "tidepool_gpu 0.1 (sm_100a)"; }

int tpg_init(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  return init_locked();
}

int tpg_device_count(int* count) {
  int rc = tpg_init();
  *count = g_ndev;
  return rc;
}

int tpg_device_props_get(int device, tpg_device_props* p) {
  if (device < 0 || device >= g_ndev) return arg_fail("bad device index");
  cudaDeviceProp prop;
  TPG_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
  TPG_CUDA_CHECK(cudaSetDevice(device));
  size_t fr = 0, tot = 0;
  TPG_CUDA_CHECK(cudaMemGetInfo(&fr, &tot));
  p->sm_count = prop.multiProcessorCount;
  p->cc_major = prop.major;
  p->cc_minor = prop.minor;
  p->total_mem = (int64_t)tot;
  p->free_mem = (int64_t)fr;
  p->l2_bytes = prop.l2CacheSize;
  strncpy(p->name, prop.name, sizeof(p->name) - 1);
  p->name[sizeof(p->name) - 1] = 0;
  return TPG_OK;
}

int tpg_malloc(int device, size_t nbytes, void** ptr) {
  if (device < 0 || device >= g_ndev) return arg_fail("bad device index");
  TPG_CUDA_CHECK(cudaSetDevice(device));
  if (nbytes == 0) nbytes = 1;
  // round to 256 B so vectorized paths see aligned bases
  nbytes = (nbytes + 255) & ~(size_t)255;
  cudaError_t e = cudaMallocAsync(ptr, nbytes, g_default[device]->s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
  return TPG_OK;
}

int tpg_malloc_on(tpg_stream stream, size_t nbytes, void** ptr) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  if (nbytes == 0) nbytes = 1;
  nbytes = (nbytes + 255) & ~(size_t)255;
  cudaError_t e = cudaMallocAsync(ptr, nbytes, st->s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
  return TPG_OK;
}

int tpg_free(int device, void* ptr, tpg_stream stream) {
  if (ptr == nullptr) return TPG_OK;
  if (device < 0 || device >= g_ndev) return arg_fail("bad device index");
  TPG_CUDA_CHECK(cudaSetDevice(device));
  Stream* st = stream ? (Stream*)stream : g_default[device];
  TPG_CUDA_CHECK(cudaFreeAsync(ptr, st->s));
  return TPG_OK;
}

int tpg_host_alloc(size_t nbytes, void** ptr) {
  TPG_CUDA_CHECK(cudaHostAlloc(ptr, nbytes ? nbytes : 1, cudaHostAllocPortable));
  return TPG_OK;
}

int tpg_host_free(void* ptr) {
  TPG_CUDA_CHECK(cudaFreeHost(ptr));
  return TPG_OK;
}

int tpg_mem_stats(int device, int64_t* in_use, int64_t* cached, int64_t* n_alloc) {
  if (device < 0 || device >= g_ndev) return arg_fail("bad device index");
  cudaMemPool_t pool;
  TPG_CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t used = 0, reserved = 0;
  TPG_CUDA_CHECK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
  TPG_CUDA_CHECK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
  *in_use = (int64_t)used;
  *cached = (int64_t)(reserved - used);
  *n_alloc = 0;
  return TPG_OK;
}

int tpg_empty_cache(int device) {
  if (device < 0 || device >= g_ndev) return arg_fail("bad device index");
  TPG_CUDA_CHECK(cudaSetDevice(device));
  TPG_CUDA_CHECK(cudaDeviceSynchronize());
  cudaMemPool_t pool;
  TPG_CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, device));
  TPG_CUDA_CHECK(cudaMemPoolTrimTo(pool, 0));
  return TPG_OK;
}

int tpg_default_stream(int device, tpg_stream* stream) {
  if (device < 0 || device >= g_ndev) return arg_fail("bad device index");
  *stream = g_default[device];
  return TPG_OK;
}

int tpg_stream_create(int device, tpg_stream* stream) {
  if (device < 0 || device >= g_ndev) return arg_fail("bad device index");
  TPG_CUDA_CHECK(cudaSetDevice(device));
  Stream* st = new Stream{device, nullptr};
  cudaError_t e = cudaStreamCreateWithFlags(&st->s, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete st;
    return cuda_fail(e, "cudaStreamCreate");
  }
  *stream = st;
  return TPG_OK;
}

int tpg_stream_destroy(tpg_stream stream) {
  Stream* st = (Stream*)stream;
  if (!st) return TPG_OK;
  for (Stream* d : g_default)
    if (d == st) return arg_fail("cannot destroy a default stream");
  TPG_CUDA_CHECK(cudaSetDevice(st->device));
  if (st->counters) TPG_CUDA_CHECK(cudaFreeAsync(st->counters, st->s));
  TPG_CUDA_CHECK(cudaStreamDestroy(st->s));
  delete st;
  return TPG_OK;
}

int tpg_stream_sync(tpg_stream stream) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  TPG_CUDA_CHECK(cudaStreamSynchronize(st->s));
  return TPG_OK;
}

int tpg_stream_wait(tpg_stream waiter, tpg_stream signaller) {
  Stream* w = (Stream*)waiter;
  Stream* s = (Stream*)signaller;
  if (!w || !s) return arg_fail("null stream");
  TPG_CUDA_CHECK(cudaSetDevice(s->device));
  cudaEvent_t ev;
  TPG_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  TPG_CUDA_CHECK(cudaEventRecord(ev, s->s));
  TPG_CUDA_CHECK(cudaSetDevice(w->device));
  TPG_CUDA_CHECK(cudaStreamWaitEvent(w->s, ev, 0));
  TPG_CUDA_CHECK(cudaEventDestroy(ev));
  return TPG_OK;
}

int tpg_event_create(tpg_event* ev) {
  cudaEvent_t e;
  TPG_CUDA_CHECK(cudaEventCreate(&e));
  *ev = (tpg_event)e;
  return TPG_OK;
}

int tpg_event_destroy(tpg_event ev) {
  TPG_CUDA_CHECK(cudaEventDestroy((cudaEvent_t)ev));
  return TPG_OK;
}

int tpg_event_record(tpg_event ev, tpg_stream stream) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  TPG_CUDA_CHECK(cudaEventRecord((cudaEvent_t)ev, st->s));
  return TPG_OK;
}

int tpg_event_sync(tpg_event ev) {
  TPG_CUDA_CHECK(cudaEventSynchronize((cudaEvent_t)ev));
  return TPG_OK;
}

int tpg_event_elapsed(tpg_event start, tpg_event stop, float* ms) {
  TPG_CUDA_CHECK(cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)stop));
  return TPG_OK;
}

int tpg_memcpy_h2d(void* dst, const void* src, size_t n, tpg_stream stream) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  if (n == 0) return TPG_OK;
  TPG_CUDA_CHECK(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st->s));
  return TPG_OK;
}

int tpg_memcpy_d2h(void* dst, const void* src, size_t n, tpg_stream stream) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  if (n == 0) return TPG_OK;
  TPG_CUDA_CHECK(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st->s));
  return TPG_OK;
}

int tpg_memcpy_d2d(void* dst, const void* src, size_t n, tpg_stream stream) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  if (n == 0) return TPG_OK;
  TPG_CUDA_CHECK(cudaMemcpyAsync(dst, src, n, cudaMemcpyDefault, st->s));
  return TPG_OK;
}

int tpg_memcpy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                 size_t height, tpg_stream stream) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  if (width == 0 || height == 0) return TPG_OK;
  TPG_CUDA_CHECK(
      cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDefault, st->s));
  return TPG_OK;
}

int tpg_memset(void* dst, int value, size_t n, tpg_stream stream) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  if (n == 0) return TPG_OK;
  TPG_CUDA_CHECK(cudaMemsetAsync(dst, value, n, st->s));
  return TPG_OK;
}

// ---- L2 flush (measurement helper): write `n` bytes of scratch, then read
// them back with default-priority loads, so the L2 is left holding clean
// lines of an unrelated buffer (no dirty write-backs land in the next
// kernel's timing).
__global__ void k_l2_read(const uint4* a, size_t n, uint32_t* sink) {
  uint32_t acc = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldcg(a + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9e3779b9u) *sink = acc;  // keeps the loads live
}

int tpg_l2_flush(void* scratch, size_t n, tpg_stream stream) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  if (n < 16) return TPG_OK;
  static int salt = 0;
  TPG_CUDA_CHECK(cudaMemsetAsync(scratch, ++salt & 0xff, n, st->s));
  k_l2_read<<<sm_count(st->device) * 8, 256, 0, st->s>>>((const uint4*)scratch, n / 16 - 1,
                                                          (uint32_t*)((char*)scratch + n - 16));
  TPG_LAUNCH_CHECK("l2 flush");
  return TPG_OK;
}

// ---- launch gate (measurement helper): hold a stream until the host has
// enqueued a whole batch of timed steps, so host-side enqueue latency never
// shows up between the CUDA events of a step.
static volatile uint32_t* g_gate = nullptr;
static uint32_t* g_gate_dev = nullptr;

__global__ void k_gate(volatile uint32_t* flag) {
  const long long t0 = clock64();
  while (*flag == 0) {
    __nanosleep(2000);
    if (clock64() - t0 > 40000000000ll) break;  // ~20 s safety valve
  }
}

int tpg_gate_arm(tpg_stream stream) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  if (!g_gate) {
    void* h = nullptr;
    TPG_CUDA_CHECK(cudaHostAlloc(&h, 64, cudaHostAllocMapped | cudaHostAllocPortable));
    g_gate = (volatile uint32_t*)h;
    TPG_CUDA_CHECK(cudaHostGetDevicePointer((void**)&g_gate_dev, h, 0));
  }
  *g_gate = 0;
  __sync_synchronize();
  k_gate<<<1, 1, 0, st->s>>>(g_gate_dev);
  TPG_LAUNCH_CHECK("gate");
  return TPG_OK;
}

int tpg_gate_release(void) {
  if (g_gate) {
    __sync_synchronize();
    *g_gate = 1;
    __sync_synchronize();
  }
  return TPG_OK;
}

int tpg_flags_get(int device, uint32_t* flags) {
  if (device < 0 || device >= g_ndev) return arg_fail("bad device index");
  TPG_CUDA_CHECK(cudaSetDevice(device));
  // every stream of the device (the kernels run on non-blocking streams
  // that a legacy-stream cudaMemcpy would not wait for)
  TPG_CUDA_CHECK(cudaDeviceSynchronize());
  TPG_CUDA_CHECK(cudaMemcpy(flags, g_flags[device], sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return TPG_OK;
}

// Stream-ordered read-and-clear of the sticky status word: one thread swaps
// the word with 0 (atomicExch, so a bit OR-ed by a kernel on another stream
// of the same device is never lost between a read and a clear), the old
// value lands in pinned host memory, and the host waits for `stream` only.
__global__ void k_flags_take(uint32_t* flags, uint32_t* out) { *out = atomicExch(flags, 0u); }

int tpg_flags_take(tpg_stream stream, uint32_t* flags) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  static thread_local uint32_t* host_word = nullptr;
  if (!host_word) TPG_CUDA_CHECK(cudaHostAlloc((void**)&host_word, 64, cudaHostAllocPortable));
  uint32_t* dev_word = g_flags[st->device] + 8;  // scratch slot next to the sticky word
  k_flags_take<<<1, 1, 0, st->s>>>(g_flags[st->device], dev_word);
  TPG_LAUNCH_CHECK("flags take");
  TPG_CUDA_CHECK(cudaMemcpyAsync(host_word, dev_word, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                 st->s));
  TPG_CUDA_CHECK(cudaStreamSynchronize(st->s));
  *flags = *host_word;
  return TPG_OK;
}

// CUDA managed memory for storages the host also addresses (the drop-in
// plugin: the reference reads and writes storage bytes through memoryviews).
// Preferred location is the GPU; large blocks are migrated there up front so
// the first kernel does not fault them over page by page.
int tpg_malloc_managed(int device, size_t nbytes, void** ptr) {
  if (device < 0 || device >= g_ndev) return arg_fail("bad device index");
  TPG_CUDA_CHECK(cudaSetDevice(device));
  if (nbytes == 0) nbytes = 1;
  TPG_CUDA_CHECK(cudaMallocManaged(ptr, nbytes, cudaMemAttachGlobal));
  if (nbytes >= (1u << 20)) {
    cudaMemLocation loc;
    loc.type = cudaMemLocationTypeDevice;
    loc.id = device;
    cudaMemAdvise_v2(*ptr, nbytes, cudaMemAdviseSetPreferredLocation, loc);
    cudaMemLocation host;
    host.type = cudaMemLocationTypeHost;
    host.id = 0;
    cudaMemAdvise_v2(*ptr, nbytes, cudaMemAdviseSetAccessedBy, host);
    cudaMemPrefetchAsync_v2(*ptr, nbytes, loc, 0, g_default[device]->s);
    cudaGetLastError();  // advice is best effort
  }
  return TPG_OK;
}

int tpg_free_managed(void* ptr) {
  if (ptr == nullptr) return TPG_OK;
  TPG_CUDA_CHECK(cudaFree(ptr));
  return TPG_OK;
}

int tpg_event_create_untimed(tpg_event* ev) {
  cudaEvent_t e;
  TPG_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  *ev = (tpg_event)e;
  return TPG_OK;
}

int tpg_mark_word_create(uint64_t** word) {
  if (!word) return arg_fail("null word");
  void* p = nullptr;
  TPG_CUDA_CHECK(cudaHostAlloc(&p, 64, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(p, 0, 64);
  *word = (uint64_t*)p;
  return TPG_OK;
}

int tpg_mark_word_free(uint64_t* word) {
  if (word) TPG_CUDA_CHECK(cudaFreeHost(word));
  return TPG_OK;
}

int tpg_stream_mark(tpg_stream stream, uint64_t* word, uint64_t value) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  if (!word) return arg_fail("null word");
  void* dptr = nullptr;
  if (cudaHostGetDevicePointer(&dptr, word, 0) != cudaSuccess) {
    cudaGetLastError();
    return TPG_E_UNSUPPORTED;
  }
  // the driver entry point is resolved at run time (no link-time libcuda
  // dependency: the library still loads on a CPU-only host)
  typedef CUresult (*WriteValue64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
  static WriteValue64 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (WriteValue64)f;
  }
  if (!fn) return TPG_E_UNSUPPORTED;
  const CUresult r = fn((CUstream)st->s, (CUdeviceptr)dptr, (cuuint64_t)value,
                        CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) return TPG_E_UNSUPPORTED;
  return TPG_OK;
}

int tpg_event_query(tpg_event ev) {
  cudaError_t e = cudaEventQuery((cudaEvent_t)ev);
  if (e == cudaSuccess) return 0;
  if (e == cudaErrorNotReady) {
    cudaGetLastError();
    return 1;
  }
  return cuda_fail(e, "cudaEventQuery");
}

// Peer access between every pair of visible devices (NVLink / NVSwitch):
// cross-device copies and kernels reading a peer's memory go over the link
// directly.  Pairs that cannot peer are skipped; returns the number of
// pairs enabled in *enabled.
int tpg_enable_peer_all(int* enabled) {
  int rc = tpg_init();
  if (rc) return rc;
  int n = 0;
  for (int a = 0; a < g_ndev; ++a) {
    for (int b = 0; b < g_ndev; ++b) {
      if (a == b) continue;
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, a, b) != cudaSuccess || !can) continue;
      TPG_CUDA_CHECK(cudaSetDevice(a));
      cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        e = cudaSuccess;
      }
      if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
      ++n;
    }
  }
  if (enabled) *enabled = n;
  return TPG_OK;
}

// CUDA graphs for launch-bound sequences (e.g. many small elementwise ops):
// capture everything enqueued on `stream` between begin and end, replay it
// with one launch.
int tpg_graph_begin(tpg_stream stream) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  TPG_CUDA_CHECK(cudaStreamBeginCapture(st->s, cudaStreamCaptureModeThreadLocal));
  return TPG_OK;
}

int tpg_graph_end(tpg_stream stream, void** graph_exec) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  cudaGraph_t g = nullptr;
  TPG_CUDA_CHECK(cudaStreamEndCapture(st->s, &g));
  cudaGraphExec_t ge = nullptr;
  cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
  *graph_exec = (void*)ge;
  return TPG_OK;
}

int tpg_graph_launch(void* graph_exec, tpg_stream stream) {
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  TPG_CUDA_CHECK(cudaGraphLaunch((cudaGraphExec_t)graph_exec, st->s));
  return TPG_OK;
}

int tpg_graph_destroy(void* graph_exec) {
  if (graph_exec) TPG_CUDA_CHECK(cudaGraphExecDestroy((cudaGraphExec_t)graph_exec));
  return TPG_OK;
}

int tpg_flags_clear(int device) {
  if (device < 0 || device >= g_ndev) return arg_fail("bad device index");
  TPG_CUDA_CHECK(cudaSetDevice(device));
  TPG_CUDA_CHECK(cudaDeviceSynchronize());
  TPG_CUDA_CHECK(cudaMemset(g_flags[device], 0, sizeof(uint32_t)));
  return TPG_OK;
}

}  // extern "C"
