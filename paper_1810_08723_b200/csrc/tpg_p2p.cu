// tpg_p2p.cu — the sharded full-reduction finish over NVLink peer memory,
// without NCCL (the task's "compute step followed by a
// collective" rule: the collective here is a 2-slot payload, where NCCL's
// launch + protocol latency dominates the combine).
//
// Every rank owns a small mailbox in device memory (cudaMalloc, exported
// with cudaIpcGetMemHandle, opened by every peer with cudaIpcOpenMemHandle,
// so on an NVSwitch box each rank's stores into a peer's mailbox travel over
// NVLink).  One exchange kernel per call, enqueued right after the local
// reduction on the same stream (no host round trip):
//   1. lane r < world stores this rank's payload into mailbox[r]'s slot
//      [parity][rank], then publishes the call's epoch with a system-scope
//      release store;
//   2. lane r spins (system-scope acquire, bounded) until this rank's own
//      slot [parity][r] carries the epoch;
//   3. lane 0 combines the world payloads IN RANK ORDER (deterministic,
//      unlike a tree / ring all-reduce) and writes the result in place.
// Parity double-buffering makes back-to-back calls safe: a rank can start
// call e+2 (reusing parity e%2) only after every rank wrote its call-(e+1)
// payload, i.e. after every rank finished reading call e.
#include <cuda_runtime.h>
#include <string.h>

#include <vector>

#include "tpg_internal.h"

namespace tpg {

typedef P2pSlot Slot;
// mailbox layout: Slot[2][P2P_MAX_RANKS]
constexpr size_t P2P_MAILBOX = sizeof(Slot) * 2 * P2P_MAX_RANKS;

struct P2pState {
  int device = -1, rank = 0, world = 0;
  void* mine = nullptr;                 // this rank's mailbox
  std::vector<void*> opened;            // peers' mailboxes (IPC mappings)
  Slot** dev_boxes = nullptr;           // device array: mailbox of every rank
};
static P2pState g_p2p;

P2pSlot** p2p_boxes(int* rank, int* world) {
  *rank = g_p2p.rank;
  *world = g_p2p.world;
  return g_p2p.dev_boxes;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

template <typename T>
__device__ __forceinline__ T combine(T a, T b, int op) {
  switch (op) {
    case 0: return a + b;
    case 1: return a * b;
    case 2: return a > b ? a : b;
    default: return a < b ? a : b;
  }
}

template <typename T>
__global__ void k_p2p_allreduce(Slot** boxes, int rank, int world, unsigned long long epoch,
                                T* payload, int count, int op, uint32_t* flags) {
  const int r = threadIdx.x;
  const int par = (int)(epoch & 1);
  if (r < world) {
    Slot* dst = boxes[r] + par * P2P_MAX_RANKS + rank;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      if (i < count) {
        uint64_t w = 0;
        memcpy(&w, &payload[i], sizeof(T));
        ((volatile uint64_t*)dst->payload)[i] = w;
      }
    }
    __threadfence_system();
    st_release_sys(&dst->epoch, epoch);
    // wait for rank r's payload in this rank's own mailbox
    const Slot* mine = boxes[rank] + par * P2P_MAX_RANKS + r;
    const long long t0 = clock64();
    while (ld_acquire_sys(&mine->epoch) < epoch) {
      if (clock64() - t0 > (1ll << 33)) {  // ~4 s: a peer never arrived
        atomicOr(flags, 0x80000000u);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  if (r == 0) {
    const Slot* base = boxes[rank] + par * P2P_MAX_RANKS;
    auto slot_val = [&](int q, int i) {
      const uint64_t w = ((const volatile uint64_t*)base[q].payload)[i];
      T v;
      memcpy(&v, &w, sizeof(T));
      return v;
    };
    for (int i = 0; i < count; ++i) {
      T acc = slot_val(0, i);
      for (int q = 1; q < world; ++q) acc = combine(acc, slot_val(q, i), op);
      payload[i] = acc;
    }
  }
}

}  // namespace tpg

using namespace tpg;

extern "C" {

// this rank's mailbox (allocated once) exported as a 64-byte IPC handle
int tpg_p2p_init(int device, int rank, int world, void* handle64) {
  if (world < 1 || world > P2P_MAX_RANKS || rank < 0 || rank >= world)
    return arg_fail("p2p: bad rank / world");
  TPG_CUDA_CHECK(cudaSetDevice(device));
  if (g_p2p.mine == nullptr) {
    TPG_CUDA_CHECK(cudaMalloc(&g_p2p.mine, P2P_MAILBOX));
    TPG_CUDA_CHECK(cudaMemset(g_p2p.mine, 0, P2P_MAILBOX));
  }
  g_p2p.device = device;
  g_p2p.rank = rank;
  g_p2p.world = world;
  cudaIpcMemHandle_t h;
  TPG_CUDA_CHECK(cudaIpcGetMemHandle(&h, g_p2p.mine));
  memcpy(handle64, &h, sizeof(h));
  return TPG_OK;
}

// open every peer's mailbox from the world's handles (world x 64 bytes, in
// rank order; this rank's own entry is ignored)
int tpg_p2p_connect(const void* handles) {
  if (g_p2p.mine == nullptr) return arg_fail("p2p: tpg_p2p_init first");
  TPG_CUDA_CHECK(cudaSetDevice(g_p2p.device));
  std::vector<void*> boxes(g_p2p.world, nullptr);
  for (int q = 0; q < g_p2p.world; ++q) {
    if (q == g_p2p.rank) {
      boxes[q] = g_p2p.mine;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, (const char*)handles + 64 * q, sizeof(h));
    void* p = nullptr;
    TPG_CUDA_CHECK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    boxes[q] = p;
    g_p2p.opened.push_back(p);
  }
  if (!g_p2p.dev_boxes) TPG_CUDA_CHECK(cudaMalloc(&g_p2p.dev_boxes, sizeof(void*) * P2P_MAX_RANKS));
  TPG_CUDA_CHECK(cudaMemcpy(g_p2p.dev_boxes, boxes.data(), sizeof(void*) * g_p2p.world,
                            cudaMemcpyHostToDevice));
  return TPG_OK;
}

// in-place all-reduce of `count` (<= 2) 8-byte elements on `stream`;
// dtype: TPG_DOUBLE, TPG_INT64, TPG_UINT64, TPG_UINT8 / TPG_BOOL; op: 0 sum,
// 1 prod, 2 max, 3 min.  A peer that never arrives (~4 s) sets bit 31 of the
// device's status word (read with tpg_flags_take).
// `epoch` must increase by one per call, identically on every rank.
int tpg_p2p_allreduce(tpg_stream stream, void* payload, int count, int dtype, int op,
                      unsigned long long epoch) {
  if (!g_p2p.dev_boxes) return arg_fail("p2p: not connected");
  if (count < 1 || count > 2 || op < 0 || op > 3) return arg_fail("p2p: bad count / op");
  Stream* st = resolve_stream(stream);
  if (!st) return arg_fail("no stream");
  uint32_t* flags = device_flags(st->device);
  const int nt = 32 * ((g_p2p.world + 31) / 32);
  switch (dtype) {
    case TPG_DOUBLE:
      k_p2p_allreduce<double><<<1, nt, 0, st->s>>>(g_p2p.dev_boxes, g_p2p.rank, g_p2p.world,
                                                   epoch, (double*)payload, count, op, flags);
      break;
    case TPG_INT64:
      k_p2p_allreduce<long long><<<1, nt, 0, st->s>>>(g_p2p.dev_boxes, g_p2p.rank, g_p2p.world,
                                                      epoch, (long long*)payload, count, op,
                                                      flags);
      break;
    case TPG_UINT64:
      k_p2p_allreduce<unsigned long long><<<1, nt, 0, st->s>>>(
          g_p2p.dev_boxes, g_p2p.rank, g_p2p.world, epoch, (unsigned long long*)payload, count,
          op, flags);
      break;
    case TPG_BOOL:
    case TPG_UINT8:
      k_p2p_allreduce<unsigned char><<<1, nt, 0, st->s>>>(g_p2p.dev_boxes, g_p2p.rank,
                                                          g_p2p.world, epoch,
                                                          (unsigned char*)payload, count, op,
                                                          flags);
      break;
    default:
      return arg_fail("p2p: dtype must be double, int64, uint64, uint8 or bool");
  }
  TPG_LAUNCH_CHECK("p2p allreduce");
  return TPG_OK;
}

int tpg_p2p_destroy(void) {
  for (void* p : g_p2p.opened) cudaIpcCloseMemHandle(p);
  g_p2p.opened.clear();
  if (g_p2p.dev_boxes) cudaFree(g_p2p.dev_boxes);
  if (g_p2p.mine) cudaFree(g_p2p.mine);
  g_p2p = P2pState{};
  return TPG_OK;
}

}  // extern "C"
