// tpg_internal.h — shared host-side plumbing for the C ABI implementation.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/tidepool_gpu.h"

namespace tpg {

struct Stream {
  int device;
  cudaStream_t s;
  // zeroed arrival counters for single-pass (last-block-finalises)
  // reductions; every kernel that uses them leaves them zero again
  uint32_t* counters = nullptr;
  int64_t ncounters = 0;
};

// cuTensorMapEncodeTiled from the driver (nullptr if unavailable); cast
// to PFN_cuTensorMapEncodeTiled_v12000 by the caller
void* tensor_map_encoder();

// at least n zeroed counters, stream-ordered on st
uint32_t* stream_counters(Stream* st, int64_t n);

void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
int arg_fail(const std::string& msg);

// Resolve a tpg_stream (NULL = default stream of the current device) and
// make its device current.
Stream* resolve_stream(tpg_stream s);
int sm_count(int device);
uint32_t* device_flags(int device);  // device-resident sticky status word

// peer-memory mailboxes (tpg_p2p.cu): Slot[2 parities][P2P_MAX_RANKS] per rank
constexpr int P2P_MAX_RANKS = 64;
struct alignas(32) P2pSlot {
  uint64_t payload[2];
  unsigned long long epoch;
  uint64_t pad;
};
// device array of every rank's mailbox (nullptr when not connected)
P2pSlot** p2p_boxes(int* rank, int* world);

#define TPG_CUDA_CHECK(expr)                                 \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) return ::tpg::cuda_fail(_e, #expr); \
  } while (0)

#define TPG_LAUNCH_CHECK(what)                                 \
  do {                                                         \
    cudaError_t _e = cudaGetLastError();                       \
    if (_e != cudaSuccess) return ::tpg::cuda_fail(_e, what);  \
  } while (0)

}  // namespace tpg
