/*
 * tidepool_gpu.h — C ABI of the B200-native "gpu" device implementation of
 * the tidepool core module (arXiv 1810.08723, reference `tidepool`).
 *
 * Every kernel entry point below replaces one entry of the reference's
 * per-device-type function table, `backend_cpu.build_core_table()`
 * (pkg/src/tidepool/backend_cpu.py:10-27), which maps the 31 op names onto
 * the strided loops of pkg/src/tidepool/kernels.py.  The Python closures the
 * reference passes across that table (store / unpack / fn / init-step-fin)
 * are replaced here by plain descriptors: dtype wire codes (dtypes.py:69-83),
 * a byte-order flag per view (dtypes.py:357-391), an op code and a compute
 * mode (dtypes.py:25).  Plans are the reference IterPlan (tensors.py:533-595)
 * flattened into a fixed-size struct.
 *
 * Conventions
 *   - all functions return 0 on success, a negative TPG_E* code on failure;
 *     tpg_last_error() returns the message of the last failure (per thread).
 *   - pointers are device pointers from tpg_malloc unless stated otherwise.
 *   - every kernel entry is asynchronous on the given stream (0 = the
 *     device's default stream created by tpg_init).
 *   - no torch types; plain C only.
 */
#ifndef TIDEPOOL_GPU_H
#define TIDEPOOL_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TPG_MAX_DIMS 8  /* tensors.py:20 MAX_DIMS */
#define TPG_MAX_VIEWS 3

/* dtype wire codes: dtypes.py:69-83.  TPG_BF16 is an extension (no
 * reference counterpart; used by the gemm extension entry only). */
enum tpg_dtype {
  TPG_BOOL = 0, TPG_INT8 = 1, TPG_UINT8 = 2, TPG_INT16 = 3, TPG_UINT16 = 4,
  TPG_INT32 = 5, TPG_UINT32 = 6, TPG_INT64 = 7, TPG_UINT64 = 8,
  TPG_HALF = 9, TPG_FLOAT = 10, TPG_DOUBLE = 11,
  TPG_CHALF = 12, TPG_CFLOAT = 13, TPG_CDOUBLE = 14,
  TPG_BF16 = 15
};

/* compute modes: dtypes.py:25 MODES */
enum tpg_mode { TPG_STANDARD = 0, TPG_WARNING = 1, TPG_ERROR = 2, TPG_COMPLEX = 3 };

/* op codes.  Binary: kernels.py:25; unary: kernels.py:26-27;
 * reductions: kernels.py:28 (table names ops.py:516-519). */
enum tpg_binary_op { TPG_ADD = 0, TPG_SUBTRACT, TPG_MULTIPLY, TPG_DIVIDE,
                     TPG_MINIMUM, TPG_MAXIMUM };
enum tpg_unary_op { TPG_NEGATE = 0, TPG_ABSOLUTE, TPG_SQRT, TPG_EXP, TPG_LOG,
                    TPG_SIN, TPG_COS, TPG_ASIN, TPG_ACOS, TPG_CONJ,
                    TPG_IDENTITY /* the `copy` entry: ops.py:681 */ };
enum tpg_reduce_op { TPG_RSUM = 0, TPG_RPRODUCT, TPG_RMIN, TPG_RMAX, TPG_RANY,
                     TPG_RALL, TPG_RNORM };

/* status flag bits (ops.py:27-38, kernels.py:22-23, dtypes.py:246-250) */
#define TPG_FLAG_DOMAIN      1u  /* "domain-violation" (unary real domain) */
#define TPG_FLAG_INT_DIV0    2u  /* "integer-division-by-zero" */
#define TPG_FLAG_CAST_LOSS   4u  /* CastContext.domain_loss (store-side) */

/* error codes */
#define TPG_OK            0
#define TPG_E_CUDA       -1
#define TPG_E_ALLOC      -2
#define TPG_E_ARG        -3
#define TPG_E_UNSUPPORTED -4
#define TPG_E_NCCL       -5

/* IterPlan (tensors.py:533-567): extents of the merged axes (axis 0 is the
 * fastest for view 0, the destination) and signed byte strides per view.
 * ndim == 0 is a single element; an extent of 0 makes an empty plan. */
typedef struct tpg_plan {
  int32_t ndim;
  int32_t nviews;
  int64_t extent[TPG_MAX_DIMS];
  int64_t stride[TPG_MAX_VIEWS][TPG_MAX_DIMS];
} tpg_plan;

/* One view: storage base pointer + byte offset of the first element
 * (the reference's `bases` tuple, ops.py:280), the dtype and the byte order
 * (Tensor.byteorder).  base == NULL means an immediate scalar held in imm
 * (already cast to `dtype` and packed in `big_endian` order); this is the
 * by-value form of ops._materialize_scalar (ops.py:105-107). */
typedef struct tpg_operand {
  void* base;
  int64_t offset;
  int32_t dtype;
  int32_t big_endian;
  uint64_t imm[2];
} tpg_operand;

typedef struct tpg_device_props {
  int32_t sm_count;
  int32_t cc_major, cc_minor;
  int64_t total_mem;
  int64_t free_mem;
  int32_t l2_bytes;
  char name[128];
} tpg_device_props;

typedef void* tpg_stream;
typedef void* tpg_event;

/* ---------------------------------------------------------------- runtime */
int tpg_init(void);
int tpg_device_count(int* count);
int tpg_device_props_get(int device, tpg_device_props* props);
const char* tpg_last_error(void);
const char* tpg_version(void);

/* Stream-ordered caching allocator (devices.py:149-160 allocate/release). */
int tpg_malloc(int device, size_t nbytes, void** ptr);
int tpg_free(int device, void* ptr, tpg_stream stream);  /* deferred past stream */
int tpg_malloc_on(tpg_stream stream, size_t nbytes, void** ptr);  /* ordered on stream */
int tpg_host_alloc(size_t nbytes, void** ptr);            /* pinned host memory */
int tpg_host_free(void* ptr);
int tpg_mem_stats(int device, int64_t* in_use, int64_t* cached, int64_t* n_alloc);
int tpg_empty_cache(int device);

/* Streams (devices.py:47-101 Stream). */
int tpg_default_stream(int device, tpg_stream* stream);
int tpg_stream_create(int device, tpg_stream* stream);
int tpg_stream_destroy(tpg_stream stream);
int tpg_stream_sync(tpg_stream stream);
int tpg_stream_wait(tpg_stream waiter, tpg_stream signaller);
int tpg_event_create(tpg_event* ev);
int tpg_event_destroy(tpg_event ev);
int tpg_event_record(tpg_event ev, tpg_stream stream);
int tpg_event_sync(tpg_event ev);
int tpg_event_elapsed(tpg_event start, tpg_event stop, float* ms);

/* Byte transfers (Storage snapshots, host staging, peer copies). */
int tpg_memcpy_h2d(void* dst, const void* src, size_t n, tpg_stream stream);
int tpg_memcpy_d2h(void* dst, const void* src, size_t n, tpg_stream stream);
int tpg_memcpy_d2d(void* dst, const void* src, size_t n, tpg_stream stream);
int tpg_memset(void* dst, int value, size_t n, tpg_stream stream);
/* pitched 2-D copy (any direction; host memory should be pinned to overlap) */
int tpg_memcpy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                 size_t height, tpg_stream stream);

/* Sticky status word (ops._status, ops.py:27-38) per device, OR-ed by
 * kernels.  tpg_flags_get / tpg_flags_clear wait for the whole device;
 * tpg_flags_take atomically reads-and-clears it in `stream` order and waits
 * for that stream only (the drop-in's Stream.sync, devices.py:93-98). */
int tpg_flags_get(int device, uint32_t* flags);
int tpg_flags_clear(int device);
int tpg_flags_take(tpg_stream stream, uint32_t* flags);

/* Host-addressable device storage for the drop-in plugin: the reference
 * object model reads and writes storage bytes on the host (storage.py:38-39,
 * tensors.py:313-318), so its gpu buffers are CUDA managed allocations
 * (preferred location: the GPU).  Devices.allocate (devices.py:149-160). */
int tpg_malloc_managed(int device, size_t nbytes, void** ptr);
int tpg_free_managed(void* ptr);
/* completion tracking for recycled blocks: 0 = complete, 1 = pending */
int tpg_event_create_untimed(tpg_event* ev);
int tpg_event_query(tpg_event ev);
/* completion words (the drop-in's block cache checks reuse without a
 * cudaEventQuery per allocation): a 64-bit word in pinned, device-mapped
 * host memory that tpg_stream_mark sets to `value` in stream order, after
 * all earlier work of the stream has completed (cuStreamWriteValue64).
 * tpg_stream_mark returns TPG_E_UNSUPPORTED where stream memory operations
 * are unavailable (the caller then uses events). */
int tpg_mark_word_create(uint64_t** word);
int tpg_mark_word_free(uint64_t* word);
int tpg_stream_mark(tpg_stream stream, uint64_t* word, uint64_t value);

/* Peer access between all visible device pairs that support it (NVLink /
 * NVSwitch); *enabled = number of (a, b) pairs enabled. */
int tpg_enable_peer_all(int* enabled);

/* CUDA graphs: capture the work enqueued on `stream` between begin and end
 * (thread-local capture mode), replay it with one launch. */
int tpg_graph_begin(tpg_stream stream);
int tpg_graph_end(tpg_stream stream, void** graph_exec);
int tpg_graph_launch(void* graph_exec, tpg_stream stream);
int tpg_graph_destroy(void* graph_exec);

/* Measurement helper: write then re-read `n` bytes of `scratch` (> L2) on
   `stream`, leaving the L2 full of clean unrelated lines. */
int tpg_l2_flush(void* scratch, size_t n, tpg_stream stream);
/* Measurement helper: hold `stream` until tpg_gate_release() so a batch of
 * timed steps is fully enqueued before the device starts on it. */
int tpg_gate_arm(tpg_stream stream);
int tpg_gate_release(void);

/* ---------------------------------------------------------------- kernels */
/* binary ×6: kernels.binary_elementwise (kernels.py:213-248), called by
 * ops.binary_elementwise (ops.py:282-283).  plan has 3 views (d, a, b).
 * compute = widen_for_compute(result dtype) code (dtypes.py:190-196); it
 * selects the int / float / complex scalar semantics of binary_scalar_fn
 * (kernels.py:50-81).  Operand dtypes may differ from `compute`: each
 * operand is converted on load exactly as ops._prepare would (ops.py:121-142),
 * so mixed-dtype operations need no materialized intermediate. */
int tpg_binary(tpg_stream stream, int op, const tpg_plan* plan,
               const tpg_operand* d, const tpg_operand* a, const tpg_operand* b,
               int compute, int mode);

/* unary ×10 and copy: kernels.unary_elementwise (kernels.py:275-302);
 * ops.py:384-385 and ops._run_copy (ops.py:683-684, op = TPG_IDENTITY).
 * force_complex: ops.py:340-352 "complex" mode promotion. */
int tpg_unary(tpg_stream stream, int op, const tpg_plan* plan,
              const tpg_operand* d, const tpg_operand* a,
              int compute, int mode, int force_complex);

/* copy/astype convenience = tpg_unary(TPG_IDENTITY) (ops._run_copy). */
int tpg_copy(tpg_stream stream, const tpg_plan* plan, const tpg_operand* d,
             const tpg_operand* a, int mode);

/* reductions ×7: kernels.reduce_strided (kernels.py:305-320) with the
 * accumulators of ops._reduction_acc (ops.py:522-556).  outer has 2 views
 * (dest, src base), inner has 1 view (reduced src axes). */
int tpg_reduce(tpg_stream stream, int op, double p, const tpg_plan* outer,
               const tpg_plan* inner, const tpg_operand* d,
               const tpg_operand* a, int compute, int mode);

/* matmul: kernels.matmul (kernels.py:323-340), ops.matmul (ops.py:633-635).
 * Strides are (row, col) byte strides.  compute = widen(result dtype). */
int tpg_matmul(tpg_stream stream, const tpg_operand* d, const int64_t d_strides[2],
               const tpg_operand* a, const int64_t a_strides[2],
               const tpg_operand* b, const int64_t b_strides[2],
               int64_t m, int64_t n, int64_t k, int compute, int mode);

/* Extension (no reference op): batched gemm, batch strides in bytes. */
int tpg_matmul_batched(tpg_stream stream, int64_t batch,
                       const tpg_operand* d, const int64_t d_strides[3],
                       const tpg_operand* a, const int64_t a_strides[3],
                       const tpg_operand* b, const int64_t b_strides[3],
                       int64_t m, int64_t n, int64_t k, int compute, int mode);

/* Extension: fused elementwise chain x = op_i(x, s_i)
 * (or op_i(s_i, x) with scalar_first) over one source view in one pass.
 * Each step has the reference binary semantics with a by-value scalar
 * (kernels.py:50-81, 213-248): compute in `compute` (widen_for_compute of
 * the step's result dtype), round once to `dtype`.  The last step's dtype
 * is the destination dtype.  plan has 2 views (d, a).  Bit-identical to
 * running the steps as separate tpg_binary calls. */
typedef struct tpg_chain_step {
  int32_t op;            /* TPG_ADD .. TPG_MAXIMUM */
  int32_t dtype;         /* the step's result (rounding) dtype */
  int32_t compute;       /* widen_for_compute(dtype) */
  int32_t scalar_first;  /* 1: op(s, x), 0: op(x, s) */
  int32_t scalar_dtype;  /* dtype of `scalar` */
  int32_t reserved;
  uint8_t scalar[16];    /* element bytes, little-endian */
} tpg_chain_step;
int tpg_chain(tpg_stream stream, const tpg_plan* plan, const tpg_operand* d,
              const tpg_operand* a, int nsteps, const tpg_chain_step* steps, int mode);
int tpg_chain_check(tpg_stream stream, const tpg_plan* plan, const tpg_operand* d,
                    const tpg_operand* a, int nsteps, const tpg_chain_step* steps, int mode);

/* fill: kernels.fill (kernels.py:343-352); `value` is the packed element
 * (dtype size bytes, already cast and byte-ordered, ops.py:752-758). */
int tpg_fill(tpg_stream stream, const tpg_plan* plan, const tpg_operand* d,
             const void* value, int32_t size);

/* arange: kernels.arange_fill (kernels.py:377-381), ops.arange (ops.py:773-784). */
int tpg_arange(tpg_stream stream, const tpg_plan* plan, const tpg_operand* d);

/* byteswap: kernels.byteswap_inplace (kernels.py:355-357), tensors.py:615-631. */
int tpg_byteswap(tpg_stream stream, const tpg_plan* plan, const tpg_operand* d);

/* gather: kernels.gather (kernels.py:360-363): byte-exact moves of `size`
 * bytes for n (dst_off, src_off) pairs; `pairs` is a HOST array of 2n int64. */
int tpg_gather(tpg_stream stream, void* dst_base, const void* src_base,
               const int64_t* pairs, int64_t n, int32_t size);

/* gather by plan (descriptor fast path of tensors._raw_gather, §8f-3):
 * byte copy along a 2-view plan (dst, src) of `size`-byte elements. */
int tpg_gather_plan(tpg_stream stream, const tpg_plan* plan, void* dst_base,
                    int64_t dst_off, const void* src_base, int64_t src_off,
                    int32_t size);

/* scatter: kernels.scatter (kernels.py:366-369): value moves with cast;
 * pairs are host (dst_off, src_off); duplicates: last pair wins. */
int tpg_scatter(tpg_stream stream, const int64_t* pairs, int64_t n,
                const tpg_operand* d, const tpg_operand* s, int mode);

/* scatter_fill: kernels.scatter_fill (kernels.py:372-374). */
int tpg_scatter_fill(tpg_stream stream, const int64_t* offsets, int64_t n,
                     void* d_base, const void* value, int32_t size);

/* ----------------------------------------------------------- multi-GPU */
/* NCCL plumbing for the full-reduction finish.  The unique id
 * (128 bytes) is produced on rank 0 and shared by the caller. */
int tpg_nccl_get_unique_id(void* id128);
int tpg_nccl_init(int device, int nranks, int rank, const void* id128);
int tpg_nccl_allreduce(tpg_stream stream, void* buf, int64_t count,
                       int dtype, int op /*0 sum,1 prod,2 max,3 min*/);
int tpg_nccl_destroy(void);
/* communicator size and this process's rank, as NCCL sees them */
int tpg_nccl_info(int* nranks, int* rank);

/* Sharded-reduction finish over NVLink peer memory, no NCCL:
 * init exports this rank's mailbox as a 64-byte IPC handle; connect opens
 * every peer's mailbox from the world's handles (world x 64 bytes, rank
 * order); allreduce enqueues ONE exchange kernel on `stream` that combines
 * the `count` (<= 2) payload elements of every rank in rank order, in place
 * (dtype double / int64 / uint64 / uint8 / bool; op 0 sum, 1 prod, 2 max,
 * 3 min; `epoch` increases by one per call, identically on every rank).  A
 * peer that never arrives (~4 s) sets bit 31 of the status word. */
#define TPG_FLAG_P2P_TIMEOUT 0x80000000u
int tpg_p2p_init(int device, int rank, int world, void* handle64);
int tpg_p2p_connect(const void* handles);
int tpg_p2p_allreduce(tpg_stream stream, void* payload, int count, int dtype, int op,
                      unsigned long long epoch);
int tpg_p2p_destroy(void);
/* The full sum of a unit-stride f32 / f64 range with the cross-rank finish
 * FUSED into the reduction kernel: its final block exchanges the rank's
 * double-double partial with every peer's mailbox and merges the world's in
 * rank order -- one kernel for compute + collective (d: the 0-dim result).
 * TPG_E_UNSUPPORTED, nothing launched, for other layouts. */
int tpg_reduce_sum_p2p(tpg_stream stream, const tpg_plan* outer, const tpg_plan* inner,
                       const tpg_operand* d, const tpg_operand* a, unsigned long long epoch);
/* min / max with the fused finish (NaN iff the tensor's first element is
 * NaN, ties keep the earliest; index_base = global plan index of this
 * rank's first element, 0 on the rank holding element 0) */
int tpg_reduce_minmax_p2p(tpg_stream stream, int op, const tpg_plan* outer, const tpg_plan* inner,
                          const tpg_operand* d, const tpg_operand* a, unsigned long long epoch,
                          int64_t index_base);
/* the same for the 2-norm: ranks exchange sum |x|^2, one root at the end */
int tpg_reduce_norm2_p2p(tpg_stream stream, const tpg_plan* outer, const tpg_plan* inner,
                         const tpg_operand* d, const tpg_operand* a, unsigned long long epoch);

/* Sharded min/max finish: pack a rank's local extreme
 * (payload slot 0: double for float sources, kind 0; int64 for signed
 * integers, kind 1; uint64 bits for unsigned, kind 2) into an order key
 * for ONE max all-reduce of the 2-slot payload, slot 1 = the first-element
 * NaN flag (ops.py:533-544; `first` = the tensor's element 0 on the rank
 * holding it, else NULL); unpack maps the reduced key back (NaN when the
 * flag is set).  has = 0: the rank holds no elements. */
int tpg_shard_pack(tpg_stream stream, int is_max, int kind, int has, void* payload,
                   const void* first, int first_dtype, int first_big_endian);
int tpg_shard_unpack(tpg_stream stream, int is_max, int kind, void* payload);

#ifdef __cplusplus
}
#endif
#endif /* TIDEPOOL_GPU_H */
