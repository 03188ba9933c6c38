/* tpg_pyfast.c -- CPython extension: the drop-in plugin's per-call host
 * machinery in C (tidepool_plugin.py imports it as _tpg_pyfast).
 *
 * The reference allocates a fresh storage for every op result and every
 * implicit dtype conversion (tensors.tensor_create -> Device.allocate,
 * tensors.py:179-188; ops._dtype_convert, ops.py:121-124) and releases it
 * when the last tensor view drops (storage.py:48-70).  In Python the gpu
 * device's allocate + release cost ~9 us per storage on the box
 * (profiles/r02s_plugin_cost_probe.txt); here they are a few hundred ns.
 *
 *   BlockPool(fns, blocks, lazy, lazy_by_src, cache_bytes, max_pending)
 *     fns = addresses of tpg_malloc_managed, tpg_free_managed,
 *           tpg_event_create_untimed, tpg_event_record, tpg_event_query,
 *           tpg_event_sync (include/tidepool_gpu.h)
 *     .allocate(device, nbytes) -> DevBuf
 *     .add_stream(device, handle)    streams whose completion gates reuse
 *     .bump()                        a new launch epoch (rt.current)
 *     .trim(device, keep_bytes)
 *     .stats() -> dict
 *   DevBuf: writable 1-D buffer (format "B") over a managed block;
 *     .ptr .nbytes .cap .device; freed blocks go back to the pool.
 *
 * Reuse rule (same as the Python version it replaces): a freed block
 * carries one completion event per stream of its device, recorded at
 * release (shared by all blocks released in the same launch epoch); it is
 * handed out again only once those events completed, never waiting while
 * fewer than max_pending blocks of its size class are in flight.
 * Everything runs under the GIL; blocking event waits release it.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/tidepool_gpu.h"

typedef int (*f_malloc_managed)(int, size_t, void**);
typedef int (*f_free_managed)(void*);
typedef int (*f_ev_create)(void**);
typedef int (*f_ev_record)(void*, void*);
typedef int (*f_ev_query)(void*);
typedef int (*f_ev_sync)(void*);
typedef int (*f_mark_create)(uint64_t**);
typedef int (*f_mark)(void*, uint64_t*, uint64_t);

#define MAX_DEV 64

#include <time.h>
/* host-time counters of the C paths (pool allocate / release, binary and
 * copy entries): exposed by counters() so the per-op host cost can be split
 * exactly (scripts/plugin_cost_probe.py) */
static long long T_alloc, T_release, T_binary, T_copy, T_launch;
static inline long long now_ns(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (long long)ts.tv_sec * 1000000000ll + ts.tv_nsec;
}

typedef struct Marker {
  int armed;     /* recorded on its stream (a pending marker collects releases first) */
  void* ev;      /* event marker (NULL for a completion-word marker) */
  uint64_t wval; /* completion-word marker: done once the stream's word >= wval */
  long refs;
  uint64_t seq; /* launch epoch it was recorded in */
  int dev, sidx; /* owning stream */
} Marker;

typedef struct {
  void* handle;
  Marker* marker;    /* newest marker recorded on the stream (NULL once freed) */
  uint64_t marker_seq;
  uint64_t done_seq; /* every marker of this stream with seq <= done_seq completed */
  volatile uint64_t* word; /* completion word (tpg_stream_mark), or NULL: events */
  uint64_t wnext;
  int wdisabled; /* tpg_stream_mark failed once: new markers use events */
  Marker* pending; /* unrecorded marker the blocks released since the last record share */
  int npending;
} StreamRec;

typedef struct {
  void* ptr;
  int nev;
  Marker** evs;
} Entry;

typedef struct SizeClass {
  int dev;
  size_t cap;
  Entry* v;  /* FIFO: [head, n) */
  size_t head, n, alloc;
  struct SizeClass* next;
} SizeClass;

#define NBUCKET 1024

typedef struct {
  PyObject_HEAD
  f_malloc_managed malloc_managed;
  f_free_managed free_managed;
  f_ev_create ev_create;
  f_ev_record ev_record;
  f_ev_query ev_query;
  f_ev_sync ev_sync;
  f_mark_create mark_create; /* optional (NULL: event markers only) */
  f_mark mark;
  PyObject* blocks;       /* dict ptr -> (device, cap) */
  PyObject* lazy;         /* dict dst ptr -> record */
  PyObject* lazy_by_src;  /* dict src ptr -> set */
  long long cache_limit;
  int max_pending;
  uint64_t seq;
  StreamRec* streams[MAX_DEV];
  int nstreams[MAX_DEV];
  long long cached[MAX_DEV];
  SizeClass* bucket[NBUCKET];
  void** evpool;
  size_t nevpool, aevpool;
  long long n_alloc, n_reuse, n_new, n_wait, n_release, n_trim;
} BlockPool;

typedef struct {
  PyObject_HEAD
  void* ptr;
  Py_ssize_t nbytes;
  size_t cap;
  int dev;
  BlockPool* pool;
  PyObject* weakreflist;
  PyObject* dict;
} DevBuf;

static PyTypeObject BlockPoolType;
static PyTypeObject DevBufType;
static PyTypeObject LazyRecordType;
static PyObject* AllocError;  /* set by the plugin: the reference's AllocationError */

/* a copy record's plan and source operand, packed by entries_copy (the
 * record's `cpack` bytes) so the binary entry reads them with one lookup */
typedef struct {
  int64_t ne, sbase, soff, sdt, sbig;
  int64_t E[TPG_MAX_DIMS], T[TPG_MAX_DIMS], S[TPG_MAX_DIMS];
} CopyPack;

/* A recorded lossless copy (tidepool_plugin._Lazy derives from this):
 * C fields, visible to Python as attributes, filled by the C copy entry
 * without attribute calls and read by the C binary entry directly. */
#include <structmember.h>
typedef struct {
  PyObject_HEAD
  PyObject *plan, *stream, *keep, *src_dtype, *dst_dtype, *src_order, *dst_ptr, *src_ptr;
  PyObject *cext, *cdst, *csrc;
  long long device, ddt, dbig, sbase, soff, sdt, sbig;
  int has_pack;
  CopyPack pack;
} LazyRecord;

static size_t size_class(size_t n) {
  if (n <= ((size_t)1 << 20)) return ((n ? n : 1) + 511) & ~(size_t)511;
  return (n + ((size_t)2 << 20) - 1) & ~(((size_t)2 << 20) - 1);
}

static SizeClass* find_class(BlockPool* p, int dev, size_t cap, int create) {
  size_t h = ((cap >> 9) * 31u + (size_t)dev) % NBUCKET;
  for (SizeClass* c = p->bucket[h]; c; c = c->next)
    if (c->dev == dev && c->cap == cap) return c;
  if (!create) return NULL;
  SizeClass* c = (SizeClass*)calloc(1, sizeof(SizeClass));
  if (!c) return NULL;
  c->dev = dev;
  c->cap = cap;
  c->next = p->bucket[h];
  p->bucket[h] = c;
  return c;
}

static void unref_markers(BlockPool* p, Entry* e) {
  for (int i = 0; i < e->nev; ++i) {
    Marker* m = e->evs[i];
    if (--m->refs > 0) continue;
    /* last user: detach from its stream and recycle the event */
    for (int d = 0; d < MAX_DEV; ++d)
      for (int s = 0; s < p->nstreams[d]; ++s) {
        if (p->streams[d][s].marker == m) p->streams[d][s].marker = NULL;
        if (p->streams[d][s].pending == m) {
          p->streams[d][s].pending = NULL;
          p->streams[d][s].npending = 0;
        }
      }
    if (m->ev) {
      if (p->nevpool == p->aevpool) {
        size_t na = p->aevpool ? 2 * p->aevpool : 64;
        void** nv = (void**)realloc(p->evpool, na * sizeof(void*));
        if (nv) {
          p->evpool = nv;
          p->aevpool = na;
        }
      }
      if (p->nevpool < p->aevpool) p->evpool[p->nevpool++] = m->ev;
    }
    free(m);
  }
  free(e->evs);
  e->evs = NULL;
  e->nev = 0;
}

/* Completion of a freed block's markers.  Events on one stream complete in
 * order, so a completed marker proves every older marker of its stream
 * complete: the stream's NEWEST marker is queried first (one query then
 * usually clears every pending block of the device -- the host runs behind
 * the GPU in steady state), and a watermark makes repeat checks free. */
static int arm_pending(BlockPool* p, int dev, int sidx);
static void arm_device(BlockPool* p, int dev);

static int entry_done(BlockPool* p, Entry* e) {
  for (int i = 0; i < e->nev; ++i) {
    Marker* m = e->evs[i];
    StreamRec* st = &p->streams[m->dev][m->sidx];
    if (!m->armed) return 0; /* not recorded yet */
    if (m->wval) { /* completion word: a host memory read, no CUDA call */
      if (*st->word >= m->wval) continue;
      return 0;
    }
    if (m->seq <= st->done_seq && st->done_seq != (uint64_t)-1) continue;
    Marker* nw = st->marker;
    if (nw && nw != m && nw->seq > m->seq && p->ev_query(nw->ev) == 0) {
      st->done_seq = nw->seq;
      continue;
    }
    if (p->ev_query(m->ev) != 0) return 0;
    if (st->done_seq == (uint64_t)-1 || m->seq > st->done_seq) st->done_seq = m->seq;
  }
  return 1;
}

static void entry_wait(BlockPool* p, Entry* e) {
  for (int i = 0; i < e->nev; ++i)
    if (!e->evs[i]->armed) arm_pending(p, e->evs[i]->dev, e->evs[i]->sidx);
  Py_BEGIN_ALLOW_THREADS
  for (int i = 0; i < e->nev; ++i) {
    Marker* m = e->evs[i];
    if (!m->armed) continue; /* recording failed (no event could be created) */
    if (m->wval) {
      volatile uint64_t* w = p->streams[m->dev][m->sidx].word;
      while (*w < m->wval) {
        struct timespec ts = {0, 20000};
        nanosleep(&ts, NULL);
      }
    } else {
      p->ev_sync(m->ev);
    }
  }
  Py_END_ALLOW_THREADS
}

static int blocks_set(BlockPool* p, void* ptr, int dev, size_t cap) {
  PyObject* k = PyLong_FromVoidPtr(ptr);
  PyObject* v = Py_BuildValue("(in)", dev, (Py_ssize_t)cap);
  int rc = (k && v) ? PyDict_SetItem(p->blocks, k, v) : -1;
  Py_XDECREF(k);
  Py_XDECREF(v);
  return rc;
}

static void blocks_del(BlockPool* p, void* ptr) {
  PyObject* k = PyLong_FromVoidPtr(ptr);
  if (!k) {
    PyErr_Clear();
    return;
  }
  if (PyDict_DelItem(p->blocks, k) < 0) PyErr_Clear();
  /* a pending lazy copy INTO this block is dead with it (a pending copy
   * keeps its source alive, so only destination records die here):
   * tidepool_plugin._Runtime._drop_lazy_locked, in C */
  PyObject* rec = PyDict_GetItemWithError(p->lazy, k);
  if (rec) {
    Py_INCREF(rec);
    if (PyDict_DelItem(p->lazy, k) < 0) PyErr_Clear();
    PyObject* src = PyObject_TypeCheck(rec, &LazyRecordType) ? ((LazyRecord*)rec)->src_ptr : NULL;
    if (src) Py_INCREF(src);
    else src = PyObject_GetAttrString(rec, "src_ptr");
    PyObject* set = src ? PyDict_GetItemWithError(p->lazy_by_src, src) : NULL;
    if (set && PySet_Check(set)) {
      if (PySet_Discard(set, k) < 0) PyErr_Clear();
      if (PySet_GET_SIZE(set) == 0 && PyDict_DelItem(p->lazy_by_src, src) < 0) PyErr_Clear();
    }
    Py_XDECREF(src);
    Py_DECREF(rec);
  }
  PyErr_Clear();
  Py_DECREF(k);
}

static void trim_dev(BlockPool* p, int dev, long long keep) {
  for (int h = 0; h < NBUCKET && p->cached[dev] > keep; ++h)
    for (SizeClass* c = p->bucket[h]; c && p->cached[dev] > keep; c = c->next) {
      if (c->dev != dev) continue;
      while (c->head < c->n && p->cached[dev] > keep) {
        Entry e = c->v[c->head++];  /* copied: the array may move while the GIL is released */
        entry_wait(p, &e);
        unref_markers(p, &e);
        p->free_managed(e.ptr);
        p->cached[dev] -= (long long)c->cap;
        p->n_trim++;
      }
      if (c->head == c->n) c->head = c->n = 0;
    }
}

/* a block of `cap` bytes on `dev`: recycled when its last GPU use is done */
static void* take(BlockPool* p, int dev, size_t cap) {
  SizeClass* c = find_class(p, dev, cap, 0);
  if (c && c->n > c->head) {
    size_t live = c->n - c->head;
    for (size_t i = c->head; i < c->n; ++i) {
      if (entry_done(p, &c->v[i])) {
        Entry e = c->v[i];
        memmove(&c->v[i], &c->v[i + 1], (c->n - i - 1) * sizeof(Entry));
        c->n--;
        if (c->head == c->n) c->head = c->n = 0;
        unref_markers(p, &e);
        p->cached[dev] -= (long long)cap;
        p->n_reuse++;
        return e.ptr;
      }
    }
    /* nothing reusable: record the device's pending markers so the blocks
     * waiting on them become reusable for the next allocations */
    arm_device(p, dev);
    if ((int)live >= p->max_pending) {
      Entry e = c->v[c->head++];
      if (c->head == c->n) c->head = c->n = 0;
      entry_wait(p, &e);
      unref_markers(p, &e);
      p->cached[dev] -= (long long)cap;
      p->n_wait++;
      return e.ptr;
    }
  }
  return NULL;
}

/* ---------------------------------------------------------------- DevBuf */

static void release_block_(BlockPool* p, void* ptr, size_t cap, int dev);
static void release_block(BlockPool* p, void* ptr, size_t cap, int dev) {
  const long long t0 = now_ns();
  release_block_(p, ptr, cap, dev);
  T_release += now_ns() - t0;
}
/* Record a stream's pending marker (completion word, else event): every
 * block attached to it was released before this point in stream order, so
 * it completes only after their last GPU use. */
static int arm_pending(BlockPool* p, int dev, int sidx) {
  StreamRec* st = &p->streams[dev][sidx];
  Marker* m = st->pending;
  if (!m) return 0;
  m->seq = p->seq;
  if (st->word && !st->wdisabled) {
    m->wval = st->wnext + 1;
    if (p->mark(st->handle, (uint64_t*)st->word, m->wval) == 0) {
      st->wnext = m->wval;
    } else {
      m->wval = 0; /* no stream memory ops: events from now on */
      st->wdisabled = 1;
    }
  }
  if (!m->wval) {
    if (p->nevpool) {
      m->ev = p->evpool[--p->nevpool];
    } else if (p->ev_create(&m->ev) != 0) {
      return -1; /* stays pending: its blocks are not reusable yet */
    }
    p->ev_record(m->ev, st->handle);
  }
  m->armed = 1;
  st->marker = m;
  st->marker_seq = p->seq;
  st->pending = NULL;
  st->npending = 0;
  return 0;
}

static void arm_device(BlockPool* p, int dev) {
  for (int s = 0; s < p->nstreams[dev]; ++s) arm_pending(p, dev, s);
}

/* releases share a stream's pending marker; it is recorded once ARM_AT
 * blocks wait on it, or when an allocation / wait needs it (one stream
 * memory op per ARM_AT releases instead of one per launch epoch; the pool
 * keeps the few extra blocks in flight this needs) */
#define ARM_AT 4

static void release_block_(BlockPool* p, void* ptr, size_t cap, int dev) {
  p->n_release++;
  blocks_del(p, ptr);
  SizeClass* c = find_class(p, dev, cap, 1);
  int ns = p->nstreams[dev];
  Entry e = {ptr, 0, NULL};
  if (ns) {
    e.evs = (Marker**)malloc(sizeof(Marker*) * ns);
    for (int s = 0; e.evs && s < ns; ++s) {
      StreamRec* st = &p->streams[dev][s];
      if (!st->pending) {
        Marker* m = (Marker*)calloc(1, sizeof(Marker));
        if (!m) break;
        m->dev = dev;
        m->sidx = s;
        st->pending = m;
      }
      st->pending->refs++;
      e.evs[e.nev++] = st->pending;
      if (++st->npending >= ARM_AT) arm_pending(p, dev, s);
    }
  }
  if (!c) { /* out of host memory: drop the block */
    entry_wait(p, &e);
    unref_markers(p, &e);
    p->free_managed(ptr);
    return;
  }
  if (c->n == c->alloc) {
    if (c->head > 0) {
      memmove(c->v, c->v + c->head, (c->n - c->head) * sizeof(Entry));
      c->n -= c->head;
      c->head = 0;
    }
    if (c->n == c->alloc) {
      size_t na = c->alloc ? 2 * c->alloc : 8;
      Entry* nv = (Entry*)realloc(c->v, na * sizeof(Entry));
      if (!nv) {
        unref_markers(p, &e);
        p->free_managed(ptr);
        return;
      }
      c->v = nv;
      c->alloc = na;
    }
  }
  c->v[c->n++] = e;
  p->cached[dev] += (long long)cap;
  if (p->cached[dev] > p->cache_limit) trim_dev(p, dev, p->cache_limit / 2);
}

static int devbuf_getbuffer(PyObject* o, Py_buffer* view, int flags) {
  DevBuf* b = (DevBuf*)o;
  return PyBuffer_FillInfo(view, o, b->ptr ? b->ptr : (void*)b, b->nbytes, 0, flags);
}

static PyBufferProcs devbuf_as_buffer = {devbuf_getbuffer, NULL};

static Py_ssize_t devbuf_len(PyObject* o) { return ((DevBuf*)o)->nbytes; }

static PySequenceMethods devbuf_as_seq = {devbuf_len};

static void devbuf_dealloc(DevBuf* b) {
  PyObject_GC_UnTrack(b);
  if (b->weakreflist) PyObject_ClearWeakRefs((PyObject*)b);
  PyObject *et, *ev, *tb;
  PyErr_Fetch(&et, &ev, &tb);
  if (b->pool && b->ptr) release_block(b->pool, b->ptr, b->cap, b->dev);
  PyErr_Restore(et, ev, tb);
  Py_CLEAR(b->dict);
  Py_CLEAR(b->pool);
  Py_TYPE(b)->tp_free((PyObject*)b);
}

static int devbuf_traverse(DevBuf* b, visitproc visit, void* arg) {
  Py_VISIT(b->dict);
  Py_VISIT(b->pool);
  return 0;
}

static int devbuf_clear(DevBuf* b) {
  Py_CLEAR(b->dict);
  return 0;
}

static PyObject* devbuf_get_ptr(DevBuf* b, void* c) { return PyLong_FromVoidPtr(b->ptr); }
static PyObject* devbuf_get_cap(DevBuf* b, void* c) { return PyLong_FromSize_t(b->cap); }
static PyObject* devbuf_get_dev(DevBuf* b, void* c) { return PyLong_FromLong(b->dev); }
static PyObject* devbuf_get_n(DevBuf* b, void* c) { return PyLong_FromSsize_t(b->nbytes); }

static PyGetSetDef devbuf_getset[] = {
    {"ptr", (getter)devbuf_get_ptr, NULL, "device (managed) address", NULL},
    {"cap", (getter)devbuf_get_cap, NULL, "block capacity (size class)", NULL},
    {"device", (getter)devbuf_get_dev, NULL, "device index", NULL},
    {"nbytes", (getter)devbuf_get_n, NULL, "storage size in bytes", NULL},
    {NULL}};

/* ------------------------------------------------------------- BlockPool */

static int pool_init(BlockPool* p, PyObject* args, PyObject* kw) {
  PyObject *fns, *blocks, *lazy, *lbs;
  long long limit;
  int maxp;
  if (!PyArg_ParseTuple(args, "OO!O!O!Li", &fns, &PyDict_Type, &blocks, &PyDict_Type, &lazy,
                        &PyDict_Type, &lbs, &limit, &maxp))
    return -1;
  const Py_ssize_t nf = PyTuple_Check(fns) ? PyTuple_GET_SIZE(fns) : 0;
  if (nf != 6 && nf != 8) {
    PyErr_SetString(PyExc_TypeError, "fns: 6 (or 8, with the completion-word pair) addresses");
    return -1;
  }
  void* f[8] = {0};
  for (int i = 0; i < nf; ++i) {
    PyObject* a = PyTuple_GET_ITEM(fns, i);
    f[i] = a == Py_None ? NULL : PyLong_AsVoidPtr(a);
    if (!f[i] && (i < 6 || PyErr_Occurred())) {
      if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "null function address");
      return -1;
    }
  }
  p->mark_create = (f_mark_create)f[6];
  p->mark = (f_mark)f[7];
  if (!p->mark) p->mark_create = NULL;
  p->malloc_managed = (f_malloc_managed)f[0];
  p->free_managed = (f_free_managed)f[1];
  p->ev_create = (f_ev_create)f[2];
  p->ev_record = (f_ev_record)f[3];
  p->ev_query = (f_ev_query)f[4];
  p->ev_sync = (f_ev_sync)f[5];
  Py_INCREF(blocks);
  Py_INCREF(lazy);
  Py_INCREF(lbs);
  p->blocks = blocks;
  p->lazy = lazy;
  p->lazy_by_src = lbs;
  p->cache_limit = limit;
  p->max_pending = maxp;
  return 0;
}

static int pool_traverse(BlockPool* p, visitproc visit, void* arg) {
  Py_VISIT(p->blocks);
  Py_VISIT(p->lazy);
  Py_VISIT(p->lazy_by_src);
  return 0;
}

static int pool_clear(BlockPool* p) {
  Py_CLEAR(p->blocks);
  Py_CLEAR(p->lazy);
  Py_CLEAR(p->lazy_by_src);
  return 0;
}

static void pool_dealloc(BlockPool* p) {
  PyObject_GC_UnTrack(p);
  pool_clear(p);
  /* cached blocks and events stay with the CUDA context (process exit) */
  Py_TYPE(p)->tp_free((PyObject*)p);
}

static PyObject* pool_allocate_(BlockPool* p, PyObject* args);
static PyObject* pool_allocate(BlockPool* p, PyObject* args) {
  const long long t0 = now_ns();
  PyObject* r = pool_allocate_(p, args);
  T_alloc += now_ns() - t0;
  return r;
}
static PyObject* pool_allocate_(BlockPool* p, PyObject* args) {
  int dev;
  Py_ssize_t n;
  if (!PyArg_ParseTuple(args, "in", &dev, &n)) return NULL;
  if (dev < 0 || dev >= MAX_DEV) {
    PyErr_SetString(PyExc_ValueError, "device index out of range");
    return NULL;
  }
  if (n < 0) {
    PyErr_SetString(AllocError ? AllocError : PyExc_MemoryError, "negative allocation size");
    return NULL;
  }
  p->n_alloc++;
  size_t cap = size_class((size_t)n);
  void* ptr = take(p, dev, cap);
  if (!ptr) {
    int rc = p->malloc_managed(dev, cap, &ptr);
    if (rc == -2) {
      trim_dev(p, dev, 0);
      rc = p->malloc_managed(dev, cap, &ptr);
    }
    if (rc != 0 || !ptr) {
      PyErr_Format(AllocError ? AllocError : PyExc_MemoryError,
                   "managed allocation of %zd bytes on gpu%d failed (rc %d)", n, dev, rc);
      return NULL;
    }
    p->n_new++;
  }
  DevBuf* b = PyObject_GC_New(DevBuf, &DevBufType);
  if (!b) {
    release_block(p, ptr, cap, dev);
    return NULL;
  }
  b->ptr = ptr;
  b->nbytes = n;
  b->cap = cap;
  b->dev = dev;
  b->weakreflist = NULL;
  b->dict = NULL;
  Py_INCREF(p);
  b->pool = p;
  PyObject_GC_Track(b);
  if (blocks_set(p, ptr, dev, cap) < 0) {
    Py_DECREF(b);
    return NULL;
  }
  return (PyObject*)b;
}

/* Device.allocate for one gpu device (devices.py:149-160 semantics:
 * negative sizes raise AllocationError, alloc_count counts calls),
 * installed as the device instance's `allocate` attribute. */
typedef struct {
  PyObject_HEAD
  BlockPool* pool;
  PyObject* device;
  int index;
} Allocator;

static PyTypeObject AllocatorType;
static PyObject *S_alloc_count, *ONE;

static PyObject* allocator_call(Allocator* a, PyObject* args, PyObject* kw) {
  Py_ssize_t n;
  if (!PyArg_ParseTuple(args, "n", &n)) return NULL;
  if (n < 0) {
    PyErr_SetString(AllocError ? AllocError : PyExc_MemoryError, "negative allocation size");
    return NULL;
  }
  PyObject* c = PyObject_GetAttr(a->device, S_alloc_count);
  if (!c) return NULL;
  PyObject* c1 = PyNumber_Add(c, ONE);
  Py_DECREF(c);
  if (!c1 || PyObject_SetAttr(a->device, S_alloc_count, c1) < 0) {
    Py_XDECREF(c1);
    return NULL;
  }
  Py_DECREF(c1);
  PyObject* t = Py_BuildValue("(in)", a->index, n);
  if (!t) return NULL;
  PyObject* r = pool_allocate(a->pool, t);
  Py_DECREF(t);
  return r;
}

static void allocator_dealloc(Allocator* a) {
  PyObject_GC_UnTrack(a);
  Py_CLEAR(a->pool);
  Py_CLEAR(a->device);
  Py_TYPE(a)->tp_free((PyObject*)a);
}

static int allocator_traverse(Allocator* a, visitproc visit, void* arg) {
  Py_VISIT(a->pool);
  Py_VISIT(a->device);
  return 0;
}

static int allocator_clear(Allocator* a) {
  Py_CLEAR(a->pool);
  Py_CLEAR(a->device);
  return 0;
}

static PyObject* pool_allocator(BlockPool* p, PyObject* args) {
  int dev;
  PyObject* device;
  if (!PyArg_ParseTuple(args, "iO", &dev, &device)) return NULL;
  if (dev < 0 || dev >= MAX_DEV) {
    PyErr_SetString(PyExc_ValueError, "device index out of range");
    return NULL;
  }
  Allocator* a = PyObject_GC_New(Allocator, &AllocatorType);
  if (!a) return NULL;
  Py_INCREF(p);
  a->pool = p;
  /* device -> allocator -> device is a cycle; both are GC-tracked */
  Py_INCREF(device);
  a->device = device;
  a->index = dev;
  PyObject_GC_Track(a);
  return (PyObject*)a;
}

static PyObject* pool_add_stream(BlockPool* p, PyObject* args) {
  int dev;
  PyObject* h;
  if (!PyArg_ParseTuple(args, "iO", &dev, &h)) return NULL;
  if (dev < 0 || dev >= MAX_DEV) {
    PyErr_SetString(PyExc_ValueError, "device index out of range");
    return NULL;
  }
  void* handle = h == Py_None ? NULL : PyLong_AsVoidPtr(h);
  if (PyErr_Occurred()) return NULL;
  StreamRec* ns = (StreamRec*)realloc(p->streams[dev], sizeof(StreamRec) * (p->nstreams[dev] + 1));
  if (!ns) return PyErr_NoMemory();
  p->streams[dev] = ns;
  ns[p->nstreams[dev]].handle = handle;
  ns[p->nstreams[dev]].marker = NULL;
  ns[p->nstreams[dev]].marker_seq = (uint64_t)-1;
  ns[p->nstreams[dev]].done_seq = (uint64_t)-1; /* nothing known yet */
  ns[p->nstreams[dev]].word = NULL;
  ns[p->nstreams[dev]].wnext = 0;
  ns[p->nstreams[dev]].wdisabled = 0;
  ns[p->nstreams[dev]].pending = NULL;
  ns[p->nstreams[dev]].npending = 0;
  if (p->mark_create) {
    uint64_t* w = NULL;
    if (p->mark_create(&w) == 0 && w) {
      *w = 0;
      ns[p->nstreams[dev]].word = w;
    }
  }
  p->nstreams[dev]++;
  Py_RETURN_NONE;
}

static PyObject* pool_bump(BlockPool* p, PyObject* unused) {
  p->seq++;
  Py_RETURN_NONE;
}

static PyObject* pool_trim(BlockPool* p, PyObject* args) {
  int dev;
  long long keep;
  if (!PyArg_ParseTuple(args, "iL", &dev, &keep)) return NULL;
  if (dev < 0 || dev >= MAX_DEV) {
    PyErr_SetString(PyExc_ValueError, "device index out of range");
    return NULL;
  }
  trim_dev(p, dev, keep);
  Py_RETURN_NONE;
}

static PyObject* pool_stats(BlockPool* p, PyObject* unused) {
  long long cached = 0;
  for (int d = 0; d < MAX_DEV; ++d) cached += p->cached[d];
  return Py_BuildValue("{s:L,s:L,s:L,s:L,s:L,s:L,s:L,s:n}", "allocate", p->n_alloc, "reused",
                       p->n_reuse, "new", p->n_new, "waited", p->n_wait, "released",
                       p->n_release, "trimmed", p->n_trim, "cached_bytes", cached, "event_pool",
                       (Py_ssize_t)p->nevpool);
}

static PyObject* pool_cached_bytes(BlockPool* p, PyObject* args) {
  int dev;
  if (!PyArg_ParseTuple(args, "i", &dev)) return NULL;
  if (dev < 0 || dev >= MAX_DEV) return PyLong_FromLong(0);
  return PyLong_FromLongLong(p->cached[dev]);
}

static PyMethodDef pool_methods[] = {
    {"allocate", (PyCFunction)pool_allocate, METH_VARARGS, "allocate(device, nbytes) -> DevBuf"},
    {"add_stream", (PyCFunction)pool_add_stream, METH_VARARGS, "add_stream(device, handle)"},
    {"allocator", (PyCFunction)pool_allocator, METH_VARARGS,
     "allocator(device index, device object) -> callable(nbytes) (Device.allocate)"},
    {"bump", (PyCFunction)pool_bump, METH_NOARGS, "start a new launch epoch"},
    {"trim", (PyCFunction)pool_trim, METH_VARARGS, "trim(device, keep_bytes)"},
    {"stats", (PyCFunction)pool_stats, METH_NOARGS, "counters"},
    {"cached_bytes", (PyCFunction)pool_cached_bytes, METH_VARARGS, "cached bytes of a device"},
    {NULL}};


/* ---------------------------------------------------------------- Entries
 * The gpu table's binary entry for the common case, in C: standard mode,
 * every operand a gpu storage of one device, no pending lazy copy that
 * must materialise first.  Decodes the reference's closures exactly as
 * tidepool_plugin.py does (store cells pack / mode, codec functions,
 * scalar fn's status cell), fuses a pending lossless cast into the load
 * (the Python _fuse_strides rule), builds the tpg_plan / tpg_operand
 * descriptors and calls tpg_binary.  Returns None when the Python entry
 * must handle the call (no side effect has happened then), else the
 * C-ABI return code.
 *
 *   Entries(pool, binary_fn_address, rt, tls, lazy, lazy_by_src, codecs,
 *           stats)
 *     codecs: {codec function: (wire code, size, big endian, compute code)}
 *     .set_default_stream(device, handle)
 *     .binary(op_code, plan, d_buf, store, a_buf, a_unpack, b_buf,
 *             b_unpack, fn, bases)
 */
typedef int (*f_binary)(void*, int, const tpg_plan*, const tpg_operand*, const tpg_operand*,
                        const tpg_operand*, int, int);
typedef int (*f_unary)(void*, int, const tpg_plan*, const tpg_operand*, const tpg_operand*, int,
                       int, int);
typedef int (*f_reduce)(void*, int, double, const tpg_plan*, const tpg_plan*, const tpg_operand*,
                        const tpg_operand*, int, int);

typedef struct {
  PyObject_HEAD
  BlockPool* pool;
  f_binary binary;
  f_unary unary; /* optional (set_unary) */
  f_reduce reduce; /* optional (set_reduce) */
  PyObject *rt, *tls, *lazy, *lazy_by_src, *codecs, *stats;
  PyObject* cell_idx; /* {(code, tag): tuple of closure indices} */
  PyObject* lazy_cls; /* tidepool_plugin._Lazy */
  PyObject* codec_objs; /* {codec function: (reference dtype, byteorder)} */
  PyObject* lossless;   /* bytes[32 * 32]: lossless_castable(src wire, dst wire) */
  PyObject* default_st[MAX_DEV]; /* default GpuStream objects */
  void* defaults[MAX_DEV];
  long long n_fast, n_fallback, n_fused, n_lazy;
} Entries;

static PyTypeObject EntriesType;
/* attribute names of a lazy-copy record (+ "lazy", the stats key) */
static const char* const L_str[19] = {"device", "plan", "stream", "dst_ptr", "src_ptr", "ddt",
                                      "dbig", "keep", "src_dtype", "dst_dtype", "src_order",
                                      "cext", "cdst", "csrc", "sbase", "soff", "sdt", "sbig",
                                      "lazy"};
static PyObject* L_names[19];
static PyObject* S_cpack;
static PyObject *S_standard, *S_stream, *S_device, *S_index, *S_handle, *S_status_sink, *S_extents,
    *S_strides, *S_fused, *S_src_ptr, *S_cext, *S_cdst, *S_csrc, *S_sbase, *S_soff, *S_sdt,
    *S_sbig, *S_pack, *S_mode, *S_ctx, *S_status, *S_store_tag, *S_status_tag;

static int entries_init(Entries* e, PyObject* args, PyObject* kw) {
  PyObject *pool, *fnaddr;
  if (!PyArg_ParseTuple(args, "O!OOOO!O!O!O", &BlockPoolType, &pool, &fnaddr, &e->rt, &e->tls,
                        &PyDict_Type, &e->lazy, &PyDict_Type, &e->lazy_by_src, &PyDict_Type,
                        &e->codecs, &e->stats))
    return -1;
  e->binary = (f_binary)PyLong_AsVoidPtr(fnaddr);
  if (!e->binary) {
    if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "null tpg_binary address");
    return -1;
  }
  Py_INCREF(pool);
  e->pool = (BlockPool*)pool;
  Py_INCREF(e->rt);
  Py_INCREF(e->tls);
  Py_INCREF(e->lazy);
  Py_INCREF(e->lazy_by_src);
  Py_INCREF(e->codecs);
  Py_INCREF(e->stats);
  e->cell_idx = PyDict_New();
  return e->cell_idx ? 0 : -1;
}

static PyObject* entries_set_copy_support(Entries* e, PyObject* args) {
  PyObject *cls, *objs, *ll;
  if (!PyArg_ParseTuple(args, "OO!O!", &cls, &PyDict_Type, &objs, &PyBytes_Type, &ll)) return NULL;
  if (PyBytes_GET_SIZE(ll) != 32 * 32) {
    PyErr_SetString(PyExc_ValueError, "lossless table must be 32 x 32 bytes");
    return NULL;
  }
  Py_INCREF(cls);
  Py_INCREF(objs);
  Py_INCREF(ll);
  Py_XSETREF(e->lazy_cls, cls);
  Py_XSETREF(e->codec_objs, objs);
  Py_XSETREF(e->lossless, ll);
  Py_RETURN_NONE;
}

static int entries_traverse(Entries* e, visitproc visit, void* arg) {
  Py_VISIT(e->pool);
  Py_VISIT(e->rt);
  Py_VISIT(e->tls);
  Py_VISIT(e->lazy);
  Py_VISIT(e->lazy_by_src);
  Py_VISIT(e->codecs);
  Py_VISIT(e->stats);
  Py_VISIT(e->cell_idx);
  Py_VISIT(e->lazy_cls);
  Py_VISIT(e->codec_objs);
  Py_VISIT(e->lossless);
  for (int d = 0; d < MAX_DEV; ++d) Py_VISIT(e->default_st[d]);
  return 0;
}

static int entries_clear(Entries* e) {
  Py_CLEAR(e->pool);
  Py_CLEAR(e->rt);
  Py_CLEAR(e->tls);
  Py_CLEAR(e->lazy);
  Py_CLEAR(e->lazy_by_src);
  Py_CLEAR(e->codecs);
  Py_CLEAR(e->stats);
  Py_CLEAR(e->cell_idx);
  Py_CLEAR(e->lazy_cls);
  Py_CLEAR(e->codec_objs);
  Py_CLEAR(e->lossless);
  for (int d = 0; d < MAX_DEV; ++d) Py_CLEAR(e->default_st[d]);
  return 0;
}

static void entries_dealloc(Entries* e) {
  PyObject_GC_UnTrack(e);
  entries_clear(e);
  Py_TYPE(e)->tp_free((PyObject*)e);
}

/* closure cell contents of `fn` for `names` (borrowed refs, NULL when
 * absent); the name -> index map is cached per code object.  Returns -1 when
 * fn is not a Python function with a closure. */
static int closure_cells(Entries* e, PyObject* fn, PyObject* tag, PyObject* const* names, int n,
                         PyObject** out) {
  if (!PyFunction_Check(fn)) return -1;
  PyObject* clos = PyFunction_GET_CLOSURE(fn);
  if (!clos) return -1;
  PyObject* code = PyFunction_GET_CODE(fn);
  /* small front cache keyed by object identity (entries hold references,
   * so a cached code object cannot be freed and its address reused) */
  static struct {
    PyObject *code, *tag;
    int n;
    long at[4];
  } fc[16];
  const unsigned h = (unsigned)(((uintptr_t)code >> 4) ^ ((uintptr_t)tag >> 4)) & 15u;
  if (fc[h].code == code && fc[h].tag == tag && fc[h].n == n) {
    for (int k = 0; k < n; ++k) {
      const long at = fc[h].at[k];
      out[k] = (at >= 0 && at < PyTuple_GET_SIZE(clos)) ? PyCell_GET(PyTuple_GET_ITEM(clos, at))
                                                         : NULL;
    }
    return 0;
  }
  PyObject* key = PyTuple_Pack(2, code, tag);
  if (!key) return -2;
  PyObject* idx = PyDict_GetItemWithError(e->cell_idx, key);
  if (!idx) {
    if (PyErr_Occurred()) {
      Py_DECREF(key);
      return -2;
    }
    PyObject* fv = PyObject_GetAttrString(code, "co_freevars");
    if (!fv) {
      Py_DECREF(key);
      return -2;
    }
    idx = PyTuple_New(n);
    for (int k = 0; idx && k < n; ++k) {
      long at = -1;
      for (Py_ssize_t i = 0; i < PyTuple_GET_SIZE(fv); ++i)
        if (PyUnicode_Compare(PyTuple_GET_ITEM(fv, i), names[k]) == 0) at = (long)i;
      PyTuple_SET_ITEM(idx, k, PyLong_FromLong(at));
    }
    Py_DECREF(fv);
    if (!idx || PyDict_SetItem(e->cell_idx, key, idx) < 0) {
      Py_XDECREF(idx);
      Py_DECREF(key);
      return -2;
    }
    Py_DECREF(idx); /* the dict holds it */
  }
  Py_DECREF(key);
  if (n <= 4) {
    Py_XSETREF(fc[h].code, (Py_INCREF(code), code));
    Py_XSETREF(fc[h].tag, (Py_INCREF(tag), tag));
    fc[h].n = n;
  }
  for (int k = 0; k < n; ++k) {
    long at = PyLong_AsLong(PyTuple_GET_ITEM(idx, k));
    if (n <= 4) fc[h].at[k] = at;
    out[k] = (at >= 0 && at < PyTuple_GET_SIZE(clos))
                 ? PyCell_GET(PyTuple_GET_ITEM(clos, at))
                 : NULL;
  }
  return 0;
}

/* DevBuf behind a memoryview (or NULL) */
static DevBuf* devbuf_of(PyObject* mv) {
  if (!PyMemoryView_Check(mv)) return NULL;
  PyObject* b = PyMemoryView_GET_BASE(mv);
  return (b && Py_TYPE(b) == &DevBufType) ? (DevBuf*)b : NULL;
}

typedef struct {
  int wire, size, big, compute;
} CodecInfo;

static int codec_info(Entries* e, PyObject* fn, CodecInfo* ci) {
  PyObject* t = fn ? PyDict_GetItemWithError(e->codecs, fn) : NULL;
  if (!t || !PyTuple_Check(t) || PyTuple_GET_SIZE(t) != 4) return -1;
  ci->wire = (int)PyLong_AsLong(PyTuple_GET_ITEM(t, 0));
  ci->size = (int)PyLong_AsLong(PyTuple_GET_ITEM(t, 1));
  ci->big = (int)PyLong_AsLong(PyTuple_GET_ITEM(t, 2));
  ci->compute = (int)PyLong_AsLong(PyTuple_GET_ITEM(t, 3));
  return PyErr_Occurred() ? -1 : 0;
}

/* int64 sequence -> array; -1 on any mismatch */
static int i64_seq(PyObject* seq, int64_t* out, int maxn) {
  PyObject* f = PySequence_Fast(seq, "sequence");
  if (!f) return -1;
  Py_ssize_t n = PySequence_Fast_GET_SIZE(f);
  if (n > maxn) {
    Py_DECREF(f);
    return -1;
  }
  for (Py_ssize_t i = 0; i < n; ++i) {
    out[i] = PyLong_AsLongLong(PySequence_Fast_GET_ITEM(f, i));
    if (out[i] == -1 && PyErr_Occurred()) {
      Py_DECREF(f);
      return -1;
    }
  }
  Py_DECREF(f);
  return (int)n;
}

static int64_t attr_i64(PyObject* o, PyObject* name, int* bad) {
  PyObject* v = PyObject_GetAttr(o, name);
  if (!v) {
    *bad = 1;
    return 0;
  }
  int64_t r = PyLong_AsLongLong(v);
  Py_DECREF(v);
  if (r == -1 && PyErr_Occurred()) *bad = 1;
  return r;
}

/* _fuse_strides (tidepool_plugin.py): re-express a binary operand reading a
 * recorded copy's dense destination as a view of the copy's source. */



static int lazyrec_traverse(LazyRecord* r, visitproc visit, void* arg) {
  Py_VISIT(r->plan);
  Py_VISIT(r->stream);
  Py_VISIT(r->keep);
  Py_VISIT(r->src_dtype);
  Py_VISIT(r->dst_dtype);
  Py_VISIT(r->src_order);
  Py_VISIT(r->dst_ptr);
  Py_VISIT(r->src_ptr);
  Py_VISIT(r->cext);
  Py_VISIT(r->cdst);
  Py_VISIT(r->csrc);
  return 0;
}
static int lazyrec_clear(LazyRecord* r) {
  Py_CLEAR(r->plan);
  Py_CLEAR(r->stream);
  Py_CLEAR(r->keep);
  Py_CLEAR(r->src_dtype);
  Py_CLEAR(r->dst_dtype);
  Py_CLEAR(r->src_order);
  Py_CLEAR(r->dst_ptr);
  Py_CLEAR(r->src_ptr);
  Py_CLEAR(r->cext);
  Py_CLEAR(r->cdst);
  Py_CLEAR(r->csrc);
  return 0;
}
static void lazyrec_dealloc(LazyRecord* r) {
  PyObject_GC_UnTrack(r);
  lazyrec_clear(r);
  Py_TYPE(r)->tp_free((PyObject*)r);
}
#define LR_OBJ(name) {#name, T_OBJECT, offsetof(LazyRecord, name), 0, NULL}
#define LR_LL(name) {#name, T_LONGLONG, offsetof(LazyRecord, name), 0, NULL}
static PyMemberDef lazyrec_members[] = {
    LR_OBJ(plan), LR_OBJ(stream), LR_OBJ(keep), LR_OBJ(src_dtype), LR_OBJ(dst_dtype),
    LR_OBJ(src_order), LR_OBJ(dst_ptr), LR_OBJ(src_ptr), LR_OBJ(cext), LR_OBJ(cdst),
    LR_OBJ(csrc), LR_LL(device), LR_LL(ddt), LR_LL(dbig), LR_LL(sbase), LR_LL(soff),
    LR_LL(sdt), LR_LL(sbig), {NULL}};

static int fuse(PyObject* lz, int nd, const int64_t* bext, const int64_t* bstr, int64_t base,
                int size, int64_t* out_str, int64_t* out_off, int64_t* sbase_out, int* sdt_out,
                int* sbig_out) {
  int64_t E[TPG_MAX_DIMS], T[TPG_MAX_DIMS], S[TPG_MAX_DIMS], dg[TPG_MAX_DIMS];
  int ne = -1, nt = -1, ns = -1;
  const CopyPack* cp = NULL;
  PyObject* pk = NULL;
  if (PyObject_TypeCheck(lz, &LazyRecordType) && ((LazyRecord*)lz)->has_pack) {
    cp = &((LazyRecord*)lz)->pack;
    ne = nt = ns = (int)cp->ne;
    memcpy(E, cp->E, sizeof E);
    memcpy(T, cp->T, sizeof T);
    memcpy(S, cp->S, sizeof S);
  } else {
    PyErr_Clear();
    PyObject *ce = PyObject_GetAttr(lz, S_cext), *cd = PyObject_GetAttr(lz, S_cdst),
             *cs = PyObject_GetAttr(lz, S_csrc);
    if (ce && cd && cs) {
      ne = i64_seq(ce, E, TPG_MAX_DIMS);
      nt = i64_seq(cd, T, TPG_MAX_DIMS);
      ns = i64_seq(cs, S, TPG_MAX_DIMS);
    }
    Py_XDECREF(ce);
    Py_XDECREF(cd);
    Py_XDECREF(cs);
  }
  if (ne < 0 || nt != ne || ns != ne || size <= 0 || base % size) {
    Py_XDECREF(pk);
    PyErr_Clear();
    return -1;
  }
  int64_t lin = base / size;
  for (int j = 0; j < ne; ++j) {
    if (E[j]) {
      dg[j] = lin % E[j];
      lin /= E[j];
    } else {
      dg[j] = 0;
    }
  }
  if (lin) {
    Py_XDECREF(pk);
    return -1;
  }
  unsigned used = 0;
  for (int i = 0; i < nd; ++i) {
    if (bext[i] == 1 || bstr[i] == 0) {
      out_str[i] = 0;
      continue;
    }
    int found = -1;
    for (int j = 0; j < ne; ++j)
      if (T[j] == bstr[i] && E[j] == bext[i] && dg[j] == 0 && !(used & (1u << j))) {
        found = j;
        break;
      }
    if (found < 0) {
      Py_XDECREF(pk);
      return -1;
    }
    used |= 1u << found;
    out_str[i] = S[found];
  }
  int64_t off = 0;
  for (int j = 0; j < ne; ++j) off += dg[j] * S[j];
  int bad = 0;
  if (cp) {
    *out_off = cp->soff + off;
    *sbase_out = cp->sbase;
    *sdt_out = (int)cp->sdt;
    *sbig_out = (int)cp->sbig;
  } else {
    *out_off = attr_i64(lz, S_soff, &bad) + off;
    *sbase_out = attr_i64(lz, S_sbase, &bad);
    *sdt_out = (int)attr_i64(lz, S_sdt, &bad);
    *sbig_out = (int)attr_i64(lz, S_sbig, &bad);
  }
  Py_XDECREF(pk);
  if (bad) {
    PyErr_Clear();
    return -1;
  }
  return 0;
}

static PyObject* entries_binary_(Entries* e, PyObject* const* args, Py_ssize_t nargs);
static PyObject* entries_binary(Entries* e, PyObject* const* args, Py_ssize_t nargs) {
  const long long t0 = now_ns();
  PyObject* r = entries_binary_(e, args, nargs);
  T_binary += now_ns() - t0;
  return r;
}
static PyObject* entries_binary_(Entries* e, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 10) {
    PyErr_SetString(PyExc_TypeError, "binary(op, plan, d_buf, store, a_buf, a_unpack, b_buf, "
                                     "b_unpack, fn, bases)");
    return NULL;
  }
  int op = (int)PyLong_AsLong(args[0]);
  PyObject *plan = args[1], *store = args[3], *fn = args[8], *bases = args[9];
  if (PyErr_Occurred()) return NULL;
#define FALLBACK()         \
  do {                     \
    PyErr_Clear();         \
    e->n_fallback++;       \
    Py_RETURN_NONE;        \
  } while (0)
  /* store closure: pack / mode */
  PyObject* sc[3];
  PyObject* const snames[3] = {S_pack, S_mode, S_ctx};
  int r = closure_cells(e, store, S_store_tag, snames, 3, sc);
  if (r == -2) return NULL;
  if (r < 0 || !sc[0]) FALLBACK();
  if (sc[1] && sc[1] != S_standard && PyUnicode_Compare(sc[1], S_standard) != 0) FALLBACK();
  CodecInfo cd, ca, cb;
  if (codec_info(e, sc[0], &cd) || codec_info(e, args[5], &ca) || codec_info(e, args[7], &cb))
    FALLBACK();
  DevBuf *bd = devbuf_of(args[2]), *ba = devbuf_of(args[4]), *bb = devbuf_of(args[6]);
  if (!bd || !ba || !bb || ba->dev != bd->dev || bb->dev != bd->dev) FALLBACK();
  const int dev = bd->dev;
  /* plan */
  int64_t ext[TPG_MAX_DIMS], str[3][TPG_MAX_DIMS];
  PyObject *pe = PyObject_GetAttr(plan, S_extents), *ps = PyObject_GetAttr(plan, S_strides);
  int nd = pe ? i64_seq(pe, ext, TPG_MAX_DIMS) : -1;
  int ok = nd >= 0 && ps && PySequence_Check(ps) && PySequence_Size(ps) == 3;
  for (int v = 0; ok && v < 3; ++v) {
    PyObject* sv = PySequence_GetItem(ps, v);
    ok = sv && i64_seq(sv, str[v], TPG_MAX_DIMS) == nd;
    Py_XDECREF(sv);
  }
  Py_XDECREF(pe);
  Py_XDECREF(ps);
  if (!ok) FALLBACK();
  if (!PyTuple_Check(bases) || PyTuple_GET_SIZE(bases) != 3) FALLBACK();
  int64_t base[3];
  for (int v = 0; v < 3; ++v) base[v] = PyLong_AsLongLong(PyTuple_GET_ITEM(bases, v));
  if (PyErr_Occurred()) FALLBACK();
  /* pending lazy copies: the destination must not have one (as dst or
   * src); an operand with one must fuse */
  tpg_operand od, oa, ob;
  memset(&od, 0, sizeof od);
  memset(&oa, 0, sizeof oa);
  memset(&ob, 0, sizeof ob);
  int nfused = 0;
  if (PyDict_GET_SIZE(e->lazy) || PyDict_GET_SIZE(e->lazy_by_src)) {
    PyObject* kd = PyLong_FromVoidPtr(bd->ptr);
    int hit = kd && (PyDict_Contains(e->lazy, kd) == 1 || PyDict_Contains(e->lazy_by_src, kd) == 1);
    Py_XDECREF(kd);
    if (hit || PyErr_Occurred()) FALLBACK();
  }
  DevBuf* bufs[2] = {ba, bb};
  CodecInfo* cis[2] = {&ca, &cb};
  tpg_operand* os[2] = {&oa, &ob};
  for (int v = 1; v <= 2; ++v) {
    DevBuf* b = bufs[v - 1];
    PyObject* lz = NULL;
    if (PyDict_GET_SIZE(e->lazy)) {
      PyObject* k = PyLong_FromVoidPtr(b->ptr);
      lz = k ? PyDict_GetItemWithError(e->lazy, k) : NULL;
      Py_XDECREF(k);
      if (PyErr_Occurred()) FALLBACK();
    }
    tpg_operand* o = os[v - 1];
    if (lz) {
      int bad = 0;
      int64_t sp = attr_i64(lz, S_src_ptr, &bad);
      if (bad || (void*)(intptr_t)sp == bd->ptr) FALLBACK();
      int64_t fstr[TPG_MAX_DIMS], off, sbase;
      int sdt, sbig;
      if (fuse(lz, nd, ext, str[v], base[v], cis[v - 1]->size, fstr, &off, &sbase, &sdt, &sbig))
        FALLBACK();
      memcpy(str[v], fstr, sizeof(int64_t) * nd);
      o->base = (void*)(intptr_t)sbase;
      o->offset = off;
      o->dtype = sdt;
      o->big_endian = sbig;
      nfused++;
    } else {
      o->base = b->ptr;
      o->offset = base[v];
      o->dtype = cis[v - 1]->wire;
      o->big_endian = cis[v - 1]->big;
    }
  }
  od.base = bd->ptr;
  od.offset = base[0];
  od.dtype = cd.wire;
  od.big_endian = cd.big;
  /* stream: the thread's current gpu stream when it is on this device */
  void* handle = dev < MAX_DEV ? e->defaults[dev] : NULL;
  PyObject* st = PyObject_GetAttr(e->tls, S_stream);
  if (!st) {
    PyErr_Clear();
  } else if (st != Py_None) {
    int bad = 0;
    PyObject* sdev = PyObject_GetAttr(st, S_device);
    int64_t sidx = sdev ? attr_i64(sdev, S_index, &bad) : (bad = 1, 0);
    Py_XDECREF(sdev);
    if (!bad && sidx == dev) handle = (void*)(intptr_t)attr_i64(st, S_handle, &bad);
    if (bad) {
      Py_DECREF(st);
      FALLBACK();
    }
  }
  Py_XDECREF(st);
  if (!handle) FALLBACK();
  /* status set the scalar fn records into (kernels.py:72-78) */
  PyObject* stc[1];
  PyObject* const stn[1] = {S_status};
  r = closure_cells(e, fn, S_status_tag, stn, 1, stc);
  if (r == -2) return NULL;
  if (r == 0 && stc[0] && PySet_Check(stc[0])) {
    PyObject* cur = PyObject_GetAttr(e->rt, S_status_sink);
    if (cur != stc[0] && PyObject_SetAttr(e->rt, S_status_sink, stc[0]) < 0) {
      Py_XDECREF(cur);
      return NULL;
    }
    Py_XDECREF(cur);
    PyErr_Clear();
  }
  /* launch */
  tpg_plan p;
  memset(&p, 0, sizeof p);
  p.ndim = nd;
  p.nviews = 3;
  for (int i = 0; i < nd; ++i) {
    p.extent[i] = ext[i];
    for (int v = 0; v < 3; ++v) p.stride[v][i] = str[v][i];
  }
  e->pool->seq++; /* rt.current(): a new launch epoch */
  const long long tl = now_ns();
  int rc = e->binary(handle, op, &p, &od, &oa, &ob, ca.compute, 0);
  T_launch += now_ns() - tl;
  e->n_fast++;
  e->n_fused += nfused;
  return PyLong_FromLong(rc);
#undef FALLBACK
}

static PyObject* entries_copy(Entries* e, PyObject* const* args, Py_ssize_t nargs);
static PyObject *S_complex_fn, *S_complex_tag;

/* The gpu table's unary entries (negate ... conjugate) for the common case:
 * standard mode, a real gpu source and destination of one device, no
 * pending copy on either, a scalar fn without the complex promotion
 * (unary_forces_complex).  Same contract as entries_binary. */
static PyObject* entries_unary(Entries* e, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 8 || !e->unary) Py_RETURN_NONE;
  const int op = (int)PyLong_AsLong(args[0]);
  PyObject *plan = args[1], *store = args[3], *fn = args[6], *bases = args[7];
  if (PyErr_Occurred()) return NULL;
#define FALLBACK()   \
  do {               \
    PyErr_Clear();   \
    e->n_fallback++; \
    Py_RETURN_NONE;  \
  } while (0)
  PyObject* sc[3];
  PyObject* const snames[3] = {S_pack, S_mode, S_ctx};
  int r = closure_cells(e, store, S_store_tag, snames, 3, sc);
  if (r == -2) return NULL;
  if (r < 0 || !sc[0]) FALLBACK();
  if (sc[1] && sc[1] != S_standard && PyUnicode_Compare(sc[1], S_standard) != 0) FALLBACK();
  CodecInfo cd, ca;
  if (codec_info(e, sc[0], &cd) || codec_info(e, args[5], &ca)) FALLBACK();
  if (ca.wire >= 12 || cd.wire >= 12) FALLBACK(); /* complex: the Python entry */
  PyObject* fc[1];
  PyObject* const fcn[1] = {S_complex_fn};
  r = closure_cells(e, fn, S_complex_tag, fcn, 1, fc);
  if (r == -2) return NULL;
  if (r == 0 && fc[0]) FALLBACK(); /* unary_forces_complex */
  DevBuf *bd = devbuf_of(args[2]), *ba = devbuf_of(args[4]);
  if (!bd || !ba || ba->dev != bd->dev) FALLBACK();
  const int dev = bd->dev;
  int64_t ext[TPG_MAX_DIMS], str[2][TPG_MAX_DIMS];
  PyObject *pe = PyObject_GetAttr(plan, S_extents), *ps = PyObject_GetAttr(plan, S_strides);
  int nd = pe ? i64_seq(pe, ext, TPG_MAX_DIMS) : -1;
  int ok = nd >= 0 && ps && PySequence_Check(ps) && PySequence_Size(ps) == 2;
  for (int v = 0; ok && v < 2; ++v) {
    PyObject* sv = PySequence_GetItem(ps, v);
    ok = sv && i64_seq(sv, str[v], TPG_MAX_DIMS) == nd;
    Py_XDECREF(sv);
  }
  Py_XDECREF(pe);
  Py_XDECREF(ps);
  if (!ok || !PyTuple_Check(bases) || PyTuple_GET_SIZE(bases) != 2) FALLBACK();
  const int64_t b0 = PyLong_AsLongLong(PyTuple_GET_ITEM(bases, 0));
  const int64_t b1 = PyLong_AsLongLong(PyTuple_GET_ITEM(bases, 1));
  if (PyErr_Occurred()) FALLBACK();
  if (PyDict_GET_SIZE(e->lazy) || PyDict_GET_SIZE(e->lazy_by_src)) {
    PyObject *kd = PyLong_FromVoidPtr(bd->ptr), *ka = PyLong_FromVoidPtr(ba->ptr);
    const int busy = !kd || !ka || PyDict_Contains(e->lazy, kd) == 1 ||
                     PyDict_Contains(e->lazy_by_src, kd) == 1 || PyDict_Contains(e->lazy, ka) == 1;
    Py_XDECREF(kd);
    Py_XDECREF(ka);
    if (busy || PyErr_Occurred()) FALLBACK();
  }
  void* handle = e->defaults[dev];
  PyObject* st = PyObject_GetAttr(e->tls, S_stream);
  if (!st) {
    PyErr_Clear();
  } else if (st != Py_None) {
    int bad = 0;
    PyObject* sdev = PyObject_GetAttr(st, S_device);
    int64_t sidx = sdev ? attr_i64(sdev, S_index, &bad) : (bad = 1, 0);
    Py_XDECREF(sdev);
    if (!bad && sidx == dev) handle = (void*)(intptr_t)attr_i64(st, S_handle, &bad);
    if (bad) {
      Py_DECREF(st);
      FALLBACK();
    }
  }
  Py_XDECREF(st);
  if (!handle) FALLBACK();
  PyObject* stc[1];
  PyObject* const stn[1] = {S_status};
  r = closure_cells(e, fn, S_status_tag, stn, 1, stc);
  if (r == -2) return NULL;
  if (r == 0 && stc[0] && PySet_Check(stc[0])) {
    PyObject* cur = PyObject_GetAttr(e->rt, S_status_sink);
    if (cur != stc[0] && PyObject_SetAttr(e->rt, S_status_sink, stc[0]) < 0) {
      Py_XDECREF(cur);
      return NULL;
    }
    Py_XDECREF(cur);
    PyErr_Clear();
  }
  tpg_plan p;
  memset(&p, 0, sizeof p);
  p.ndim = nd;
  p.nviews = 2;
  for (int i = 0; i < nd; ++i) {
    p.extent[i] = ext[i];
    p.stride[0][i] = str[0][i];
    p.stride[1][i] = str[1][i];
  }
  tpg_operand od, oa;
  memset(&od, 0, sizeof od);
  memset(&oa, 0, sizeof oa);
  od.base = bd->ptr;
  od.offset = b0;
  od.dtype = cd.wire;
  od.big_endian = cd.big;
  oa.base = ba->ptr;
  oa.offset = b1;
  oa.dtype = ca.wire;
  oa.big_endian = ca.big;
  e->pool->seq++;
  const int rc = e->unary(handle, op, &p, &od, &oa, ca.compute, 0, 0);
  e->n_fast++;
  return PyLong_FromLong(rc);
#undef FALLBACK
}

/* plan attributes -> tpg_plan with `nv` views; -1 on mismatch */
static int read_plan(PyObject* plan, int nv, tpg_plan* p) {
  int64_t ext[TPG_MAX_DIMS];
  PyObject *pe = PyObject_GetAttr(plan, S_extents), *ps = PyObject_GetAttr(plan, S_strides);
  int nd = pe ? i64_seq(pe, ext, TPG_MAX_DIMS) : -1;
  int ok = nd >= 0 && ps && PySequence_Check(ps) && PySequence_Size(ps) == nv;
  memset(p, 0, sizeof *p);
  for (int v = 0; ok && v < nv; ++v) {
    PyObject* sv = PySequence_GetItem(ps, v);
    ok = sv && i64_seq(sv, p->stride[v], TPG_MAX_DIMS) == nd;
    Py_XDECREF(sv);
  }
  Py_XDECREF(pe);
  Py_XDECREF(ps);
  if (!ok) return -1;
  p->ndim = nd;
  p->nviews = nv;
  for (int i = 0; i < nd; ++i) p->extent[i] = ext[i];
  return 0;
}

static PyObject *S_p, *S_norm_tag;

/* The gpu table's reduction entries (reference signature (outer, inner,
 * d_buf, store, a_buf, a_unpack, init, step, fin, bases), ops.py:522-556)
 * for the common case: standard mode, gpu source and destination of one
 * device, no pending copy on either.  args[0] = op code, args[1] = 1 for
 * the norm (its order is the `p` cell of the step closure). */
static PyObject* entries_reduce(Entries* e, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 12 || !e->reduce) Py_RETURN_NONE;
  const int op = (int)PyLong_AsLong(args[0]);
  const int is_norm = PyObject_IsTrue(args[1]);
  PyObject *outer = args[2], *inner = args[3], *store = args[5], *step = args[9],
           *bases = args[11];
  if (PyErr_Occurred()) return NULL;
#define FALLBACK()   \
  do {               \
    PyErr_Clear();   \
    e->n_fallback++; \
    Py_RETURN_NONE;  \
  } while (0)
  PyObject* sc[3];
  PyObject* const snames[3] = {S_pack, S_mode, S_ctx};
  int r = closure_cells(e, store, S_store_tag, snames, 3, sc);
  if (r == -2) return NULL;
  if (r < 0 || !sc[0]) FALLBACK();
  if (sc[1] && sc[1] != S_standard && PyUnicode_Compare(sc[1], S_standard) != 0) FALLBACK();
  CodecInfo cd, ca;
  if (codec_info(e, sc[0], &cd) || codec_info(e, args[7], &ca)) FALLBACK();
  double pnorm = 2.0;
  if (is_norm) {
    PyObject* pc[1];
    PyObject* const pn[1] = {S_p};
    r = closure_cells(e, step, S_norm_tag, pn, 1, pc);
    if (r == -2) return NULL;
    if (r == 0 && pc[0]) {
      pnorm = PyFloat_AsDouble(pc[0]);
      if (PyErr_Occurred()) FALLBACK();
    }
  }
  DevBuf *bd = devbuf_of(args[4]), *ba = devbuf_of(args[6]);
  if (!bd || !ba || ba->dev != bd->dev) FALLBACK();
  const int dev = bd->dev;
  tpg_plan po, pi;
  if (read_plan(outer, 2, &po) || read_plan(inner, 1, &pi)) FALLBACK();
  if (!PyTuple_Check(bases) || PyTuple_GET_SIZE(bases) != 2) FALLBACK();
  const int64_t b0 = PyLong_AsLongLong(PyTuple_GET_ITEM(bases, 0));
  const int64_t b1 = PyLong_AsLongLong(PyTuple_GET_ITEM(bases, 1));
  if (PyErr_Occurred()) FALLBACK();
  if (PyDict_GET_SIZE(e->lazy) || PyDict_GET_SIZE(e->lazy_by_src)) {
    PyObject *kd = PyLong_FromVoidPtr(bd->ptr), *ka = PyLong_FromVoidPtr(ba->ptr);
    const int busy = !kd || !ka || PyDict_Contains(e->lazy, kd) == 1 ||
                     PyDict_Contains(e->lazy_by_src, kd) == 1 || PyDict_Contains(e->lazy, ka) == 1;
    Py_XDECREF(kd);
    Py_XDECREF(ka);
    if (busy || PyErr_Occurred()) FALLBACK();
  }
  void* handle = e->defaults[dev];
  PyObject* st = PyObject_GetAttr(e->tls, S_stream);
  if (!st) {
    PyErr_Clear();
  } else if (st != Py_None) {
    int bad = 0;
    PyObject* sdev = PyObject_GetAttr(st, S_device);
    int64_t sidx = sdev ? attr_i64(sdev, S_index, &bad) : (bad = 1, 0);
    Py_XDECREF(sdev);
    if (!bad && sidx == dev) handle = (void*)(intptr_t)attr_i64(st, S_handle, &bad);
    if (bad) {
      Py_DECREF(st);
      FALLBACK();
    }
  }
  Py_XDECREF(st);
  if (!handle) FALLBACK();
  tpg_operand od, oa;
  memset(&od, 0, sizeof od);
  memset(&oa, 0, sizeof oa);
  od.base = bd->ptr;
  od.offset = b0;
  od.dtype = cd.wire;
  od.big_endian = cd.big;
  oa.base = ba->ptr;
  oa.offset = b1;
  oa.dtype = ca.wire;
  oa.big_endian = ca.big;
  e->pool->seq++;
  const int rc = e->reduce(handle, op, pnorm, &po, &pi, &od, &oa, ca.compute, 0);
  e->n_fast++;
  return PyLong_FromLong(rc);
#undef FALLBACK
}

static PyObject* entries_set_reduce(Entries* e, PyObject* addr) {
  e->reduce = (f_reduce)PyLong_AsVoidPtr(addr);
  if (PyErr_Occurred()) return NULL;
  Py_RETURN_NONE;
}

static PyObject* entries_set_unary(Entries* e, PyObject* addr) {
  e->unary = (f_unary)PyLong_AsVoidPtr(addr);
  if (PyErr_Occurred()) return NULL;
  Py_RETURN_NONE;
}

/* A gpu table entry callable in C: tries the fast path (when the plugin's
 * profiling hook is off) and otherwise calls the Python entry `slow` with
 * the same arguments.  kind 0 = binary (9 table arguments), 1 = copy (7). */
typedef struct {
  PyObject_HEAD
  Entries* e;
  int kind;
  PyObject* opobj; /* binary op code */
  PyObject* slow;
} FastEntry;

static PyTypeObject FastEntryType;
static PyObject *S_profile, *S_check, *S_kernel;

static PyObject* fastentry_call(FastEntry* f, PyObject* args, PyObject* kw) {
  if ((!kw || (PyDict_Check(kw) && PyDict_GET_SIZE(kw) == 0)) && PyTuple_Check(args)) {
    PyObject* prof = PyObject_GetAttr(f->e->rt, S_profile);
    const int off = prof == Py_None;
    if (!prof) PyErr_Clear();
    Py_XDECREF(prof);
    const Py_ssize_t n = PyTuple_GET_SIZE(args);
    PyObject* r = NULL;
    int tried = 0;
    if (off && f->kind == 0 && n == 9) {
      PyObject* a[10];
      a[0] = f->opobj;
      for (int i = 0; i < 9; ++i) a[i + 1] = PyTuple_GET_ITEM(args, i);
      r = entries_binary(f->e, a, 10);
      tried = 1;
    } else if (off && f->kind == 1 && n == 7) {
      r = entries_copy(f->e, ((PyTupleObject*)args)->ob_item, 7);
      tried = 1;
    } else if (off && f->kind == 2 && n == 7) {
      PyObject* a[8];
      a[0] = f->opobj;
      for (int i = 0; i < 7; ++i) a[i + 1] = PyTuple_GET_ITEM(args, i);
      r = entries_unary(f->e, a, 8);
      tried = 1;
    } else if (off && (f->kind == 3 || f->kind == 4) && n == 10) {
      PyObject* a[12];
      a[0] = f->opobj;
      a[1] = f->kind == 4 ? Py_True : Py_False;
      for (int i = 0; i < 10; ++i) a[i + 2] = PyTuple_GET_ITEM(args, i);
      r = entries_reduce(f->e, a, 12);
      tried = 1;
    }
    if (tried) {
      if (!r) return NULL;
      if (r != Py_None) {
        if (f->kind != 1) {
          const long rc = PyLong_AsLong(r);
          Py_DECREF(r);
          if (rc) {
            PyObject* rco = PyLong_FromLong(rc);
            PyObject* res = rco ? PyObject_CallMethodObjArgs(f->e->rt, S_check, rco, S_kernel, NULL)
                                : NULL;
            Py_XDECREF(rco);
            return res;  /* rt.check raises the reference's DeviceError */
          }
          Py_RETURN_NONE;
        }
        Py_DECREF(r);
        Py_RETURN_NONE;  /* copy recorded */
      }
      Py_DECREF(r);
    }
  }
  return PyObject_Call(f->slow, args, kw);
}

static void fastentry_dealloc(FastEntry* f) {
  PyObject_GC_UnTrack(f);
  Py_CLEAR(f->e);
  Py_CLEAR(f->opobj);
  Py_CLEAR(f->slow);
  Py_TYPE(f)->tp_free((PyObject*)f);
}
static int fastentry_traverse(FastEntry* f, visitproc visit, void* arg) {
  Py_VISIT(f->e);
  Py_VISIT(f->opobj);
  Py_VISIT(f->slow);
  return 0;
}
static int fastentry_clear(FastEntry* f) {
  Py_CLEAR(f->e);
  Py_CLEAR(f->opobj);
  Py_CLEAR(f->slow);
  return 0;
}

static PyObject* entries_entry(Entries* e, PyObject* args) {
  int kind, op;
  PyObject* slow;
  if (!PyArg_ParseTuple(args, "iiO", &kind, &op, &slow)) return NULL;
  if (kind < 0 || kind > 4) {
    PyErr_SetString(PyExc_ValueError, "kind: 0 binary, 1 copy, 2 unary, 3 reduce, 4 norm");
    return NULL;
  }
  FastEntry* f = PyObject_GC_New(FastEntry, &FastEntryType);
  if (!f) return NULL;
  Py_INCREF(e);
  f->e = e;
  f->kind = kind;
  f->opobj = PyLong_FromLong(op);
  Py_INCREF(slow);
  f->slow = slow;
  PyObject_GC_Track(f);
  if (!f->opobj) {
    Py_DECREF(f);
    return NULL;
  }
  return (PyObject*)f;
}

static PyObject* entries_set_default(Entries* e, PyObject* args) {
  int dev;
  PyObject *h, *obj;
  if (!PyArg_ParseTuple(args, "iOO", &dev, &h, &obj)) return NULL;
  if (dev < 0 || dev >= MAX_DEV) {
    PyErr_SetString(PyExc_ValueError, "device index out of range");
    return NULL;
  }
  e->defaults[dev] = PyLong_AsVoidPtr(h);
  if (PyErr_Occurred()) return NULL;
  Py_INCREF(obj);
  Py_XSETREF(e->default_st[dev], obj);
  Py_RETURN_NONE;
}

/* The gpu table's `copy` entry when it can be RECORDED instead of launched
 * (tidepool_plugin._try_lazy; ops._dtype_convert, ops.py:121-124): standard
 * mode, a lossless dtype change from a gpu source into a fresh dense gpu
 * destination of the same device, neither with a pending copy.  Returns
 * True when recorded, None when the Python entry must handle the call. */
static PyObject* entries_copy_(Entries* e, PyObject* const* args, Py_ssize_t nargs);
static PyObject* entries_copy(Entries* e, PyObject* const* args, Py_ssize_t nargs) {
  const long long t0 = now_ns();
  PyObject* r = entries_copy_(e, args, nargs);
  T_copy += now_ns() - t0;
  return r;
}
static PyObject* entries_copy_(Entries* e, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 7) {
    PyErr_SetString(PyExc_TypeError, "copy(plan, d_buf, store, a_buf, a_unpack, fn, bases)");
    return NULL;
  }
  PyObject *plan = args[0], *store = args[2], *a_unpack = args[4], *bases = args[6];
#define FALLBACK()   \
  do {               \
    PyErr_Clear();   \
    e->n_fallback++; \
    Py_RETURN_NONE;  \
  } while (0)
  if (!e->lazy_cls) FALLBACK();
  PyObject* sc[3];
  PyObject* const snames[3] = {S_pack, S_mode, S_ctx};
  int r = closure_cells(e, store, S_store_tag, snames, 3, sc);
  if (r == -2) return NULL;
  if (r < 0 || !sc[0]) FALLBACK();
  if (sc[1] && sc[1] != S_standard && PyUnicode_Compare(sc[1], S_standard) != 0) FALLBACK();
  CodecInfo cd, ca;
  if (codec_info(e, sc[0], &cd) || codec_info(e, a_unpack, &ca)) FALLBACK();
  PyObject* dobj = PyDict_GetItemWithError(e->codec_objs, sc[0]);
  PyObject* aobj = PyDict_GetItemWithError(e->codec_objs, a_unpack);
  if (!dobj || !aobj || !PyTuple_Check(dobj) || !PyTuple_Check(aobj)) FALLBACK();
  PyObject *dd = PyTuple_GET_ITEM(dobj, 0), *da = PyTuple_GET_ITEM(aobj, 0);
  if (dd == da) FALLBACK();
  if (cd.wire < 0 || cd.wire >= 32 || ca.wire < 0 || ca.wire >= 32 ||
      !PyBytes_AS_STRING(e->lossless)[ca.wire * 32 + cd.wire])
    FALLBACK();
  DevBuf *bd = devbuf_of(args[1]), *ba = devbuf_of(args[3]);
  if (!bd || !ba || ba->dev != bd->dev || ba->ptr == bd->ptr) FALLBACK();
  const int dev = bd->dev;
  if (!PyTuple_Check(bases) || PyTuple_GET_SIZE(bases) != 2) FALLBACK();
  int64_t b0 = PyLong_AsLongLong(PyTuple_GET_ITEM(bases, 0));
  int64_t b1 = PyLong_AsLongLong(PyTuple_GET_ITEM(bases, 1));
  if (PyErr_Occurred() || b0 != 0) FALLBACK();
  /* dense destination, non-empty (a fresh tensor_create layout) */
  int64_t ext[TPG_MAX_DIMS], s0[TPG_MAX_DIMS], s1[TPG_MAX_DIMS];
  PyObject *pe = PyObject_GetAttr(plan, S_extents), *ps = PyObject_GetAttr(plan, S_strides);
  int nd = pe ? i64_seq(pe, ext, TPG_MAX_DIMS) : -1;
  int ok = nd >= 0 && ps && PySequence_Check(ps) && PySequence_Size(ps) == 2;
  PyObject *v0 = NULL, *v1 = NULL;
  if (ok) {
    v0 = PySequence_GetItem(ps, 0);
    v1 = PySequence_GetItem(ps, 1);
    ok = v0 && v1 && i64_seq(v0, s0, TPG_MAX_DIMS) == nd && i64_seq(v1, s1, TPG_MAX_DIMS) == nd;
  }
  int64_t step = cd.size, total = 1;
  for (int i = 0; ok && i < nd; ++i) {
    total *= ext[i];
    if (ext[i] == 1) continue;
    if (s0[i] != step) ok = 0;
    step *= ext[i];
  }
  if (!ok || total == 0) {
    Py_XDECREF(pe);
    Py_XDECREF(ps);
    Py_XDECREF(v0);
    Py_XDECREF(v1);
    FALLBACK();
  }
  /* neither side may have a pending copy */
  PyObject *kd = PyLong_FromVoidPtr(bd->ptr), *ka = PyLong_FromVoidPtr(ba->ptr);
  int busy = !kd || !ka || PyDict_Contains(e->lazy, kd) == 1 ||
             PyDict_Contains(e->lazy_by_src, kd) == 1 || PyDict_Contains(e->lazy, ka) == 1;
  /* the stream the copy is recorded on (rt.current) */
  PyObject* st = busy ? NULL : PyObject_GetAttr(e->tls, S_stream);
  if (!busy && !st) PyErr_Clear();
  if (!busy && st == Py_None) Py_CLEAR(st);
  if (!busy && st) {
    int bad = 0;
    PyObject* sdev = PyObject_GetAttr(st, S_device);
    int64_t sidx = sdev ? attr_i64(sdev, S_index, &bad) : (bad = 1, 0);
    Py_XDECREF(sdev);
    if (bad) busy = 1;
    else if (sidx != dev) Py_CLEAR(st);
  }
  if (!busy && !st) {
    st = e->default_st[dev];
    Py_XINCREF(st);
    if (!st) busy = 1;
  }
  if (busy) {
    Py_XDECREF(kd);
    Py_XDECREF(ka);
    Py_XDECREF(st);
    Py_XDECREF(pe);
    Py_XDECREF(ps);
    Py_XDECREF(v0);
    Py_XDECREF(v1);
    FALLBACK();
  }
  e->pool->seq++; /* rt.current() */
  PyObject* lz = PyObject_CallNoArgs(e->lazy_cls);
  int err = !lz;
  if (lz && !PyObject_TypeCheck(lz, &LazyRecordType)) {
    PyErr_SetString(PyExc_TypeError, "the copy record class must derive from LazyRecord");
    err = 1;
  }
  if (!err) {
    LazyRecord* r = (LazyRecord*)lz;
#define LR_SET(field, val) \
  do {                     \
    PyObject* v_ = (val);  \
    Py_XINCREF(v_);        \
    Py_XSETREF(r->field, v_); \
  } while (0)
    LR_SET(plan, plan);
    LR_SET(stream, st);
    LR_SET(dst_ptr, kd);
    LR_SET(src_ptr, ka);
    LR_SET(keep, args[3]);
    LR_SET(src_dtype, da);
    LR_SET(dst_dtype, dd);
    LR_SET(src_order, PyTuple_GET_ITEM(aobj, 1));
#undef LR_SET
    r->device = dev;
    r->ddt = cd.wire;
    r->dbig = cd.big;
    r->sbase = (long long)(intptr_t)ba->ptr;
    r->soff = b1;
    r->sdt = ca.wire;
    r->sbig = ca.big;
    memset(&r->pack, 0, sizeof r->pack);
    r->pack.ne = nd;
    r->pack.sbase = r->sbase;
    r->pack.soff = b1;
    r->pack.sdt = ca.wire;
    r->pack.sbig = ca.big;
    for (int i = 0; i < nd; ++i) {
      r->pack.E[i] = ext[i];
      r->pack.T[i] = s0[i];
      r->pack.S[i] = s1[i];
    }
    r->has_pack = 1;
  }
  PyObject* set = NULL;
  if (!err) err = PyDict_SetItem(e->lazy, kd, lz) < 0;
  if (!err) {
    set = PyDict_GetItemWithError(e->lazy_by_src, ka);
    if (set) {
      err = PySet_Add(set, kd) < 0;
    } else if (!PyErr_Occurred()) {
      set = PySet_New(NULL);
      err = !set || PySet_Add(set, kd) < 0 || PyDict_SetItem(e->lazy_by_src, ka, set) < 0;
      Py_XDECREF(set);
    } else {
      err = 1;
    }
  }
  if (!err) e->n_lazy++;
  Py_XDECREF(lz);
  Py_DECREF(kd);
  Py_DECREF(ka);
  Py_DECREF(st);
  Py_XDECREF(pe);
  Py_XDECREF(ps);
  Py_XDECREF(v0);
  Py_XDECREF(v1);
  if (err) return NULL;
  e->n_fast++;
  Py_RETURN_TRUE;
#undef FALLBACK
}

static PyObject* entries_counts(Entries* e, PyObject* unused) {
  return Py_BuildValue("{s:L,s:L,s:L,s:L,s:L,s:L,s:L,s:L,s:L}", "fast", e->n_fast, "fallback",
                       e->n_fallback, "fused", e->n_fused, "lazy", e->n_lazy, "ns_allocate",
                       T_alloc, "ns_release", T_release, "ns_binary", T_binary, "ns_copy", T_copy,
                       "ns_launch", T_launch);
}

static PyMethodDef entries_methods[] = {
    {"binary", (PyCFunction)(void (*)(void))entries_binary, METH_FASTCALL,
     "binary(op, plan, d_buf, store, a_buf, a_unpack, b_buf, b_unpack, fn, bases) -> rc | None"},
    {"set_default_stream", (PyCFunction)entries_set_default, METH_VARARGS,
     "set_default_stream(device, handle, stream object)"},
    {"copy", (PyCFunction)(void (*)(void))entries_copy, METH_FASTCALL,
     "copy(plan, d_buf, store, a_buf, a_unpack, fn, bases) -> True | None"},
    {"set_copy_support", (PyCFunction)entries_set_copy_support, METH_VARARGS,
     "set_copy_support(lazy class, {codec fn: (dtype, order)}, lossless table bytes)"},
    {"counts", (PyCFunction)entries_counts, METH_NOARGS, "fast / fallback call counts"},
    {"entry", (PyCFunction)entries_entry, METH_VARARGS,
     "entry(kind, op code, python entry) -> table callable (kind 0 binary, 1 copy, 2 unary)"},
    {"set_unary", (PyCFunction)entries_set_unary, METH_O, "set_unary(tpg_unary address)"},
    {"set_reduce", (PyCFunction)entries_set_reduce, METH_O, "set_reduce(tpg_reduce address)"},
    {NULL}};

static int intern_names(void) {
#define IN(var, str) \
  if (!(var = PyUnicode_InternFromString(str))) return -1;
  IN(S_standard, "standard");
  IN(S_stream, "stream");
  IN(S_device, "device");
  IN(S_index, "index");
  IN(S_handle, "handle");
  IN(S_status_sink, "status_sink");
  IN(S_extents, "extents");
  IN(S_strides, "strides");
  IN(S_fused, "fused");
  IN(S_src_ptr, "src_ptr");
  IN(S_cext, "cext");
  IN(S_cdst, "cdst");
  IN(S_csrc, "csrc");
  IN(S_sbase, "sbase");
  IN(S_soff, "soff");
  IN(S_sdt, "sdt");
  IN(S_sbig, "sbig");
  IN(S_cpack, "cpack");
  IN(S_pack, "pack");
  IN(S_mode, "mode");
  IN(S_ctx, "ctx");
  IN(S_status, "status");
  IN(S_store_tag, "#store");
  IN(S_status_tag, "#status");
#undef IN
  for (int i = 0; i < 19; ++i)
    if (!(L_names[i] = PyUnicode_InternFromString(L_str[i]))) return -1;
  return 0;
}

static PyObject* set_alloc_error(PyObject* m, PyObject* cls) {
  Py_XDECREF(AllocError);
  Py_INCREF(cls);
  AllocError = cls;
  Py_RETURN_NONE;
}

static PyMethodDef module_methods[] = {
    {"set_allocation_error", set_alloc_error, METH_O,
     "exception class raised when a managed allocation fails"},
    {NULL}};

static struct PyModuleDef moddef = {PyModuleDef_HEAD_INIT, "_tpg_pyfast",
                                    "drop-in plugin host fast path (see tpg_pyfast.c)", -1,
                                    module_methods};

PyMODINIT_FUNC PyInit__tpg_pyfast(void) {
  DevBufType.tp_name = "_tpg_pyfast.DevBuf";
  DevBufType.tp_basicsize = sizeof(DevBuf);
  DevBufType.tp_flags = Py_TPFLAGS_DEFAULT | Py_TPFLAGS_HAVE_GC;
  DevBufType.tp_doc = "host-visible buffer over a managed gpu block";
  DevBufType.tp_dealloc = (destructor)devbuf_dealloc;
  DevBufType.tp_traverse = (traverseproc)devbuf_traverse;
  DevBufType.tp_clear = (inquiry)devbuf_clear;
  DevBufType.tp_as_buffer = &devbuf_as_buffer;
  DevBufType.tp_as_sequence = &devbuf_as_seq;
  DevBufType.tp_getset = devbuf_getset;
  DevBufType.tp_weaklistoffset = offsetof(DevBuf, weakreflist);
  DevBufType.tp_dictoffset = offsetof(DevBuf, dict);
  if (PyType_Ready(&DevBufType) < 0) return NULL;

  BlockPoolType.tp_name = "_tpg_pyfast.BlockPool";
  BlockPoolType.tp_basicsize = sizeof(BlockPool);
  BlockPoolType.tp_flags = Py_TPFLAGS_DEFAULT | Py_TPFLAGS_HAVE_GC;
  BlockPoolType.tp_doc = "per-registration managed block cache";
  BlockPoolType.tp_new = PyType_GenericNew;
  BlockPoolType.tp_init = (initproc)pool_init;
  BlockPoolType.tp_dealloc = (destructor)pool_dealloc;
  BlockPoolType.tp_traverse = (traverseproc)pool_traverse;
  BlockPoolType.tp_clear = (inquiry)pool_clear;
  BlockPoolType.tp_methods = pool_methods;
  if (PyType_Ready(&BlockPoolType) < 0) return NULL;

  if (intern_names() < 0) return NULL;
  LazyRecordType.tp_name = "_tpg_pyfast.LazyRecord";
  LazyRecordType.tp_basicsize = sizeof(LazyRecord);
  LazyRecordType.tp_flags = Py_TPFLAGS_DEFAULT | Py_TPFLAGS_BASETYPE | Py_TPFLAGS_HAVE_GC;
  LazyRecordType.tp_doc = "a recorded lossless gpu->gpu copy (base of tidepool_plugin._Lazy)";
  LazyRecordType.tp_new = PyType_GenericNew;
  LazyRecordType.tp_dealloc = (destructor)lazyrec_dealloc;
  LazyRecordType.tp_traverse = (traverseproc)lazyrec_traverse;
  LazyRecordType.tp_clear = (inquiry)lazyrec_clear;
  LazyRecordType.tp_members = lazyrec_members;
  if (PyType_Ready(&LazyRecordType) < 0) return NULL;
  if (!(S_alloc_count = PyUnicode_InternFromString("alloc_count"))) return NULL;
  if (!(ONE = PyLong_FromLong(1))) return NULL;
  AllocatorType.tp_name = "_tpg_pyfast.Allocator";
  AllocatorType.tp_basicsize = sizeof(Allocator);
  AllocatorType.tp_flags = Py_TPFLAGS_DEFAULT | Py_TPFLAGS_HAVE_GC;
  AllocatorType.tp_doc = "Device.allocate of one gpu device";
  AllocatorType.tp_call = (ternaryfunc)allocator_call;
  AllocatorType.tp_dealloc = (destructor)allocator_dealloc;
  AllocatorType.tp_traverse = (traverseproc)allocator_traverse;
  AllocatorType.tp_clear = (inquiry)allocator_clear;
  if (PyType_Ready(&AllocatorType) < 0) return NULL;
  EntriesType.tp_name = "_tpg_pyfast.Entries";
  EntriesType.tp_basicsize = sizeof(Entries);
  EntriesType.tp_flags = Py_TPFLAGS_DEFAULT | Py_TPFLAGS_HAVE_GC;
  EntriesType.tp_doc = "C fast path of the gpu table's binary entry";
  EntriesType.tp_new = PyType_GenericNew;
  EntriesType.tp_init = (initproc)entries_init;
  EntriesType.tp_dealloc = (destructor)entries_dealloc;
  EntriesType.tp_traverse = (traverseproc)entries_traverse;
  EntriesType.tp_clear = (inquiry)entries_clear;
  EntriesType.tp_methods = entries_methods;
  if (PyType_Ready(&EntriesType) < 0) return NULL;
  if (!(S_profile = PyUnicode_InternFromString("profile"))) return NULL;
  if (!(S_complex_fn = PyUnicode_InternFromString("complex_fn"))) return NULL;
  if (!(S_complex_tag = PyUnicode_InternFromString("#complex"))) return NULL;
  if (!(S_p = PyUnicode_InternFromString("p"))) return NULL;
  if (!(S_norm_tag = PyUnicode_InternFromString("#norm"))) return NULL;
  if (!(S_check = PyUnicode_InternFromString("check"))) return NULL;
  if (!(S_kernel = PyUnicode_InternFromString("kernel"))) return NULL;
  FastEntryType.tp_name = "_tpg_pyfast.FastEntry";
  FastEntryType.tp_basicsize = sizeof(FastEntry);
  FastEntryType.tp_flags = Py_TPFLAGS_DEFAULT | Py_TPFLAGS_HAVE_GC;
  FastEntryType.tp_doc = "gpu table entry: C fast path, Python entry otherwise";
  FastEntryType.tp_call = (ternaryfunc)fastentry_call;
  FastEntryType.tp_dealloc = (destructor)fastentry_dealloc;
  FastEntryType.tp_traverse = (traverseproc)fastentry_traverse;
  FastEntryType.tp_clear = (inquiry)fastentry_clear;
  if (PyType_Ready(&FastEntryType) < 0) return NULL;

  PyObject* m = PyModule_Create(&moddef);
  if (!m) return NULL;
  Py_INCREF(&DevBufType);
  PyModule_AddObject(m, "DevBuf", (PyObject*)&DevBufType);
  Py_INCREF(&BlockPoolType);
  PyModule_AddObject(m, "BlockPool", (PyObject*)&BlockPoolType);
  Py_INCREF(&EntriesType);
  PyModule_AddObject(m, "Entries", (PyObject*)&EntriesType);
  Py_INCREF(&LazyRecordType);
  PyModule_AddObject(m, "LazyRecord", (PyObject*)&LazyRecordType);
  return m;
}
