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
 *   BlockPool(fns, blocks, lazy, lazy_by_src, drop_lazy, cache_bytes,
 *             max_pending)
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

typedef int (*f_malloc_managed)(int, size_t, void**);
typedef int (*f_free_managed)(void*);
typedef int (*f_ev_create)(void**);
typedef int (*f_ev_record)(void*, void*);
typedef int (*f_ev_query)(void*);
typedef int (*f_ev_sync)(void*);

#define MAX_DEV 64

typedef struct Marker {
  void* ev;
  long refs;
} Marker;

typedef struct {
  void* handle;
  Marker* marker;
  uint64_t marker_seq;
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
  PyObject* blocks;       /* dict ptr -> (device, cap) */
  PyObject* lazy;         /* dict dst ptr -> record */
  PyObject* lazy_by_src;  /* dict src ptr -> set */
  PyObject* drop_lazy;    /* callable(ptr) */
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
static PyObject* AllocError;  /* set by the plugin: the reference's AllocationError */

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
      for (int s = 0; s < p->nstreams[d]; ++s)
        if (p->streams[d][s].marker == m) p->streams[d][s].marker = NULL;
    if (p->nevpool == p->aevpool) {
      size_t na = p->aevpool ? 2 * p->aevpool : 64;
      void** nv = (void**)realloc(p->evpool, na * sizeof(void*));
      if (nv) {
        p->evpool = nv;
        p->aevpool = na;
      }
    }
    if (p->nevpool < p->aevpool) p->evpool[p->nevpool++] = m->ev;
    free(m);
  }
  free(e->evs);
  e->evs = NULL;
  e->nev = 0;
}

static int entry_done(BlockPool* p, Entry* e) {
  for (int i = 0; i < e->nev; ++i)
    if (p->ev_query(e->evs[i]->ev) != 0) return 0;
  return 1;
}

static void entry_wait(BlockPool* p, Entry* e) {
  Py_BEGIN_ALLOW_THREADS
  for (int i = 0; i < e->nev; ++i) p->ev_sync(e->evs[i]->ev);
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
  /* a pending lazy copy into / out of this block is dead with it */
  if (p->drop_lazy != Py_None &&
      (PyDict_Contains(p->lazy, k) == 1 || PyDict_Contains(p->lazy_by_src, k) == 1)) {
    PyObject* r = PyObject_CallOneArg(p->drop_lazy, k);
    if (!r) PyErr_WriteUnraisable(p->drop_lazy);
    Py_XDECREF(r);
  }
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

static void release_block(BlockPool* p, void* ptr, size_t cap, int dev) {
  p->n_release++;
  blocks_del(p, ptr);
  SizeClass* c = find_class(p, dev, cap, 1);
  int ns = p->nstreams[dev];
  Entry e = {ptr, 0, NULL};
  if (ns) {
    e.evs = (Marker**)malloc(sizeof(Marker*) * ns);
    for (int s = 0; e.evs && s < ns; ++s) {
      StreamRec* st = &p->streams[dev][s];
      if (!st->marker || st->marker_seq != p->seq) {
        Marker* m = (Marker*)calloc(1, sizeof(Marker));
        if (!m) break;
        if (p->nevpool) {
          m->ev = p->evpool[--p->nevpool];
        } else if (p->ev_create(&m->ev) != 0) {
          free(m);
          break;
        }
        p->ev_record(m->ev, st->handle);
        st->marker = m;
        st->marker_seq = p->seq;
      }
      st->marker->refs++;
      e.evs[e.nev++] = st->marker;
    }
  }
  if (!c) { /* out of host memory: drop the block */
    Py_BEGIN_ALLOW_THREADS
    for (int i = 0; i < e.nev; ++i) p->ev_sync(e.evs[i]->ev);
    Py_END_ALLOW_THREADS
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
  PyObject *fns, *blocks, *lazy, *lbs, *drop;
  long long limit;
  int maxp;
  if (!PyArg_ParseTuple(args, "OO!O!O!OLi", &fns, &PyDict_Type, &blocks, &PyDict_Type, &lazy,
                        &PyDict_Type, &lbs, &drop, &limit, &maxp))
    return -1;
  if (!PyTuple_Check(fns) || PyTuple_GET_SIZE(fns) != 6) {
    PyErr_SetString(PyExc_TypeError, "fns: 6 function addresses");
    return -1;
  }
  void* f[6];
  for (int i = 0; i < 6; ++i) {
    f[i] = PyLong_AsVoidPtr(PyTuple_GET_ITEM(fns, i));
    if (!f[i]) {
      if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "null function address");
      return -1;
    }
  }
  p->malloc_managed = (f_malloc_managed)f[0];
  p->free_managed = (f_free_managed)f[1];
  p->ev_create = (f_ev_create)f[2];
  p->ev_record = (f_ev_record)f[3];
  p->ev_query = (f_ev_query)f[4];
  p->ev_sync = (f_ev_sync)f[5];
  Py_INCREF(blocks);
  Py_INCREF(lazy);
  Py_INCREF(lbs);
  Py_INCREF(drop);
  p->blocks = blocks;
  p->lazy = lazy;
  p->lazy_by_src = lbs;
  p->drop_lazy = drop;
  p->cache_limit = limit;
  p->max_pending = maxp;
  return 0;
}

static int pool_traverse(BlockPool* p, visitproc visit, void* arg) {
  Py_VISIT(p->blocks);
  Py_VISIT(p->lazy);
  Py_VISIT(p->lazy_by_src);
  Py_VISIT(p->drop_lazy);
  return 0;
}

static int pool_clear(BlockPool* p) {
  Py_CLEAR(p->blocks);
  Py_CLEAR(p->lazy);
  Py_CLEAR(p->lazy_by_src);
  Py_CLEAR(p->drop_lazy);
  return 0;
}

static void pool_dealloc(BlockPool* p) {
  PyObject_GC_UnTrack(p);
  pool_clear(p);
  /* cached blocks and events stay with the CUDA context (process exit) */
  Py_TYPE(p)->tp_free((PyObject*)p);
}

static PyObject* pool_allocate(BlockPool* p, PyObject* args) {
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
    {"bump", (PyCFunction)pool_bump, METH_NOARGS, "start a new launch epoch"},
    {"trim", (PyCFunction)pool_trim, METH_VARARGS, "trim(device, keep_bytes)"},
    {"stats", (PyCFunction)pool_stats, METH_NOARGS, "counters"},
    {"cached_bytes", (PyCFunction)pool_cached_bytes, METH_VARARGS, "cached bytes of a device"},
    {NULL}};

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

  PyObject* m = PyModule_Create(&moddef);
  if (!m) return NULL;
  Py_INCREF(&DevBufType);
  PyModule_AddObject(m, "DevBuf", (PyObject*)&DevBufType);
  Py_INCREF(&BlockPoolType);
  PyModule_AddObject(m, "BlockPool", (PyObject*)&BlockPoolType);
  return m;
}
