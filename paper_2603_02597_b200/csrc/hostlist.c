/* hostlist.c -- CPython helper of the host API.
 *
 * 1. The data addresses and lengths of a list of `bytes` documents, read
 *    through the C API (PyBytes_AS_STRING / PyBytes_GET_SIZE) in one call.
 * 2. encode_one: the single-document latency path (tokenize_batch with one
 *    input) as one C call -- the document's bytes object, its chunk offsets,
 *    gpubpe_encode_host (GIL released) and gpubpe_query -- so the Python
 *    side pays one call instead of a dozen ctypes conversions.
 *
 * The batch path (chunker.tokenize_batch -> device.encode_ptrs_host ->
 * gpubpe_encode_host_gather) hands the documents' own buffers to the native
 * gather, so it needs each object's data pointer.  Reading it here replaces
 * any assumption about the object layout on the Python side.
 *
 *   _hostlist.ptrs_lens(list, ptrs_addr, lens_addr) -> total bytes
 *     list       a list of exact `bytes` objects (TypeError otherwise)
 *     ptrs_addr  address of uint64[len(list)]: data addresses (written)
 *     lens_addr  address of uint64[len(list)]: lengths (written)
 * The caller keeps the list alive while the addresses are used.
 *
 * 3. split_views: the per-document result arrays of a batch (BatchResult.
 *    token_ids) as views of the one result array, built in C (a Python
 *    slicing loop costs ~0.1 us per document; C2 has 4,096).
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#define NPY_NO_DEPRECATED_API NPY_1_7_API_VERSION
#include <numpy/arrayobject.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/gpubpe.h"

static PyObject *ptrs_lens(PyObject *self, PyObject *args) {
    PyObject *lst;
    unsigned long long pa, la;
    (void)self;
    if (!PyArg_ParseTuple(args, "O!KK", &PyList_Type, &lst, &pa, &la)) return NULL;
    const Py_ssize_t n = PyList_GET_SIZE(lst);
    uint64_t *ptrs = (uint64_t *)(uintptr_t)pa, *lens = (uint64_t *)(uintptr_t)la;
    if (n > 0 && (!ptrs || !lens)) {
        PyErr_SetString(PyExc_ValueError, "ptrs_lens: null output buffer");
        return NULL;
    }
    unsigned long long total = 0;
    for (Py_ssize_t i = 0; i < n; ++i) {
        PyObject *b = PyList_GET_ITEM(lst, i);
        if (!PyBytes_CheckExact(b)) {
            PyErr_Format(PyExc_TypeError, "ptrs_lens: item %zd is %.80s, not bytes", i, Py_TYPE(b)->tp_name);
            return NULL;
        }
        const Py_ssize_t len = PyBytes_GET_SIZE(b);
        ptrs[i] = (uint64_t)(uintptr_t)PyBytes_AS_STRING(b);
        lens[i] = (uint64_t)len;
        total += (unsigned long long)len;
    }
    return PyLong_FromUnsignedLongLong(total);
}

typedef int (*encode_host_fn)(gpubpe_ctx *, const uint8_t *, uint64_t, const int64_t *, uint64_t, uint64_t,
                              uint64_t, uint32_t *, int64_t *, uint64_t *, float *, void *);
typedef int (*query_fn)(gpubpe_ctx *, void *, gpubpe_stats *);
static encode_host_fn g_encode_host;
static query_fn g_query;

/* bind(encode_host_addr, query_addr): the libgpubpe.so entry points (their
 * addresses from the ctypes binding, so this module needs no link to it). */
static PyObject *bind(PyObject *self, PyObject *args) {
    unsigned long long e, q;
    (void)self;
    if (!PyArg_ParseTuple(args, "KK", &e, &q)) return NULL;
    g_encode_host = (encode_host_fn)(uintptr_t)e;
    g_query = (query_fn)(uintptr_t)q;
    Py_RETURN_NONE;
}

/* encode_one(ctx, doc, max_seq_len, chunk_budget, ids_addr, offs_addr, n_units, stream)
 *   -> (rc, n_ids, kernel_ms, stats tuple | None)
 * doc: bytes; n_units = 1 (one unit [0, n)) or ceil(n / chunk_budget) when
 * n > max_seq_len (the reference's fixed-offset chunks, chunker.py:42-53);
 * ids_addr: uint32[>= n], offs_addr: int64[n_units + 1] (written).  rc is the
 * gpubpe status (the caller raises); stats are gpubpe_query's fields. */
static PyObject *encode_one(PyObject *self, PyObject *args) {
    unsigned long long ctx, msl, cb, ids, offs, units, stream;
    PyObject *doc;
    (void)self;
    if (!PyArg_ParseTuple(args, "KO!KKKKKK", &ctx, &PyBytes_Type, &doc, &msl, &cb, &ids, &offs, &units, &stream))
        return NULL;
    if (!g_encode_host || !g_query) {
        PyErr_SetString(PyExc_RuntimeError, "encode_one: bind() first");
        return NULL;
    }
    const uint64_t n = (uint64_t)PyBytes_GET_SIZE(doc);
    const uint8_t *data = (const uint8_t *)PyBytes_AS_STRING(doc);
    if (units < 1 || (units > 1 && (cb == 0 || (n + cb - 1) / cb != units))) {
        PyErr_SetString(PyExc_ValueError, "encode_one: n_units does not match the chunking");
        return NULL;
    }
    int64_t one[2] = {0, (int64_t)n};
    int64_t *doc_offs = one;
    if (units > 1) {
        doc_offs = (int64_t *)malloc((units + 1) * sizeof(int64_t));
        if (!doc_offs) return PyErr_NoMemory();
        for (uint64_t k = 0; k < units; ++k) doc_offs[k] = (int64_t)(k * cb);
        doc_offs[units] = (int64_t)n;
    }
    uint64_t n_ids = 0;
    float ms = 0.f;
    gpubpe_stats st;
    int rc, rq = 1;
    Py_BEGIN_ALLOW_THREADS
    rc = g_encode_host((gpubpe_ctx *)(uintptr_t)ctx, data, n, doc_offs, units, msl, cb, (uint32_t *)(uintptr_t)ids,
                       (int64_t *)(uintptr_t)offs, &n_ids, &ms, (void *)(uintptr_t)stream);
    if (rc == 0) rq = g_query((gpubpe_ctx *)(uintptr_t)ctx, (void *)(uintptr_t)stream, &st);
    Py_END_ALLOW_THREADS
    if (doc_offs != one) free(doc_offs);
    if (rc != 0 || rq != 0) return Py_BuildValue("iKdO", rc ? rc : rq, (unsigned long long)n_ids, (double)ms, Py_None);
    const uint64_t *f = &st.n_bytes;
    PyObject *t = PyTuple_New(sizeof(gpubpe_stats) / 8);
    if (!t) return NULL;
    for (Py_ssize_t i = 0; i < (Py_ssize_t)(sizeof(gpubpe_stats) / 8); ++i)
        PyTuple_SET_ITEM(t, i, PyLong_FromUnsignedLongLong(f[i]));
    return Py_BuildValue("iKdN", 0, (unsigned long long)n_ids, (double)ms, t);
}

/* split_views(arr, offs_addr, n) -> list of n views arr[offs[i]:offs[i+1]]
 * arr: a 1-D C-contiguous numpy array (each view keeps it alive);
 * offs_addr: address of int64[n + 1], ascending, within [0, len(arr)]. */
static PyObject *split_views(PyObject *self, PyObject *args) {
    PyArrayObject *arr;
    unsigned long long oa;
    Py_ssize_t n;
    (void)self;
    if (!PyArg_ParseTuple(args, "O!Kn", &PyArray_Type, &arr, &oa, &n)) return NULL;
    if (PyArray_NDIM(arr) != 1 || !PyArray_IS_C_CONTIGUOUS(arr) || n < 0 || (n > 0 && !oa)) {
        PyErr_SetString(PyExc_ValueError, "split_views: a 1-D contiguous array and n + 1 offsets");
        return NULL;
    }
    const int64_t *o = (const int64_t *)(uintptr_t)oa;
    const npy_intp len = PyArray_DIM(arr, 0), isz = PyArray_ITEMSIZE(arr);
    for (Py_ssize_t i = 0; i < n; ++i)
        if (o[i] < 0 || o[i] > o[i + 1] || o[i + 1] > len) {
            PyErr_SetString(PyExc_ValueError, "split_views: offsets out of order or range");
            return NULL;
        }
    PyObject *out = PyList_New(n);
    if (!out) return NULL;
    char *data = PyArray_BYTES(arr);
    PyArray_Descr *descr = PyArray_DESCR(arr);
    const int flags = PyArray_FLAGS(arr) & (NPY_ARRAY_C_CONTIGUOUS | NPY_ARRAY_ALIGNED | NPY_ARRAY_WRITEABLE);
    for (Py_ssize_t i = 0; i < n; ++i) {
        npy_intp dim = (npy_intp)(o[i + 1] - o[i]);
        Py_INCREF(descr);  /* stolen */
        PyObject *v = PyArray_NewFromDescr(&PyArray_Type, descr, 1, &dim, NULL, data + o[i] * isz, flags, NULL);
        if (!v) {
            Py_DECREF(out);
            return NULL;
        }
        Py_INCREF(arr);
        if (PyArray_SetBaseObject((PyArrayObject *)v, (PyObject *)arr) < 0) {  /* steals arr */
            Py_DECREF(v);
            Py_DECREF(out);
            return NULL;
        }
        PyList_SET_ITEM(out, i, v);
    }
    return out;
}

static PyMethodDef methods[] = {
    {"ptrs_lens", ptrs_lens, METH_VARARGS, "data addresses and lengths of a list of bytes"},
    {"bind", bind, METH_VARARGS, "bind the libgpubpe.so entry points"},
    {"encode_one", encode_one, METH_VARARGS, "single-document host encode"},
    {"split_views", split_views, METH_VARARGS, "per-document views of a result array"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_hostlist", NULL, -1, methods};

PyMODINIT_FUNC PyInit__hostlist(void) {
    import_array();
    return PyModule_Create(&module);
}
