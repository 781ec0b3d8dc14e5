/* hostlist.c -- CPython helper of the host API: the data addresses and
 * lengths of a list of `bytes` documents, read through the C API
 * (PyBytes_AS_STRING / PyBytes_GET_SIZE) in one call.
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
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

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

static PyMethodDef methods[] = {
    {"ptrs_lens", ptrs_lens, METH_VARARGS, "data addresses and lengths of a list of bytes"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_hostlist", NULL, -1, methods};

PyMODINIT_FUNC PyInit__hostlist(void) { return PyModule_Create(&module); }
