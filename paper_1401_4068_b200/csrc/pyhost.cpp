// _pyhost: CPython helper for the host side of batch_search (not part of the
// C ABI).  Reading the data pointer of ten thousand numpy chunks one Python
// attribute at a time costs ~2 us each (arr.ctypes.data); here the buffer
// protocol does it in C, so a batch of many small chunks hands its pointers
// and sizes to ente_host_gather without a per-chunk Python step.
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <string.h>

// scan(seq) -> (addresses: bytes of int64, sizes: bytes of int64, rows: bytes of int64)
// Every item must expose a C-contiguous buffer (numpy arrays do); rows is
// the first dimension (1 for a 0-d buffer).  The caller keeps the items
// alive while the addresses are in use.
static PyObject *scan(PyObject *, PyObject *arg) {
    PyObject *seq = PySequence_Fast(arg, "scan expects a sequence of arrays");
    if (!seq) return nullptr;
    const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
    PyObject *addr = PyBytes_FromStringAndSize(nullptr, n * 8);
    PyObject *size = PyBytes_FromStringAndSize(nullptr, n * 8);
    PyObject *rows = PyBytes_FromStringAndSize(nullptr, n * 8);
    if (!addr || !size || !rows) {
        Py_XDECREF(addr);
        Py_XDECREF(size);
        Py_XDECREF(rows);
        Py_DECREF(seq);
        return nullptr;
    }
    int64_t *pa = reinterpret_cast<int64_t *>(PyBytes_AS_STRING(addr));
    int64_t *ps = reinterpret_cast<int64_t *>(PyBytes_AS_STRING(size));
    int64_t *pr = reinterpret_cast<int64_t *>(PyBytes_AS_STRING(rows));
    PyObject **items = PySequence_Fast_ITEMS(seq);
    for (Py_ssize_t i = 0; i < n; ++i) {
        Py_buffer v;
        if (PyObject_GetBuffer(items[i], &v, PyBUF_C_CONTIGUOUS) != 0) {
            Py_DECREF(addr);
            Py_DECREF(size);
            Py_DECREF(rows);
            Py_DECREF(seq);
            return nullptr;
        }
        pa[i] = (int64_t)(intptr_t)v.buf;
        ps[i] = (int64_t)v.len;
        pr[i] = v.ndim > 0 ? (int64_t)v.shape[0] : 1;
        PyBuffer_Release(&v);
    }
    Py_DECREF(seq);
    PyObject *out = PyTuple_Pack(3, addr, size, rows);
    Py_DECREF(addr);
    Py_DECREF(size);
    Py_DECREF(rows);
    return out;
}

static PyMethodDef kMethods[] = {
    {"scan", scan, METH_O, "(addresses, sizes, rows) of C-contiguous buffers as int64 bytes"},
    {nullptr, nullptr, 0, nullptr},
};

static struct PyModuleDef kModule = {PyModuleDef_HEAD_INIT, "_pyhost", nullptr, -1, kMethods};

PyMODINIT_FUNC PyInit__pyhost(void) { return PyModule_Create(&kModule); }
