/* counts_dict.c — the reference's CountsTable.counts ({bitstring: count}, qubit 0 leftmost,
 * statevec.py:64-73, 229-234) built straight from the sampler's (index, count) int64 arrays:
 * one ASCII str per outcome written in place (8 characters per index byte from a table)
 * and one dict insert, instead of numpy string arrays and per-item Python conversions
 * (~30 ms -> a few ms for 1e5 outcomes on the GPU box's host). Host-side formatting only. */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <string.h>

static char bit_chars[256][8];

static PyObject* counts_dict(PyObject* self, PyObject* args) {
    (void)self;
    Py_buffer bi, bc;
    int n;
    if (!PyArg_ParseTuple(args, "y*y*i", &bi, &bc, &n)) return NULL;
    PyObject* d = NULL;
    if (bi.len != bc.len || bi.len % 8 != 0 || n < 0 || n > 64) {
        PyErr_SetString(PyExc_ValueError, "counts_dict: int64 index / count arrays of equal length, 0 <= n_qubits <= 64");
        goto done;
    }
    d = _PyDict_NewPresized(bi.len / 8);  /* one allocation for all outcomes */
    if (!d) goto done;
    const int64_t* idx = (const int64_t*)bi.buf;
    const int64_t* cnt = (const int64_t*)bc.buf;
    const Py_ssize_t m = bi.len / 8;
    for (Py_ssize_t i = 0; i < m; ++i) {
        PyObject* s = PyUnicode_New(n, 127);
        if (!s) { Py_CLEAR(d); goto done; }
        char* out = (char*)PyUnicode_DATA(s);
        const uint64_t v = (uint64_t)idx[i];
        for (int b = 0; b < n; b += 8) {
            const int w = n - b < 8 ? n - b : 8;
            memcpy(out + b, bit_chars[(v >> b) & 0xffu], (size_t)w);
        }
        PyObject* c = PyLong_FromLongLong(cnt[i]);
        if (!c || PyDict_SetItem(d, s, c) < 0) {
            Py_XDECREF(c);
            Py_DECREF(s);
            Py_CLEAR(d);
            goto done;
        }
        Py_DECREF(c);
        Py_DECREF(s);
    }
done:
    PyBuffer_Release(&bi);
    PyBuffer_Release(&bc);
    return d;
}

static PyMethodDef methods[] = {
    {"counts_dict", counts_dict, METH_VARARGS,
     "counts_dict(indices_int64, counts_int64, n_qubits) -> {bitstring (qubit 0 leftmost): count}"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_counts", NULL, -1, methods, NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__counts(void) {
    for (int v = 0; v < 256; ++v)
        for (int k = 0; k < 8; ++k) bit_chars[v][k] = (char)('0' + ((v >> k) & 1));
    return PyModule_Create(&module);
}
