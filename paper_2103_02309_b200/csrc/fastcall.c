/* fastcall.c -- the per-tile call of the kernel protocol without Python-level
 * argument handling (CPython extension `paper_2103_02309_b200._fastcall`).
 *
 * The reference renderer calls batch.cast_rays once per 16x16 tile (256 rays)
 * from a thread pool (/root/reference/pkg/src/tetray/render.py:192-207,
 * 300-331, 538-541); batch.cast_rays then calls kernels.cast_rays
 * (batch.py:47-51) and runs its numpy epilogue, all under the GIL.  At that
 * granularity every microsecond the backend holds the GIL is taken from all
 * sixteen threads, and the ctypes wrapper (argument conversion, four output
 * allocations, the start-tet range check in numpy) held it for ~45 us per
 * call.  This function does the same work in C: validates the three inputs
 * (already float32 / int32 and contiguous -- what batch.cast_rays passes),
 * range-checks the start tets, allocates the four outputs and calls
 * tb_cast_rays_host (include/tetb200.h) with the GIL released.  Anything it
 * does not handle (other dtypes or layouts) returns None and the caller takes
 * the general ctypes path; errors raise the same exceptions as that path.
 *
 * The C-ABI entry points are bound by address from the ctypes handle of
 * libtetb200.so (bind()), so both paths call into the one loaded library.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#define NPY_NO_DEPRECATED_API NPY_2_0_API_VERSION
#include <numpy/arrayobject.h>
#include <stdint.h>

typedef int (*cast_host_fn)(void*, int64_t, const float*, const float*, const int32_t*, uint8_t*, int32_t*,
                            int32_t*, int32_t*, int32_t*, double*, int32_t*);
typedef const char* (*last_error_fn)(void);

static cast_host_fn g_cast_host = NULL;
static last_error_fn g_last_error = NULL;
static PyObject* g_error = NULL; /* _lib.TetB200Error */

static PyObject* bind(PyObject* self, PyObject* args) {
  unsigned long long cast_host, last_error;
  PyObject* err;
  if (!PyArg_ParseTuple(args, "KKO", &cast_host, &last_error, &err)) return NULL;
  g_cast_host = (cast_host_fn)(uintptr_t)cast_host;
  g_last_error = (last_error_fn)(uintptr_t)last_error;
  Py_XDECREF(g_error);
  Py_INCREF(err);
  g_error = err;
  Py_RETURN_NONE;
}

/* The array as a C-contiguous, aligned buffer of `type` with `cols` columns
 * (0 = 1-D), or NULL when it is anything else (the caller falls back). */
static PyArrayObject* plain(PyObject* o, int type, int cols) {
  if (!PyArray_Check(o)) return NULL;
  PyArrayObject* a = (PyArrayObject*)o;
  if (PyArray_TYPE(a) != type || !PyArray_IS_C_CONTIGUOUS(a) || !PyArray_ISALIGNED(a)) return NULL;
  if (cols == 0) return PyArray_NDIM(a) == 1 ? a : NULL;
  return (PyArray_NDIM(a) == 2 && PyArray_DIM(a, 1) == cols) ? a : NULL;
}

/* cast4(handle, n_tets, o (n, 3) f32, d (n, 3) f32, start (n,) i32)
 *   -> (status u8, cf i32, tet i32, visited i32) or None */
static PyObject* cast4(PyObject* self, PyObject* args) {
  unsigned long long handle;
  long long n_tets;
  PyObject *oo, *od, *os;
  if (!PyArg_ParseTuple(args, "KLOOO", &handle, &n_tets, &oo, &od, &os)) return NULL;
  PyArrayObject* o = plain(oo, NPY_FLOAT32, 3);
  PyArrayObject* d = plain(od, NPY_FLOAT32, 3);
  PyArrayObject* st = plain(os, NPY_INT32, 0);
  if (!o || !d || !st || g_cast_host == NULL) Py_RETURN_NONE;
  const npy_intp n = PyArray_DIM(st, 0);
  if (PyArray_DIM(o, 0) != n || PyArray_DIM(d, 0) != n) {
    PyErr_Format(PyExc_ValueError, "length mismatch: %zd origins, %zd dirs, %zd starts", (Py_ssize_t)PyArray_DIM(o, 0),
                 (Py_ssize_t)PyArray_DIM(d, 0), (Py_ssize_t)n);
    return NULL;
  }
  const int32_t* s = (const int32_t*)PyArray_DATA(st);
  for (npy_intp i = 0; i < n; ++i) {
    if (s[i] < 0 || (long long)s[i] >= n_tets) {
      PyErr_Format(PyExc_IndexError, "start[%zd] = %d is not a tet index (n_tets=%lld)", (Py_ssize_t)i, (int)s[i],
                   n_tets);
      return NULL;
    }
  }
  npy_intp dims[1] = {n};
  PyObject* status = PyArray_EMPTY(1, dims, NPY_UINT8, 0);
  PyObject* cf = PyArray_EMPTY(1, dims, NPY_INT32, 0);
  PyObject* tet = PyArray_EMPTY(1, dims, NPY_INT32, 0);
  PyObject* visited = PyArray_EMPTY(1, dims, NPY_INT32, 0);
  if (!status || !cf || !tet || !visited) {
    Py_XDECREF(status);
    Py_XDECREF(cf);
    Py_XDECREF(tet);
    Py_XDECREF(visited);
    return NULL;
  }
  int rc = 0;
  if (n > 0) {
    const float* po = (const float*)PyArray_DATA(o);
    const float* pd = (const float*)PyArray_DATA(d);
    uint8_t* pst = (uint8_t*)PyArray_DATA((PyArrayObject*)status);
    int32_t* pcf = (int32_t*)PyArray_DATA((PyArrayObject*)cf);
    int32_t* ptet = (int32_t*)PyArray_DATA((PyArrayObject*)tet);
    int32_t* pvis = (int32_t*)PyArray_DATA((PyArrayObject*)visited);
    Py_BEGIN_ALLOW_THREADS
    rc = g_cast_host((void*)(uintptr_t)handle, (int64_t)n, po, pd, s, pst, pcf, ptet, pvis, NULL, NULL, NULL);
    Py_END_ALLOW_THREADS
  }
  if (rc != 0) {
    const char* msg = g_last_error ? g_last_error() : NULL;
    PyErr_Format(g_error ? g_error : PyExc_RuntimeError, "tb_cast_rays_host failed (%d): %s", rc,
                 msg ? msg : "unknown error");
    Py_DECREF(status);
    Py_DECREF(cf);
    Py_DECREF(tet);
    Py_DECREF(visited);
    return NULL;
  }
  return Py_BuildValue("(NNNN)", status, cf, tet, visited);
}

static PyMethodDef methods[] = {
    {"bind", bind, METH_VARARGS, "bind(cast_host_addr, last_error_addr, error_type)"},
    {"cast4", cast4, METH_VARARGS, "cast4(handle, n_tets, o, d, start) -> (status, cf, tet, visited) or None"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_fastcall", NULL, -1, methods};

PyMODINIT_FUNC PyInit__fastcall(void) {
  import_array();
  return PyModule_Create(&module);
}
