/* pyfast.c — a CPython fast-call shim for the per-token hot entry of the C ABI.
 *
 * ctypes marshals each argument through generic converters (~0.3 us per argument on the GPU box's
 * host: a 15-argument flashnorm_linear_ws call costs ~5 us of Python before the launch), which made
 * eager decode host-bound (profiles/r02q_host_overhead.txt).  This module takes the SAME C-ABI
 * function (its address is handed over by the ctypes-loaded libflashnorm.so, so there is one
 * library instance) and calls it from a METH_FASTCALL function with plain PyLong / PyFloat
 * conversions.  Argument marshalling only: every step of the path runs in libflashnorm.so.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

typedef int (*linear_ws_fn)(const void*, const void*, const float*, int64_t, int64_t, int64_t, float, float, int, int,
                            void*, int, void*, int64_t, void*);
static linear_ws_fn g_linear_ws = NULL;

static void* as_ptr(PyObject* o) { return o == Py_None ? NULL : PyLong_AsVoidPtr(o); }

/* bind(address_of_flashnorm_linear_ws) */
static PyObject* py_bind(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 1) {
    PyErr_SetString(PyExc_TypeError, "bind(address)");
    return NULL;
  }
  g_linear_ws = (linear_ws_fn)PyLong_AsVoidPtr(args[0]);
  if (PyErr_Occurred()) return NULL;
  Py_RETURN_NONE;
}

/* linear_ws(a, Wt_star, c_star, M, K, N, eps, alpha, mode, dtype, z, path, workspace, ws_bytes, stream)
 * pointers: int or None; returns the fn_status */
static PyObject* py_linear_ws(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (g_linear_ws == NULL) {
    PyErr_SetString(PyExc_RuntimeError, "pyfast: bind() not called");
    return NULL;
  }
  if (nargs != 15) {
    PyErr_SetString(PyExc_TypeError, "linear_ws takes 15 arguments");
    return NULL;
  }
  const void* a = as_ptr(args[0]);
  const void* w = as_ptr(args[1]);
  const float* c = (const float*)as_ptr(args[2]);
  const int64_t M = PyLong_AsLongLong(args[3]), K = PyLong_AsLongLong(args[4]), N = PyLong_AsLongLong(args[5]);
  const float eps = (float)PyFloat_AsDouble(args[6]), alpha = (float)PyFloat_AsDouble(args[7]);
  const int mode = (int)PyLong_AsLong(args[8]), dtype = (int)PyLong_AsLong(args[9]);
  void* z = as_ptr(args[10]);
  const int path = (int)PyLong_AsLong(args[11]);
  void* ws = as_ptr(args[12]);
  const int64_t wsb = PyLong_AsLongLong(args[13]);
  void* stream = as_ptr(args[14]);
  if (PyErr_Occurred()) return NULL;
  int st;
  Py_BEGIN_ALLOW_THREADS
  st = g_linear_ws(a, w, c, M, K, N, eps, alpha, mode, dtype, z, path, ws, wsb, stream);
  Py_END_ALLOW_THREADS
  return PyLong_FromLong(st);
}

static PyMethodDef methods[] = {
    {"bind", (PyCFunction)(void (*)(void))py_bind, METH_FASTCALL, "bind(address of flashnorm_linear_ws)"},
    {"linear_ws", (PyCFunction)(void (*)(void))py_linear_ws, METH_FASTCALL, "flashnorm_linear_ws fast call"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_pyfast", NULL, -1, methods};

PyMODINIT_FUNC PyInit__pyfast(void) { return PyModule_Create(&module); }
