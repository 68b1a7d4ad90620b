/* _cprrtc_fast: the single-query latency path of planner.plan() in one
 * CPython call (METH_FASTCALL) instead of a ctypes call plus a Python decode.
 *
 * plan_one() calls cprrtc_plan (through the function pointer the ctypes
 * binding resolved, so both share one libcprrtc.so instance and its
 * contexts) with the GIL released, and returns the result already shaped for
 * PlanStats / PlanResult: the path as a tuple of fresh float64 row arrays
 * (the C call wrote the exact FP64 endpoints into the first and last rows)
 * and the edge sources as a tuple of the interned names.  Everything else of
 * plan() -- sessions, the context lock, error mapping, PlanResult -- stays in
 * planner.py; with the module missing, planner.py takes the ctypes path.
 * r2 (GPU box): the Python side of plan() ~12 -> ~5 us per call. */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#define NPY_NO_DEPRECATED_API NPY_1_7_API_VERSION
#include <numpy/arrayobject.h>

#include <string.h>
#include <time.h>

#include "cprrtc.h"

typedef int (*plan_fn)(void*, const cprrtc_params*, int, const double*, const double*, const int64_t*,
                       cprrtc_result*, double*, int32_t*);

static plan_fn g_plan = NULL;
static PyObject* g_src[3] = {NULL, NULL, NULL};   /* "start", "junction", "goal" */

/* setup(plan_fn_address, (name0, name1, name2)) */
static PyObject* fast_setup(PyObject* self, PyObject* args) {
    PyObject* addr;
    PyObject* names;
    (void)self;
    if (!PyArg_ParseTuple(args, "OO!", &addr, &PyTuple_Type, &names)) return NULL;
    if (PyTuple_GET_SIZE(names) != 3) {
        PyErr_SetString(PyExc_ValueError, "three edge-source names expected");
        return NULL;
    }
    void* f = PyLong_AsVoidPtr(addr);
    if (!f) {
        if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "NULL cprrtc_plan");
        return NULL;
    }
    g_plan = (plan_fn)f;
    for (int k = 0; k < 3; k++) {
        PyObject* s = PyTuple_GET_ITEM(names, k);
        Py_INCREF(s);
        Py_XDECREF(g_src[k]);
        g_src[k] = s;
    }
    Py_RETURN_NONE;
}

static const double* vec_data(PyObject* o, npy_intp n) {
    if (!PyArray_Check(o)) return NULL;
    PyArrayObject* a = (PyArrayObject*)o;
    if (PyArray_TYPE(a) != NPY_FLOAT64 || PyArray_NDIM(a) != 1 || PyArray_DIM(a, 0) != n ||
        !PyArray_IS_C_CONTIGUOUS(a))
        return NULL;
    return (const double*)PyArray_DATA(a);
}

/* plan_one(ctx, params, start, goal, seed, result, paths, sources, n)
 *   ctx / params / result / paths / sources: addresses (the session's
 *   buffers: one cprrtc_result, (path_capacity, n) doubles, path_capacity
 *   int32); start / goal: float64 C-contiguous (n,) arrays.
 * Returns None when an argument does not fit this fast path (the caller
 * takes the ctypes path), else
 *   (rc, wall_ms)                                            when rc != 0
 *   (0, status, setup_code, stats15, path, sources)          otherwise,
 * stats15 in PlanStats field order (wall_ms included) and path / sources
 * None unless solved. */
static PyObject* fast_plan_one(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
    (void)self;
    if (nargs != 9) {
        PyErr_SetString(PyExc_TypeError, "plan_one takes 9 arguments");
        return NULL;
    }
    if (!g_plan) {
        PyErr_SetString(PyExc_RuntimeError, "_cprrtc_fast.setup() not called");
        return NULL;
    }
    void* ctx = PyLong_AsVoidPtr(args[0]);
    const cprrtc_params* prm = (const cprrtc_params*)PyLong_AsVoidPtr(args[1]);
    const long n = PyLong_AsLong(args[8]);
    const long long seed_in = PyLong_AsLongLong(args[4]);
    cprrtc_result* res = (cprrtc_result*)PyLong_AsVoidPtr(args[5]);
    double* paths = (double*)PyLong_AsVoidPtr(args[6]);
    int32_t* srcs = (int32_t*)PyLong_AsVoidPtr(args[7]);
    if (PyErr_Occurred()) return NULL;
    const double* s = vec_data(args[2], n);
    const double* g = vec_data(args[3], n);
    if (!s || !g || !ctx || !prm || !res || !paths || !srcs || n < 1) Py_RETURN_NONE;
    const int64_t seed = (int64_t)seed_in;
    struct timespec t0, t1;
    int rc;
    Py_BEGIN_ALLOW_THREADS
    clock_gettime(CLOCK_MONOTONIC, &t0);
    rc = g_plan(ctx, prm, 1, s, g, &seed, res, paths, srcs);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    Py_END_ALLOW_THREADS
    const double wall = (double)(t1.tv_sec - t0.tv_sec) * 1e3 + (double)(t1.tv_nsec - t0.tv_nsec) * 1e-6;
    if (rc) return Py_BuildValue("(id)", rc, wall);

    const cprrtc_result* r = res;
    const uint64_t* st = r->stats;
    PyObject* stats = PyTuple_New(15);
    if (!stats) return NULL;
    for (int k = 0; k < 7; k++) PyTuple_SET_ITEM(stats, k, PyLong_FromUnsignedLongLong(st[k]));
    PyTuple_SET_ITEM(stats, 7, PyFloat_FromDouble(wall));
    PyTuple_SET_ITEM(stats, 8, PyLong_FromLong(r->nodes_start));
    PyTuple_SET_ITEM(stats, 9, PyLong_FromLong(r->nodes_goal));
    PyTuple_SET_ITEM(stats, 10, PyFloat_FromDouble(r->device_ms));
    for (int k = 8; k < 12; k++) PyTuple_SET_ITEM(stats, 3 + k, PyLong_FromUnsignedLongLong(st[k]));
    for (int k = 0; k < 15; k++)
        if (!PyTuple_GET_ITEM(stats, k)) {   /* an allocation failed: no tuple with holes */
            Py_DECREF(stats);
            return NULL;
        }

    PyObject* path = Py_None;
    PyObject* sources = Py_None;
    Py_INCREF(Py_None);
    Py_INCREF(Py_None);
    if (r->status == 0 && r->path_len >= 1) {
        const int L = r->path_len;
        Py_DECREF(path);
        Py_DECREF(sources);
        path = PyTuple_New(L);
        sources = PyTuple_New(L > 0 ? L - 1 : 0);
        if (!path || !sources) {
            Py_XDECREF(path);
            Py_XDECREF(sources);
            Py_DECREF(stats);
            return NULL;
        }
        npy_intp dim = (npy_intp)n;
        for (int i = 0; i < L; i++) {
            PyObject* row = PyArray_SimpleNew(1, &dim, NPY_FLOAT64);
            if (!row) {
                Py_DECREF(path);
                Py_DECREF(sources);
                Py_DECREF(stats);
                return NULL;
            }
            memcpy(PyArray_DATA((PyArrayObject*)row), paths + (size_t)i * n, (size_t)n * sizeof(double));
            PyTuple_SET_ITEM(path, i, row);
        }
        for (int i = 0; i < L - 1; i++) {
            int k = srcs[i];
            if (k < 0 || k > 2) k = 2;
            Py_INCREF(g_src[k]);
            PyTuple_SET_ITEM(sources, i, g_src[k]);
        }
    }
    PyObject* out = PyTuple_New(6);
    if (!out) {
        Py_DECREF(path);
        Py_DECREF(sources);
        Py_DECREF(stats);
        return NULL;
    }
    PyTuple_SET_ITEM(out, 0, PyLong_FromLong(0));
    PyTuple_SET_ITEM(out, 1, PyLong_FromLong(r->status));
    PyTuple_SET_ITEM(out, 2, PyLong_FromLong(r->setup_code));
    PyTuple_SET_ITEM(out, 3, stats);
    PyTuple_SET_ITEM(out, 4, path);
    PyTuple_SET_ITEM(out, 5, sources);
    if (!PyTuple_GET_ITEM(out, 0) || !PyTuple_GET_ITEM(out, 1) || !PyTuple_GET_ITEM(out, 2)) {
        Py_DECREF(out);
        return NULL;
    }
    return out;
}

static PyMethodDef methods[] = {
    {"setup", fast_setup, METH_VARARGS, "setup(cprrtc_plan address, edge-source names)"},
    {"plan_one", (PyCFunction)(void (*)(void))fast_plan_one, METH_FASTCALL,
     "plan_one(ctx, params, start, goal, seed, result, paths, sources, n)"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_cprrtc_fast",
                                    "single-query plan() fast path over libcprrtc.so", -1, methods,
                                    NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__cprrtc_fast(void) {
    import_array();
    return PyModule_Create(&module);
}
