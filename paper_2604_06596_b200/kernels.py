"""``dynlp.kernels``-compatible backend running on the B200.

Same module surface as /root/reference/pkg/src/dynlp/kernels/__init__.py:
``jacobi_step``, ``jacobi_run``, ``gauss_seidel_step``, ``BACKEND`` and
``available_backends()``, with the argument conventions of
kernels/_csr.pyx:61-70, 94-102, 114-125 (int64 CSR, int8 gt, fp64 f,
uint8 eligible).  Select it from the reference with the adapter shown in
INTEGRATION.md (DYNLP_KERNELS=b200).  Arrays are copied to the device per
call; results are written back in place exactly where the reference
mutates (f in jacobi_run / gauss_seidel_step, eligible in jacobi_run).
``jacobi_run`` returns its leftover frontier sorted ascending.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native
from .errors import CudaError

BACKEND = "b200"


def _arr(a, dt):
    a = np.asarray(a)
    if a.dtype != dt or not a.flags.c_contiguous:
        a = np.ascontiguousarray(a, dtype=dt)
    return a


def _inplace(a, dt, name):
    if not isinstance(a, np.ndarray) or a.dtype != dt or not a.flags.c_contiguous:
        raise TypeError(f"{name} must be a C-contiguous {np.dtype(dt).name} array (mutated in place)")
    return a


def _check(rc):
    if rc != 0:
        raise CudaError(_native.load().dlp_plugin_last_error().decode())


def jacobi_step(indptr, indices, weights, gt, f, frontier, out_vals, out_deltas, threads=1):
    lib = _native.load()
    ip = _arr(indptr, np.int64)
    ix, w, g = _arr(indices, np.int64), _arr(weights, np.float64), _arr(gt, np.int8)
    ff, fr = _arr(f, np.float64), _arr(frontier, np.int64)
    ov = _inplace(out_vals, np.float64, "out_vals")
    od = _inplace(out_deltas, np.float64, "out_deltas")
    n = len(ip) - 1
    _check(lib.dlp_jacobi_step(_native.ptr(ip), _native.ptr(ix), _native.ptr(w), _native.ptr(g),
                               _native.ptr(ff), n, _native.ptr(fr), len(fr), _native.ptr(ov),
                               _native.ptr(od)))


def gauss_seidel_step(indptr, indices, weights, gt, f, frontier, out_deltas):
    lib = _native.load()
    ip = _arr(indptr, np.int64)
    ix, w, g = _arr(indices, np.int64), _arr(weights, np.float64), _arr(gt, np.int8)
    ff = _inplace(f, np.float64, "f")
    fr = _arr(frontier, np.int64)
    od = _inplace(out_deltas, np.float64, "out_deltas")
    _check(lib.dlp_gauss_seidel_step(_native.ptr(ip), _native.ptr(ix), _native.ptr(w), _native.ptr(g),
                                     _native.ptr(ff), len(ip) - 1, _native.ptr(fr), len(fr),
                                     _native.ptr(od)))


def jacobi_run(indptr, indices, weights, gt, f, frontier_init, eligible, delta, max_iters, threads=1):
    lib = _native.load()
    ip = _arr(indptr, np.int64)
    ix, w, g = _arr(indices, np.int64), _arr(weights, np.float64), _arr(gt, np.int8)
    ff = _inplace(f, np.float64, "f")
    el = eligible.view(np.uint8) if isinstance(eligible, np.ndarray) and eligible.dtype == bool else eligible
    el = _inplace(el, np.uint8, "eligible")
    fr = _arr(frontier_init, np.int64)
    n = len(ip) - 1
    left = np.empty(max(n, len(fr)) + 1, dtype=np.int64)
    it, upd, warn, nl = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    mc = C.c_double()
    _check(lib.dlp_jacobi_run(_native.ptr(ip), _native.ptr(ix), _native.ptr(w), _native.ptr(g),
                              _native.ptr(ff), n, _native.ptr(fr), len(fr), _native.ptr(el),
                              float(delta), int(max_iters), C.byref(it), C.byref(upd), C.byref(mc),
                              C.byref(warn), _native.ptr(left), C.byref(nl)))
    return it.value, upd.value, mc.value, warn.value, left[: nl.value].copy()


def available_backends():
    import sys

    return {"b200": sys.modules[__name__]}
