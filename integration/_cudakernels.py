"""qapsolve/_cudakernels.py -- the reference's kernel-backend interface served by libqapb.so.

This is the file a maintainer of `qapsolve` adds next to `_kernels.pyx` / `_purekernels.py`
(/root/reference/pkg/src/qapsolve/backend.py:14-25 picks a module with these five names).  It binds only the
C ABI of include/qapb.h with ctypes: no torch, nothing from this repository's Python package.  The library
is found through $QAPB_LIB (default: "libqapb.so" on the loader path).  There is no CPU fallback.

`multistart(...)` is the batched addition `run_multistart` uses ("Batched multi-start").
"""
import ctypes
import os

import numpy as np

BACKEND_NAME = "cuda-sm100a"
try:
    _L = ctypes.CDLL(os.environ.get("QAPB_LIB", "libqapb.so"))
except OSError as exc:  # backend.py treats a missing compiled module as ImportError
    raise ImportError(f"libqapb.so not found (set QAPB_LIB): {exc}") from exc
_L.qapb_last_error.restype = ctypes.c_char_p
_P = ctypes.c_void_p
_handles = {}  # keyed by matrix contents: the interface passes (flow, dist) on every call


def _check(rc):
    if rc == 1:  # QAPB_ERR_INVALID -> DomainError(ValueError)
        from .errors import DomainError

        raise DomainError(_L.qapb_last_error().decode())
    if rc:       # CUDA / memory / unsupported
        from .errors import QapError

        raise QapError(_L.qapb_last_error().decode())


def _handle(flow, dist):
    f = np.ascontiguousarray(flow, np.int64)
    d = np.ascontiguousarray(dist, np.int64)
    key = (f.shape, f.tobytes(), d.tobytes())
    if key not in _handles:
        if len(_handles) >= 64:
            _, (old, _) = _handles.popitem()
            _L.qapb_destroy(old)
        h = _P()
        _check(_L.qapb_create(f.shape[0], _P(f.ctypes.data), _P(d.ctypes.data), 0, ctypes.byref(h)))
        _handles[key] = (h, f.shape[0])
    return _handles[key]


def _a(x):
    return _P(x.ctypes.data)


def full_cost(flow, dist, perm):                    # _kernels.pyx:48-55
    h, n = _handle(flow, dist)
    p = np.ascontiguousarray(perm, np.int64)
    out = np.empty(1, np.int64)
    _check(_L.qapb_full_cost_host(h, _a(p), 1, _a(out)))
    return int(out[0])


def all_deltas(flow, dist, perm):                   # _kernels.pyx:58-70
    h, n = _handle(flow, dist)
    p = np.ascontiguousarray(perm, np.int64)
    out = np.empty(n * (n - 1) // 2, np.int64)
    _check(_L.qapb_all_deltas_host(h, _a(p), 1, _a(out)))
    return out


def two_opt_run(flow, dist, perm, iterations):      # _kernels.pyx:73-118 -> the same 7-tuple
    h, n = _handle(flow, dist)
    p = np.ascontiguousarray(perm, np.int64)
    iterations = int(iterations)
    if iterations == 0:  # the loop of _kernels.pyx:94 does not run
        c = full_cost(flow, dist, p)
        e = np.zeros(0, np.int64)
        return p.copy(), c, p.copy(), c, e, e.copy(), e.copy()
    best, cur = np.empty(n, np.int64), np.empty(n, np.int64)
    bc, cc = np.empty(1, np.int64), np.empty(1, np.int64)
    mi, mj, md = (np.empty(iterations, np.int64) for _ in range(3))
    _check(_L.qapb_two_opt_host(h, _a(p), 1, iterations, _a(best), _a(bc), _a(cur), _a(cc), _a(mi), _a(mj), _a(md)))
    return best, int(bc[0]), cur, int(cc[0]), mi, mj, md


def tabu_run(flow, dist, perm, iterations, tenures):  # _kernels.pyx:121-197 -> the same 8-tuple
    h, n = _handle(flow, dist)
    p = np.ascontiguousarray(perm, np.int64)
    t = np.ascontiguousarray(tenures, np.int64)
    iterations = int(iterations)
    if iterations == 0:
        c = full_cost(flow, dist, p)
        return (p.copy(), c, p.copy(), c, np.zeros((n, n), np.int64), False, 0,
                tuple(np.zeros(0, np.int64) for _ in range(6)))
    best, cur = np.empty(n, np.int64), np.empty(n, np.int64)
    bc, cc, stop, steps = (np.empty(1, np.int64) for _ in range(4))
    cells = np.empty((n, n), np.int64)
    ti, tj, td, tt = (np.zeros(iterations, np.int64) for _ in range(4))
    _check(_L.qapb_tabu_host(h, _a(p), 1, iterations, _a(t), _a(best), _a(bc), _a(cur), _a(cc), _a(cells),
                             _a(stop), _a(steps), _a(ti), _a(tj), _a(td), _a(tt)))
    k = int(steps[0])
    trail = (ti[:k].copy(), tj[:k].copy(), td[:k].copy(), tt[:k].copy(), tt[:k].copy(), t[:k].copy())
    return best, int(bc[0]), cur, int(cc[0]), cells, bool(stop[0]), k, trail


def multistart(flow, dist, algorithm, master_seed, n_starts, iterations, ten_low, ten_high):
    """The whole map + local reduce of run_multistart (multistart.py:86-118, 156) in one launch:
    (per_start_costs[n_starts], best cost, best start index, best permutation)."""
    h, n = _handle(flow, dist)
    costs, key, perm = np.empty(n_starts, np.int64), np.empty(2, np.int64), np.empty(n, np.int64)
    _check(_L.qapb_multistart_host(h, 1 if algorithm == "tabu" else 0, ctypes.c_uint64(master_seed & (2 ** 64 - 1)),
                                   ctypes.c_uint64(0), int(n_starts), int(iterations), ctypes.c_int64(ten_low),
                                   ctypes.c_int64(ten_high), _a(costs), _a(key), _a(perm)))
    return costs, int(key[0]), int(key[1]), perm
