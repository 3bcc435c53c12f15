"""CPU oracle for the QAP swap-delta hot path -- TEST INFRASTRUCTURE ONLY.

ctypes front-end to ``oracle/liboracle.so`` (built from ``qap_oracle.c``, a plain-C
restatement of the reference's ``_kernels.pyx`` / ``rng.py`` / ``multistart.py``
semantics; each C function cites the reference lines it follows) plus a loader
for ``oracle/_ref`` -- the reference's *own* Cython kernel compiled from
``/root/reference`` by ``oracle/Makefile``.

Nothing under ``paper_2307_11248_b200/`` imports this package.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
legs may use it, and only as the checker or the timed CPU baseline.

Parity status: pinned (see the header of ``qap_oracle.c`` and ``tests/test_oracle.py``).
"""

from __future__ import annotations

import ctypes
import glob
import importlib.util
import os
import subprocess
from ctypes import POINTER, c_int, c_int64, c_uint64

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64p = POINTER(c_int64)


def build(force: bool = False) -> None:
    """Compile liboracle.so and (when /root/reference is present) oracle/_ref."""
    src = os.path.join(_HERE, "qap_oracle.c")
    stale = not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)
    have_ref = bool(glob.glob(os.path.join(_HERE, "_ref", "_kernels*.so")))
    if force or stale or not have_ref:
        subprocess.run(["make", "-C", _HERE], check=True, capture_output=True)


def _ptr(a: np.ndarray | None):
    if a is None:
        return ctypes.cast(None, _i64p)
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_i64p)


def _as64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_mix64.restype = c_uint64
        L.orc_mix64.argtypes = [c_uint64]
        L.orc_next64.restype = c_uint64
        L.orc_next64.argtypes = [POINTER(c_uint64)]
        L.orc_randbelow.restype = c_uint64
        L.orc_randbelow.argtypes = [POINTER(c_uint64), c_uint64]
        L.orc_derive_seed.restype = c_uint64
        L.orc_derive_seed.argtypes = [c_uint64, c_uint64]
        L.orc_random_permutation.restype = None
        L.orc_random_permutation.argtypes = [c_int, POINTER(c_uint64), _i64p]
        L.orc_tenure_bounds.restype = None
        L.orc_tenure_bounds.argtypes = [c_int, _i64p, _i64p]
        L.orc_draw_tenures.restype = None
        L.orc_draw_tenures.argtypes = [POINTER(c_uint64), c_int64, c_int64, c_int, _i64p]
        L.orc_random_instance.restype = None
        L.orc_random_instance.argtypes = [c_int, POINTER(c_uint64), c_int64, c_int64, _i64p, _i64p]
        L.orc_full_cost.restype = c_int64
        L.orc_full_cost.argtypes = [c_int, _i64p, _i64p, _i64p]
        L.orc_delta.restype = c_int64
        L.orc_delta.argtypes = [c_int, _i64p, _i64p, _i64p, c_int, c_int]
        L.orc_all_deltas.restype = None
        L.orc_all_deltas.argtypes = [c_int, _i64p, _i64p, _i64p, _i64p]
        L.orc_two_opt_run.restype = None
        L.orc_two_opt_run.argtypes = [c_int, _i64p, _i64p, _i64p, c_int] + [_i64p] * 7
        L.orc_tabu_run.restype = c_int
        L.orc_tabu_run.argtypes = (
            [c_int, _i64p, _i64p, _i64p, c_int, _i64p] + [_i64p] * 5 + [POINTER(c_int)] + [_i64p] * 6
        )
        L.orc_multistart.restype = c_int
        L.orc_multistart.argtypes = [
            c_int, _i64p, _i64p, c_int, c_uint64, c_uint64, c_int, c_int, c_int64, c_int64, c_int,
            _i64p, _i64p, _i64p, _i64p,
        ]
        L.orc_max_threads.restype = c_int
        L.orc_max_threads.argtypes = []
        _lib = L
    return _lib


_M64 = (1 << 64) - 1


class Rng:
    """SplitMix64 stream held in a C uint64 (restates rng.py:23-59)."""

    def __init__(self, seed: int):
        self._s = c_uint64(seed & _M64)

    @property
    def state(self) -> int:
        return int(self._s.value)

    def next64(self) -> int:
        return int(lib().orc_next64(ctypes.byref(self._s)))

    def randbelow(self, bound: int) -> int:
        return int(lib().orc_randbelow(ctypes.byref(self._s), bound))

    def permutation(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.int64)
        lib().orc_random_permutation(n, ctypes.byref(self._s), _ptr(out))
        return out

    def tenures(self, low: int, high: int, iterations: int) -> np.ndarray:
        out = np.empty(iterations, dtype=np.int64)
        lib().orc_draw_tenures(ctypes.byref(self._s), low, high, iterations, _ptr(out))
        return out

    def instance(self, n: int, low: int = 0, high: int = 99):
        f = np.empty((n, n), dtype=np.int64)
        d = np.empty((n, n), dtype=np.int64)
        lib().orc_random_instance(n, ctypes.byref(self._s), low, high, _ptr(f), _ptr(d))
        return f, d


def mix64(z: int) -> int:
    return int(lib().orc_mix64(z & _M64))


def derive_seed(master_seed: int, start_index: int) -> int:
    return int(lib().orc_derive_seed(master_seed & _M64, start_index))


def tenure_bounds(n: int) -> tuple[int, int]:
    lo, hi = c_int64(), c_int64()
    lib().orc_tenure_bounds(n, ctypes.byref(lo), ctypes.byref(hi))
    return int(lo.value), int(hi.value)


def full_cost(flow, dist, perm) -> int:
    f, d, p = _as64(flow), _as64(dist), _as64(perm)
    return int(lib().orc_full_cost(len(p), _ptr(f), _ptr(d), _ptr(p)))


def delta(flow, dist, perm, i: int, j: int) -> int:
    f, d, p = _as64(flow), _as64(dist), _as64(perm)
    return int(lib().orc_delta(len(p), _ptr(f), _ptr(d), _ptr(p), i, j))


def all_deltas(flow, dist, perm) -> np.ndarray:
    f, d, p = _as64(flow), _as64(dist), _as64(perm)
    n = len(p)
    out = np.empty(n * (n - 1) // 2, dtype=np.int64)
    lib().orc_all_deltas(n, _ptr(f), _ptr(d), _ptr(p), _ptr(out))
    return out


def two_opt_run(flow, dist, perm, iterations: int):
    """Same 7-tuple as the reference kernels.two_opt_run (_kernels.pyx:118)."""
    f, d, p = _as64(flow), _as64(dist), _as64(perm)
    n = len(p)
    best, cur = np.empty(n, np.int64), np.empty(n, np.int64)
    mi, mj, md = (np.empty(iterations, np.int64) for _ in range(3))
    bc, cc = c_int64(), c_int64()
    lib().orc_two_opt_run(
        n, _ptr(f), _ptr(d), _ptr(p), iterations, _ptr(best),
        ctypes.cast(ctypes.byref(bc), _i64p), _ptr(cur), ctypes.cast(ctypes.byref(cc), _i64p),
        _ptr(mi), _ptr(mj), _ptr(md),
    )
    return best, int(bc.value), cur, int(cc.value), mi, mj, md


def tabu_run(flow, dist, perm, iterations: int, tenures):
    """Same 8-tuple as the reference kernels.tabu_run (_kernels.pyx:189-197)."""
    f, d, p, t = _as64(flow), _as64(dist), _as64(perm), _as64(tenures)
    n = len(p)
    best, cur = np.empty(n, np.int64), np.empty(n, np.int64)
    cells = np.empty((n, n), np.int64)
    tr = [np.empty(iterations, np.int64) for _ in range(6)]
    bc, cc, stopped = c_int64(), c_int64(), c_int()
    steps = lib().orc_tabu_run(
        n, _ptr(f), _ptr(d), _ptr(p), iterations, _ptr(t), _ptr(best),
        ctypes.cast(ctypes.byref(bc), _i64p), _ptr(cur), ctypes.cast(ctypes.byref(cc), _i64p),
        _ptr(cells), ctypes.byref(stopped), *[_ptr(a) for a in tr],
    )
    trail = tuple(a[:steps].copy() for a in tr)
    return best, int(bc.value), cur, int(cc.value), cells, bool(stopped.value), int(steps), trail


def multistart(flow, dist, algorithm: str, master_seed: int, n_starts: int, iterations: int,
               tenure: tuple[int, int] | None = None, first_index: int = 0, threads: int = 1):
    """Restates run_multistart (multistart.py:121-172) for starts
    [first_index, first_index + n_starts).  Returns
    (per_start_costs, best_cost, best_index, best_perm)."""
    f, d = _as64(flow), _as64(dist)
    n = f.shape[0]
    lo, hi = tenure if tenure is not None else tenure_bounds(n)
    costs = np.empty(n_starts, np.int64)
    perm = np.empty(n, np.int64)
    bc, bi = c_int64(), c_int64()
    rc = lib().orc_multistart(
        n, _ptr(f), _ptr(d), 1 if algorithm == "tabu" else 0, master_seed & _M64, first_index,
        n_starts, iterations, lo, hi, threads, _ptr(costs),
        ctypes.cast(ctypes.byref(bc), _i64p), ctypes.cast(ctypes.byref(bi), _i64p), _ptr(perm),
    )
    if rc != 0:
        raise MemoryError("oracle multistart scratch allocation failed")
    return costs, int(bc.value), int(bi.value), perm


def max_threads() -> int:
    return int(lib().orc_max_threads())


def load_ref_kernels():
    """The reference's own compiled kernel module (oracle/_ref), or None if absent."""
    hits = sorted(glob.glob(os.path.join(_HERE, "_ref", "_kernels*.so")))
    if not hits:
        return None
    spec = importlib.util.spec_from_file_location("_kernels", hits[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod
