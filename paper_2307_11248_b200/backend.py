"""The kernel backend: same plugin interface as the reference's `backend.kernels`
(/root/reference/pkg/src/qapsolve/backend.py:16-29), served by the CUDA library.

`kernels` exposes `BACKEND_NAME`, `full_cost`, `all_deltas`, `two_opt_run` and
`tabu_run` with the argument order, return tuples and dtypes of
`_kernels.pyx:48,58,73,121`, so `core`, `two_opt`, `tabu` and the reference's own
`tests/test_backends.py` pattern work against it unchanged.  Batched entries
(`*_batch`, `multistart`) are additions used by `run_multistart`.

There is exactly one backend.  If `libqapb.so` is missing or no CUDA device is
visible the calls raise; nothing here computes on the CPU.
"""

from __future__ import annotations

import ctypes
import hashlib
import threading
import weakref
from collections import OrderedDict

import numpy as np

from . import _lib
from .errors import DomainError

_i64 = np.int64


def _mat(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=_i64)


def _addr(a: np.ndarray | None) -> int | None:
    return None if a is None else a.ctypes.data


class DeviceInstance:
    """Owns a `qapb_handle`: the instance resident on one GPU plus its kernel plan."""

    def __init__(self, flow, dist, device: int = 0):
        f, d = _mat(flow), _mat(dist)
        if f.ndim != 2 or f.shape[0] != f.shape[1] or f.shape != d.shape:
            raise DomainError(f"flow {f.shape} and distance {d.shape} must be equal square matrices")
        self.n = int(f.shape[0])
        self.device = device
        self._h = ctypes.c_void_p()
        _lib.check(_lib.lib().qapb_create(self.n, _addr(f), _addr(d), device, ctypes.byref(self._h)))
        info = _lib.Info()
        _lib.check(_lib.lib().qapb_get_info(self._h, ctypes.byref(info)))
        self.info = {name: int(getattr(info, name)) for name, _ in _lib.Info._fields_}

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def close(self) -> None:
        if self._h:
            _lib.lib().qapb_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- host-buffer calls (NumPy in, NumPy out) --------------------------------
    def _perms(self, perms) -> np.ndarray:
        p = np.ascontiguousarray(perms, dtype=_i64)
        if p.ndim == 1:
            p = p[None, :]
        if p.ndim != 2 or p.shape[1] != self.n:
            raise DomainError(f"permutation size {p.shape[-1]} != instance size {self.n}")
        return p

    def full_cost(self, perms) -> np.ndarray:
        p = self._perms(perms)
        out = np.empty(p.shape[0], _i64)
        _lib.check(_lib.lib().qapb_full_cost_host(self._h, _addr(p), p.shape[0], _addr(out)))
        return out

    def all_deltas(self, perms) -> np.ndarray:
        p = self._perms(perms)
        out = np.empty((p.shape[0], self.n * (self.n - 1) // 2), _i64)
        _lib.check(_lib.lib().qapb_all_deltas_host(self._h, _addr(p), p.shape[0], _addr(out)))
        return out

    def two_opt(self, perms, iterations: int, moves: bool = True):
        if iterations < 1:
            raise DomainError(f"iterations must be >= 1, got {iterations}")
        p = self._perms(perms)
        b = p.shape[0]
        best, cur = np.empty((b, self.n), _i64), np.empty((b, self.n), _i64)
        bc, cc = np.empty(b, _i64), np.empty(b, _i64)
        mv = [np.empty((b, iterations), _i64) if moves else None for _ in range(3)]
        _lib.check(_lib.lib().qapb_two_opt_host(
            self._h, _addr(p), b, iterations, _addr(best), _addr(bc), _addr(cur), _addr(cc),
            _addr(mv[0]), _addr(mv[1]), _addr(mv[2])))
        return best, bc, cur, cc, mv[0], mv[1], mv[2]

    def tabu(self, perms, iterations: int, tenures, cells: bool = True, trail: bool = True):
        if iterations < 1:
            raise DomainError(f"iterations must be >= 1, got {iterations}")
        p = self._perms(perms)
        b = p.shape[0]
        t = np.ascontiguousarray(tenures, dtype=_i64)
        if t.ndim == 1:
            t = t[None, :]
        if t.shape != (b, iterations):
            raise DomainError(f"tenures shape {t.shape} != {(b, iterations)}")
        best, cur = np.empty((b, self.n), _i64), np.empty((b, self.n), _i64)
        bc, cc = np.empty(b, _i64), np.empty(b, _i64)
        stop, steps = np.empty(b, _i64), np.empty(b, _i64)
        cz = np.empty((b, self.n, self.n), _i64) if cells else None
        tr = [np.zeros((b, iterations), _i64) if trail else None for _ in range(4)]
        _lib.check(_lib.lib().qapb_tabu_host(
            self._h, _addr(p), b, iterations, _addr(t), _addr(best), _addr(bc), _addr(cur), _addr(cc),
            _addr(cz), _addr(stop), _addr(steps), _addr(tr[0]), _addr(tr[1]), _addr(tr[2]), _addr(tr[3])))
        return best, bc, cur, cc, cz, stop, steps, tr, t

    def multistart(self, algorithm: str, master_seed: int, first_index: int, count: int,
                   iterations: int, ten_low: int = 1, ten_high: int = 1):
        """Host-buffer multistart: (per_start_costs[count], best_cost, best_index, best_perm[n])."""
        costs = np.empty(count, _i64)
        key = np.empty(2, _i64)
        perm = np.empty(self.n, _i64)
        algo = _lib.ALGO_TABU if algorithm == "tabu" else _lib.ALGO_2OPT
        _lib.check(_lib.lib().qapb_multistart_host(
            self._h, algo, master_seed & 0xFFFFFFFFFFFFFFFF, first_index, count, iterations,
            ten_low, ten_high, _addr(costs), _addr(key), _addr(perm)))
        return costs, int(key[0]), int(key[1]), perm

    def multistart_seeds(self, algorithm: str, seeds, iterations: int, ten_low: int = 1, ten_high: int = 1):
        """Host-buffer multistart over explicit per-start SplitMix64 states (`derive_seed` values):
        (per_start_costs[count], best_perms[count, n]).  One launch for any mix of master seeds."""
        sd = np.ascontiguousarray(seeds, dtype=np.uint64)
        if sd.ndim != 1 or sd.size < 1:
            raise DomainError("seeds must be a non-empty 1-d array")
        count = int(sd.size)
        costs = np.empty(count, _i64)
        perms = np.empty((count, self.n), _i64)
        algo = _lib.ALGO_TABU if algorithm == "tabu" else _lib.ALGO_2OPT
        _lib.check(_lib.lib().qapb_multistart_seeds_host(
            self._h, algo, _addr(sd), count, iterations, ten_low, ten_high, _addr(costs), _addr(perms)))
        return costs, perms

    def multistart_trace(self, algorithm: str, seeds, iterations: int, ten_low: int = 1, ten_high: int = 1):
        """`multistart_seeds` with every start's trajectory: (per_start_costs[count], best_perms[count, n],
        steps_done[count], move_i, move_j, move_delta -- each [count, iterations], zero past steps_done)."""
        sd = np.ascontiguousarray(seeds, dtype=np.uint64)
        if sd.ndim != 1 or sd.size < 1:
            raise DomainError("seeds must be a non-empty 1-d array")
        if iterations < 1:
            raise DomainError(f"iterations must be >= 1, got {iterations}")
        count = int(sd.size)
        costs, steps = np.empty(count, _i64), np.empty(count, _i64)
        perms = np.empty((count, self.n), _i64)
        mv = [np.empty((count, iterations), _i64) for _ in range(3)]
        algo = _lib.ALGO_TABU if algorithm == "tabu" else _lib.ALGO_2OPT
        _lib.check(_lib.lib().qapb_multistart_trace_host(
            self._h, algo, _addr(sd), count, iterations, ten_low, ten_high, _addr(costs), _addr(perms), _addr(steps),
            _addr(mv[0]), _addr(mv[1]), _addr(mv[2])))
        return costs, perms, steps, mv[0], mv[1], mv[2]

    def multistart_device(self, algorithm: str, master_seed: int, first_index: int, count: int,
                          iterations: int, ten_low: int, ten_high: int,
                          costs_ptr: int, key_ptr: int, perm_ptr: int, stream: int = 0) -> None:
        """Device-pointer multistart (torch `data_ptr()`s), asynchronous on `stream`."""
        algo = _lib.ALGO_TABU if algorithm == "tabu" else _lib.ALGO_2OPT
        _lib.check(_lib.lib().qapb_multistart(
            self._h, algo, master_seed & 0xFFFFFFFFFFFFFFFF, first_index, count, iterations,
            ten_low, ten_high, costs_ptr, key_ptr, perm_ptr, stream or None))

    def _refresh_info(self) -> None:
        info = _lib.Info()
        _lib.check(_lib.lib().qapb_get_info(self._h, ctypes.byref(info)))
        self.info = {name: int(getattr(info, name)) for name, _ in _lib.Info._fields_}

    def plan_candidates(self) -> list[tuple[int, int, int, int]]:
        """Launch configurations that fit this instance: (register units per thread, threads carrying
        off-diagonal units, shared-memory units per thread, diagonal blocks in shared memory); register
        units 0 is the one-warp-per-search kernel (n <= 32), listed first where it applies.  Empty for
        instances served by the generic kernel."""
        buf = np.zeros((16, 4), np.int32)
        count = ctypes.c_int(0)
        _lib.check(_lib.lib().qapb_plan_candidates(self._h, _addr(buf), 16, ctypes.byref(count)))
        return [tuple(int(x) for x in row) for row in buf[: min(count.value, 16)]]

    def set_plan(self, plan: tuple[int, int, int, int]) -> None:
        """Re-plan with one of `plan_candidates()`; results do not depend on the plan."""
        _lib.check(_lib.lib().qapb_set_plan(self._h, *[int(x) for x in plan]))
        self._refresh_info()

    def last_total_steps(self) -> int:
        """Sum of steps_done over the starts of the last `multistart*` call on this handle."""
        v = ctypes.c_int64(0)
        _lib.check(_lib.lib().qapb_last_total_steps(self._h, ctypes.byref(v)))
        return int(v.value)

    def last_kernel_ms(self) -> float:
        ms = ctypes.c_float(0)
        _lib.check(_lib.lib().qapb_last_kernel_ms(self._h, ctypes.byref(ms)))
        return float(ms.value)


# ---- handle cache: reference kernels take (flow, dist) on every call ------------
_CACHE: "OrderedDict[tuple, DeviceInstance]" = OrderedDict()
_CACHE_LOCK = threading.Lock()
_CACHE_MAX = 8


# read-only matrices (every `Instance` freezes its arrays, instance.py:47) are recognised by identity, so
# repeated calls on one instance do not re-hash 2 n^2 words: (id(flow), id(dist), device) -> weak refs + handle
_ID_CACHE: dict = {}


def _frozen(a) -> bool:
    # owndata: a read-only VIEW of a writeable base can still change underneath us -> hash those
    return (isinstance(a, np.ndarray) and a.dtype == _i64 and a.flags.c_contiguous and not a.flags.writeable
            and a.flags.owndata)


_SERIAL = [0]


def device_instance(flow, dist, device: int = 0) -> DeviceInstance:
    """Cached `DeviceInstance`: by identity for frozen arrays (no hashing), else keyed by matrix contents.
    Both kinds live in one LRU; eviction only drops the cache's reference."""
    by_id = _frozen(flow) and _frozen(dist)
    with _CACHE_LOCK:
        if by_id:
            hit = _ID_CACHE.get((id(flow), id(dist), device))
            if hit is not None and hit[0]() is flow and hit[1]() is dist and hit[2]._h:
                if hit[3] in _CACHE:
                    _CACHE.move_to_end(hit[3])
                return hit[2]
            _SERIAL[0] += 1
            key = ("id", _SERIAL[0])
            f, d = flow, dist
        else:
            f, d = _mat(flow), _mat(dist)
            key = (f.shape, hashlib.blake2b(f.tobytes() + d.tobytes(), digest_size=16).digest(), device)
        inst = _CACHE.get(key)
        if inst is not None:
            _CACHE.move_to_end(key)
            return inst
        inst = DeviceInstance(f, d, device)
        _CACHE[key] = inst
        while len(_CACHE) > _CACHE_MAX:
            # drop the cache's reference only: a caller (or another thread inside a C call) may still hold
            # the evicted instance; its handle is destroyed when the last reference goes (__del__)
            _, old = _CACHE.popitem(last=False)
            for k in [k for k, v in _ID_CACHE.items() if v[2] is old]:
                del _ID_CACHE[k]
        if by_id:
            for k in [k for k, v in _ID_CACHE.items() if v[0]() is None or v[1]() is None or not v[2]._h]:
                del _ID_CACHE[k]
            _ID_CACHE[(id(flow), id(dist), device)] = (weakref.ref(flow), weakref.ref(dist), inst, key)
        return inst


def clear_cache() -> None:
    with _CACHE_LOCK:
        _ID_CACHE.clear()
        while _CACHE:
            _, old = _CACHE.popitem()
            old.close()


class _CudaKernels:
    """Drop-in for the module object `qapsolve.backend.kernels`."""

    BACKEND_NAME = "cuda-sm100a"

    @staticmethod
    def full_cost(flow, dist, perm) -> int:
        return int(device_instance(flow, dist).full_cost(perm)[0])

    @staticmethod
    def all_deltas(flow, dist, perm) -> np.ndarray:
        return device_instance(flow, dist).all_deltas(perm)[0]

    @staticmethod
    def two_opt_run(flow, dist, perm, iterations: int):
        """(best, best_cost, current, current_cost, move_i, move_j, move_delta) -- _kernels.pyx:118."""
        if int(iterations) == 0:  # no sweep: the start is the answer (the loop of _kernels.pyx:94 does not run)
            p0 = np.array(perm, dtype=_i64)
            c0 = _CudaKernels.full_cost(flow, dist, p0)
            empty = np.zeros(0, _i64)
            return p0, c0, p0.copy(), c0, empty, empty.copy(), empty.copy()
        best, bc, cur, cc, mi, mj, md = device_instance(flow, dist).two_opt(perm, int(iterations))
        return best[0], int(bc[0]), cur[0], int(cc[0]), mi[0], mj[0], md[0]

    @staticmethod
    def tabu_run(flow, dist, perm, iterations: int, tenures):
        """(best, best_cost, current, current_cost, cells, stopped_early, steps_done, trail)
        with trail = (i, j, delta, tabu_flag, aspirated_flag, tenure), each cut to
        steps_done -- _kernels.pyx:189-197."""
        if int(iterations) == 0:
            p0 = np.array(perm, dtype=_i64)
            c0 = _CudaKernels.full_cost(flow, dist, p0)
            n = p0.shape[0]
            return (p0, c0, p0.copy(), c0, np.zeros((n, n), _i64), False, 0,
                    tuple(np.zeros(0, _i64) for _ in range(6)))
        best, bc, cur, cc, cz, stop, steps, tr, ten = device_instance(flow, dist).tabu(
            perm, int(iterations), tenures)
        k = int(steps[0])
        flags = tr[3][0, :k].copy()
        trail = (tr[0][0, :k].copy(), tr[1][0, :k].copy(), tr[2][0, :k].copy(), flags, flags.copy(),
                 ten[0, :k].copy())
        return best[0], int(bc[0]), cur[0], int(cc[0]), cz[0], bool(stop[0]), k, trail

    # batched additions -------------------------------------------------------------
    @staticmethod
    def full_cost_batch(flow, dist, perms) -> np.ndarray:
        return device_instance(flow, dist).full_cost(perms)

    @staticmethod
    def all_deltas_batch(flow, dist, perms) -> np.ndarray:
        return device_instance(flow, dist).all_deltas(perms)

    @staticmethod
    def two_opt_run_batch(flow, dist, perms, iterations: int, moves: bool = True):
        return device_instance(flow, dist).two_opt(perms, int(iterations), moves)

    @staticmethod
    def tabu_run_batch(flow, dist, perms, iterations: int, tenures, cells: bool = True, trail: bool = True):
        return device_instance(flow, dist).tabu(perms, int(iterations), tenures, cells, trail)[:8]

    @staticmethod
    def multistart(flow, dist, algorithm: str, master_seed: int, first_index: int, count: int,
                   iterations: int, ten_low: int = 1, ten_high: int = 1, device: int = 0):
        return device_instance(flow, dist, device).multistart(
            algorithm, master_seed, first_index, count, iterations, ten_low, ten_high)


kernels = _CudaKernels()


def backend_name() -> str:
    return kernels.BACKEND_NAME
