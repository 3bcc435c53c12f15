"""Build and bind `libqapb.so` (the C ABI declared in include/qapb.h).

The library is compiled in-tree with nvcc for sm_100a only and loaded with
ctypes.  There is no CPU or PyTorch fallback: if the library is missing or no
CUDA device is present, every compute entry raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, Structure, c_char_p, c_double, c_float, c_int, c_int32, c_int64, c_uint64, c_void_p

from .errors import DomainError, QapError

_PKG = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_PKG, "csrc")
# QAPB_LIB: development override (a single-instantiation build from scripts/devbuild.sh)
LIB_PATH = os.environ.get("QAPB_LIB") or os.path.join(_PKG, "libqapb.so")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
]

OK, ERR_INVALID, ERR_CUDA, ERR_NOMEM, ERR_UNSUPPORTED = 0, 1, 2, 3, 4
ALGO_2OPT, ALGO_TABU = 0, 1

_i64p = POINTER(c_int64)


class Info(Structure):
    _fields_ = [
        ("n", c_int32), ("device", c_int32), ("acc_bits", c_int32), ("symmetric", c_int32),
        ("threads", c_int32), ("units_per_thread", c_int32), ("storage", c_int32),
        ("smem_bytes", c_int32), ("ctas_per_sm", c_int32), ("sm_count", c_int32),
        ("delta_bound", c_int64),
    ]


def _sources() -> list[str]:
    return [os.path.join(_SRC, f) for f in sorted(os.listdir(_SRC)) if f.endswith((".cu", ".cuh"))] + [
        os.path.join(os.path.dirname(_PKG), "include", "qapb.h")
    ]


def _source_digest() -> str:
    """sha256 over the sources and the compiler flags: decides whether the in-tree library is current
    (file times do not survive being copied to another machine)."""
    import hashlib

    h = hashlib.sha256(" ".join(NVCC_FLAGS + os.environ.get("NVCC_EXTRA", "").split()).encode())
    for path in _sources():
        with open(path, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def build_library(force: bool = False, verbose: bool = False) -> str:
    """nvcc -gencode arch=compute_100a,code=sm_100a ... -> paper_2307_11248_b200/libqapb.so"""
    digest, stamp = _source_digest(), LIB_PATH + ".hash"
    if not force and os.path.exists(LIB_PATH) and os.path.exists(stamp):
        with open(stamp) as fh:
            if fh.read().strip() == digest:
                return LIB_PATH
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, *os.environ.get("NVCC_EXTRA", "").split(), "-o", LIB_PATH, os.path.join(_SRC, "qapb.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise QapError(f"nvcc failed:\n{proc.stdout}\n{proc.stderr}")
    with open(stamp, "w") as fh:
        fh.write(digest + "\n")
    if verbose:
        print(proc.stderr)
    return LIB_PATH


_lib = None

# name -> (restype, argtypes); kept in one table so tests can check that every
# symbol declared in include/qapb.h is exported and bound.
_P = c_void_p  # device or host pointer, passed as an integer address
SIGNATURES = {
    "qapb_version": (c_int, []),
    "qapb_last_error": (c_char_p, []),
    "qapb_device_count": (c_int, [POINTER(c_int)]),
    "qapb_create": (c_int, [c_int, _P, _P, c_int, POINTER(c_void_p)]),
    "qapb_destroy": (c_int, [c_void_p]),
    "qapb_get_info": (c_int, [c_void_p, POINTER(Info)]),
    "qapb_full_cost": (c_int, [c_void_p, _P, c_int, _P, c_void_p]),
    "qapb_all_deltas": (c_int, [c_void_p, _P, c_int, _P, c_void_p]),
    "qapb_two_opt": (c_int, [c_void_p, _P, c_int, c_int] + [_P] * 7 + [c_void_p]),
    "qapb_tabu": (c_int, [c_void_p, _P, c_int, c_int, _P] + [_P] * 11 + [c_void_p]),
    "qapb_multistart": (c_int, [c_void_p, c_int, c_uint64, c_uint64, c_int, c_int, c_int64, c_int64, _P, _P, _P, c_void_p]),
    "qapb_multistart_seeds": (c_int, [c_void_p, c_int, _P, c_int, c_int, c_int64, c_int64, _P, _P, c_void_p]),
    "qapb_multistart_trace": (c_int, [c_void_p, c_int, _P, c_int, c_int, c_int64, c_int64] + [_P] * 6 + [c_void_p]),
    "qapb_full_cost_host": (c_int, [c_void_p, _P, c_int, _P]),
    "qapb_all_deltas_host": (c_int, [c_void_p, _P, c_int, _P]),
    "qapb_two_opt_host": (c_int, [c_void_p, _P, c_int, c_int] + [_P] * 7),
    "qapb_tabu_host": (c_int, [c_void_p, _P, c_int, c_int, _P] + [_P] * 11),
    "qapb_multistart_host": (c_int, [c_void_p, c_int, c_uint64, c_uint64, c_int, c_int, c_int64, c_int64, _P, _P, _P]),
    "qapb_multistart_seeds_host": (c_int, [c_void_p, c_int, _P, c_int, c_int, c_int64, c_int64, _P, _P]),
    "qapb_multistart_trace_host": (c_int, [c_void_p, c_int, _P, c_int, c_int, c_int64, c_int64] + [_P] * 6),
    "qapb_plan_candidates": (c_int, [c_void_p, _P, c_int, POINTER(c_int)]),
    "qapb_set_plan": (c_int, [c_void_p, c_int, c_int, c_int, c_int]),
    "qapb_last_kernel_ms": (c_int, [c_void_p, POINTER(c_float)]),
    "qapb_probe_int_peak": (c_int, [c_int, c_int, POINTER(c_double)]),
    "qapb_probe_smem_peak": (c_int, [c_int, POINTER(c_double)]),
    "qapb_last_total_steps": (c_int, [c_void_p, POINTER(c_int64)]),
}


def lib():
    """The loaded library.  Raises ImportError if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(nvcc, sm_100a).  There is no CPU fallback."
            )
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        L.qapb_debug_force_seq_rng.restype = c_int
        L.qapb_debug_force_seq_rng.argtypes = [c_void_p, c_int]
        _lib = L
    return _lib


def check(status: int) -> None:
    """Map a C-ABI status onto the reference's exception classes."""
    if status == OK:
        return
    msg = lib().qapb_last_error().decode(errors="replace")
    if status == ERR_INVALID:
        raise DomainError(msg)
    raise QapError(f"libqapb status {status}: {msg}")


def device_count() -> int:
    n = c_int(0)
    check(lib().qapb_device_count(ctypes.byref(n)))
    return int(n.value)
