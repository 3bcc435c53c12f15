"""Locate the reference package `qapsolve`.

BASELINE.json's north_star keeps the reference's loader, result objects and error types UNCHANGED around
the accelerated path.  So when a `qapsolve` can be imported this package does not define its own: it
re-exports the reference's `Instance`, `parse_instance`, `SolutionRecord`, `TabuTrail`,
`replay_and_audit`, error classes ... and plugs the CUDA kernels in underneath.  Only when no `qapsolve` is
around does a small independent fallback (instance.py, errors.py, tabu.py) provide the few types the hot
path itself needs.

Search order: an importable `qapsolve`; `$QAPSOLVE_SRC`; the copy under `baseline/_ref/pkg/src` that
scripts/ref_suite_on_cuda.py makes for the test-suite.  `QAPB_NO_QAPSOLVE=1` forces the fallback."""

from __future__ import annotations

import importlib
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_cached = False
_module = None


def reference():
    """The `qapsolve` module, or None."""
    global _cached, _module
    if _cached:
        return _module
    _cached = True
    if os.environ.get("QAPB_NO_QAPSOLVE") == "1":
        return None
    candidates = [None, os.environ.get("QAPSOLVE_SRC"), os.path.join(_ROOT, "baseline", "_ref", "pkg", "src")]
    for path in candidates:
        if path is not None and not os.path.isdir(os.path.join(path, "qapsolve")):
            continue
        added = path is not None and path not in sys.path
        if added:
            sys.path.append(path)
        # host-side objects only: the reference's own kernel backend is not what runs here, so let it settle
        # on its pure fallback instead of looking for a compiled module
        forced = "QAPSOLVE_BACKEND" not in os.environ and path is not None
        if forced:
            os.environ["QAPSOLVE_BACKEND"] = "python"
        try:
            _module = importlib.import_module("qapsolve")
            return _module
        except ImportError:
            if added:
                sys.path.remove(path)
        finally:
            if forced:
                del os.environ["QAPSOLVE_BACKEND"]
    return None


def missing(name: str):
    """Placeholder for a reference function that has no fallback here."""

    def _unavailable(*_args, **_kwargs):
        raise ImportError(f"{name} is provided by the reference package `qapsolve` (unchanged around the CUDA path); "
                          "install it or point QAPSOLVE_SRC at its src directory")

    _unavailable.__name__ = name
    return _unavailable
