#!/usr/bin/env python
"""Put the UNMODIFIED reference package next to the CUDA backend and make it selectable there.

    python scripts/ref_suite_on_cuda.py            (in the build container, where /root/reference exists)

Copies /root/reference/pkg to baseline/_ref/pkg (git-ignored, ships to the GPU box with the snapshot) and
applies exactly what INTEGRATION.md tells a maintainer of `qapsolve` to do:
  1. add integration/_cudakernels.py as qapsolve/_cudakernels.py;
  2. one branch in backend.py: QAPSOLVE_BACKEND=cuda selects it;
  3. run_multistart hands the whole map + reduce to the batched entry when that backend is active
     (the reference forks a process pool, which cannot follow a CUDA context: multistart.py:141-150);
  4. qapsolve/_kernels.py re-exports the CUDA stub, so that the reference's own tests/test_backends.py --
     which imports `qapsolve._kernels` and `qapsolve._purekernels` and compares every returned array --
     compares the CUDA kernels with the pure backend, unchanged.
Nothing else of the copy is touched; tests/test_reference_suite_gpu.py runs its test files on the B200."""
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/pkg"
DST = os.path.join(ROOT, "baseline", "_ref", "pkg")


def patch(path, anchor, replacement):
    with open(path) as fh:
        text = fh.read()
    assert text.count(anchor) == 1, f"{path}: anchor not found exactly once: {anchor!r}"
    with open(path, "w") as fh:
        fh.write(text.replace(anchor, replacement))


def main():
    if not os.path.isdir(SRC):
        sys.exit(f"{SRC} is not here; run this in the build container")
    if os.path.isdir(DST):
        shutil.rmtree(DST)
    shutil.copytree(SRC, DST, ignore=shutil.ignore_patterns("__pycache__", "*.so", "build", "*.egg-info", ".pytest_cache", ".hypothesis"))
    pkg = os.path.join(DST, "src", "qapsolve")
    shutil.copy(os.path.join(ROOT, "integration", "_cudakernels.py"), os.path.join(pkg, "_cudakernels.py"))
    with open(os.path.join(pkg, "_kernels.py"), "w") as fh:
        fh.write('"""The compiled-kernel slot of this copy is served by the CUDA library (see _cudakernels.py)."""\n'
                 "from ._cudakernels import BACKEND_NAME, all_deltas, full_cost, tabu_run, two_opt_run  # noqa: F401\n")
    patch(os.path.join(pkg, "backend.py"),
          'elif _forced == "c":\n',
          'elif _forced == "cuda":\n    from . import _cudakernels as kernels  # type: ignore[no-redef]\nelif _forced == "c":\n')
    patch(os.path.join(pkg, "multistart.py"),
          '    t0 = time.perf_counter()\n    workers = cfg.resolved_workers()\n',
          '    t0 = time.perf_counter()\n'
          '    from . import backend as _backend\n\n'
          '    if _backend.kernels.BACKEND_NAME.startswith("cuda"):  # batched persistent-kernel multi-start, one launch\n'
          '        from .tabu import tenure_bounds\n\n'
          '        ten = cfg.tenure or tenure_bounds(inst.n)\n'
          '        costs, b_cost, b_index, b_perm = _backend.kernels.multistart(\n'
          '            inst.flow, inst.distance, cfg.algorithm, cfg.master_seed, cfg.n_starts,\n'
          '            cfg.resolved_iterations(inst.n), ten.low, ten.high)\n'
          '        cfg.resolved_workers()  # still validated\n'
          '        digest = config_digest(inst, cfg)\n'
          '        best = SolutionRecord(instance_name=inst.name, permutation=b_perm, cost=int(b_cost), algorithm=cfg.algorithm,\n'
          '                              seed=derive_seed(cfg.master_seed, b_index), config_digest=digest)\n'
          '        return MultiStartResult(best=best, per_start_costs=costs, wall_time=time.perf_counter() - t0,\n'
          '                                config_digest=digest, best_start_index=int(b_index))\n'
          '    workers = cfg.resolved_workers()\n')
    print("reference copy with the CUDA backend:", DST)


if __name__ == "__main__":
    main()
