"""Launch-configuration space and its autotuner.

`ThreadConfig`, `validate_config` and `enumerate_configs` keep the reference's (N, t, b) set
(/root/reference/pkg/src/qapsolve/tuner.py:18-78: N starts in b blocks of t threads, everything in
warp multiples, 1024 <= N <= 12288, 32 <= t <= 1024, b = N / t).  On the reference the set only
parameterises sweeps ("execution itself uses a flat worker pool", tuner.py:8-9).  Here the launch
configuration is real: N is the grid (one CTA per start), and how one search is laid out on an SM --
CTA size, units per thread in registers / shared memory, where the diagonal blocks live -- is a
*plan* of the search kernel (csrc/qapb.cu: plan_hybrid).  `autotune` times every plan that fits an
instance on the device and installs the fastest; results are bit-identical under every plan.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import DomainError, QapError
from .instance import Instance
from .tabu import tenure_bounds

N_STARTS_MIN, N_STARTS_MAX = 1024, 12288
THREADS_MIN, THREADS_MAX = 32, 1024
WARP = 32


@dataclass(frozen=True)
class ThreadConfig:
    n_starts: int
    threads_per_block: int
    blocks: int


def validate_config(c: ThreadConfig) -> tuple[bool, list[str]]:
    """Every constraint of the (N, t, b) set; violations name the failed rule (tuner.py:35-61)."""
    bad: list[str] = []
    if not N_STARTS_MIN <= c.n_starts <= N_STARTS_MAX:
        bad.append(f"n_starts {c.n_starts} outside [{N_STARTS_MIN}, {N_STARTS_MAX}]")
    if c.n_starts % WARP:
        bad.append(f"n_starts {c.n_starts} not a multiple of warp size {WARP}")
    if not THREADS_MIN <= c.threads_per_block <= THREADS_MAX:
        bad.append(f"threads_per_block {c.threads_per_block} outside [{THREADS_MIN}, {THREADS_MAX}]")
    if c.threads_per_block % WARP:
        bad.append(f"threads_per_block {c.threads_per_block} not a multiple of warp size {WARP}")
    if c.threads_per_block <= 0 or c.n_starts % c.threads_per_block:
        bad.append(f"n_starts {c.n_starts} not divisible by threads_per_block {c.threads_per_block}")
    elif c.blocks != c.n_starts // c.threads_per_block:
        bad.append(f"blocks {c.blocks} != n_starts / threads_per_block ({c.n_starts // c.threads_per_block})")
    return not bad, bad


def enumerate_configs(n_starts_filter: int | None = None) -> list[ThreadConfig]:
    """All valid (N, t, b) triples ordered by (N, t) (tuner.py:64-78)."""
    starts = [n_starts_filter] if n_starts_filter is not None else range(N_STARTS_MIN, N_STARTS_MAX + 1, WARP)
    out = []
    for n in starts:
        if not (N_STARTS_MIN <= n <= N_STARTS_MAX and n % WARP == 0):
            continue
        out.extend(ThreadConfig(n, t, n // t) for t in range(THREADS_MIN, THREADS_MAX + 1, WARP) if n % t == 0)
    return out


@dataclass(frozen=True)
class PlanTiming:
    plan: tuple[int, int, int, int]  # (register units, unit threads, shared-memory units, diagonal blocks in shared memory)
    threads: int                     # CTA size
    ctas_per_sm: int                 # resident searches per SM
    milliseconds: float
    evals_per_second: float


def autotune(inst: Instance, *, algorithm: str = "tabu", n_starts: int | None = None,
             iterations: int | None = None, device: int = 0, repeats: int = 2) -> list[PlanTiming]:
    """Time every launch plan that fits `inst` (a short multi-start each, CUDA events) and leave the
    fastest installed on the cached device instance.  Returns the timings, fastest first; an empty
    list for instances served by the generic kernel (a single configuration)."""
    from .backend import device_instance

    if algorithm not in ("2opt", "tabu"):
        raise DomainError(f"unknown algorithm {algorithm!r}")
    di = device_instance(inst.flow, inst.distance, device)
    plans = di.plan_candidates()
    if not plans:
        return []
    sm = di.info["sm_count"]
    ten = tenure_bounds(inst.n)
    iters = iterations if iterations is not None else max(32, 2 * inst.n)
    timings = []
    for plan in plans:
        di.set_plan(plan)
        # fill every SM for two waves under this plan unless the caller fixed the batch
        count = n_starts if n_starts is not None else 2 * sm * max(1, di.info["ctas_per_sm"])
        best, steps = None, 0
        for rep in range(max(1, repeats)):
            di.multistart(algorithm, rep, 0, count, iters, ten.low, ten.high)
            ms = di.last_kernel_ms()
            if best is None or ms < best:
                best, steps = ms, di.last_total_steps()  # a tabu start can stop early: count the steps it did
        evals = steps * inst.n * (inst.n - 1) // 2
        timings.append(PlanTiming(plan, di.info["threads"], di.info["ctas_per_sm"], best, evals / (best * 1e-3)))
    timings.sort(key=lambda t: -t.evals_per_second)
    if not timings:
        raise QapError("no launch plan could be timed")
    di.set_plan(timings[0].plan)
    return timings
