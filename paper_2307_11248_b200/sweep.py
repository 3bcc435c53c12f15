"""Batched repetitions and parameter sweeps: many `run_multistart` calls in one launch.

The reference's bench and sweep commands call `run_multistart` once per repetition
(`master_seed + rep`, /root/reference/pkg/src/qapsolve/cli.py:109-116) and once per sweep point
(`cli.py:162-175`; the seeds axis runs `value` master seeds `seed + 7919 * idx`), each call
paying a process-pool start-up.  On the GPU every start is one CTA of one persistent launch,
so all runs that share (algorithm, iterations, tenure) are concatenated into a single
`qapb_multistart_seeds` launch -- start `index` of a run with master seed `m` still uses
`derive_seed(m, index)` (multistart.py:88), so each run's `MultiStartResult` is bit-identical
to a separate `run_multistart` call.  `SweepPlan`, `make_sweep` and `expand` keep the
reference's names and validation rules (tuner.py:83-131).  The batch runs on the calling rank's
GPU; sharding over ranks is `run_multistart`'s job (one config at a time).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, replace
from typing import Iterator, Sequence

import numpy as np

from .errors import DomainError, QapError
from .instance import Instance, SolutionRecord
from .multistart import MultiStartResult, SearchConfig, config_digest
from .rng import GAMMA, derive_seed

SWEEP_AXES = ("neighborhoods", "instances", "seeds")
MAX_SWEEP_INSTANCES = 1024
SEED_STRIDE = 7919  # cli.py:173


def derive_seeds(master_seed: int, first_index: int, count: int) -> np.ndarray:
    """`derive_seed(master_seed, i)` for i in [first_index, first_index + count), vectorised (uint64)."""
    with np.errstate(over="ignore"):
        k = np.arange(first_index + 1, first_index + count + 1, dtype=np.uint64)
        z = np.uint64(master_seed & 0xFFFFFFFFFFFFFFFF) + np.uint64(GAMMA) * k
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _group_key(inst: Instance, cfg: SearchConfig):
    ten = cfg.resolved_tenure(inst.n)
    return (cfg.algorithm, cfg.resolved_iterations(inst.n), ten.low, ten.high)


def _cuda_seed_runner(inst: Instance, algorithm: str, seeds: np.ndarray, iterations: int, low: int, high: int):
    import torch

    from .backend import device_instance

    if not torch.cuda.is_available():
        raise QapError("no CUDA device: the multi-start path has no CPU fallback")
    di = device_instance(inst.flow, inst.distance, torch.cuda.current_device())
    return di.multistart_seeds(algorithm, seeds, iterations, low, high)


def run_multistart_many(inst: Instance, configs: Sequence[SearchConfig], *, _seed_runner=None) -> list[MultiStartResult]:
    """`[run_multistart(inst, c) for c in configs]`, with every group of configs that shares
    (algorithm, iterations, tenure) executed as ONE launch.  `_seed_runner` exists for the CPU
    tests of the grouping/splitting logic; production calls never pass it."""
    runner = _seed_runner or _cuda_seed_runner
    t0 = time.perf_counter()
    groups: dict[tuple, list[int]] = {}
    for k, cfg in enumerate(configs):
        groups.setdefault(_group_key(inst, cfg), []).append(k)
    out: list[MultiStartResult | None] = [None] * len(configs)
    for (algorithm, iterations, low, high), members in groups.items():
        seeds = np.concatenate([derive_seeds(configs[k].master_seed, 0, configs[k].n_starts) for k in members])
        costs, perms = runner(inst, algorithm, seeds, iterations, low, high)
        offset = 0
        for k in members:
            cfg = configs[k]
            mine = np.asarray(costs[offset:offset + cfg.n_starts], dtype=np.int64)
            best_index = int(mine.argmin())  # first minimum: ties -> lowest index (multistart.py:114,156)
            digest = config_digest(inst, cfg)
            best = SolutionRecord(
                instance_name=inst.name,
                permutation=np.asarray(perms[offset + best_index], dtype=np.int64).copy(),
                cost=int(mine[best_index]),
                algorithm=cfg.algorithm,
                seed=derive_seed(cfg.master_seed, best_index),
                config_digest=digest,
            )
            out[k] = MultiStartResult(best=best, per_start_costs=mine.copy(), wall_time=0.0,
                                      config_digest=digest, best_start_index=best_index)
            offset += cfg.n_starts
    elapsed = time.perf_counter() - t0
    for res in out:
        res.wall_time = elapsed  # the batch ran as a whole
    return out  # type: ignore[return-value]


def _cuda_trace_runner(inst: Instance, algorithm: str, seeds: np.ndarray, iterations: int, low: int, high: int):
    import torch

    from .backend import device_instance

    if not torch.cuda.is_available():
        raise QapError("no CUDA device: the multi-start path has no CPU fallback")
    di = device_instance(inst.flow, inst.distance, torch.cuda.current_device())
    costs, _perms, steps, _mi, _mj, deltas = di.multistart_trace(algorithm, seeds, iterations, low, high)
    return costs, steps, deltas


def best_costs_at_budgets(inst: Instance, cfg: SearchConfig, budgets: Sequence[int], *, _trace_runner=None) -> np.ndarray:
    """Best cost of every start of `cfg` after each iteration budget in `budgets`, from ONE run at the
    largest budget: array [len(budgets), n_starts], row k equal to
    `run_multistart(inst, replace(cfg, iterations=budgets[k])).per_start_costs`.

    A run's tenure stream is drawn in order after its start permutation (tabu.py:184-186), so the
    run with budget v is the first v iterations of any longer run (and a start that stops early,
    _kernels.pyx:168-170, stops at the same step under every budget that reaches it).  The recorded
    move deltas give the cost after each step; the running minimum is the best-so-far."""
    if not budgets or any(v < 1 for v in budgets):
        raise DomainError("budgets must be a non-empty list of positive iteration counts")
    runner = _trace_runner or _cuda_trace_runner
    ten = cfg.resolved_tenure(inst.n)
    top = max(budgets)
    seeds = derive_seeds(cfg.master_seed, 0, cfg.n_starts)
    costs, steps, deltas = runner(inst, cfg.algorithm, seeds, top, ten.low, ten.high)
    costs = np.asarray(costs, dtype=np.int64)
    steps = np.asarray(steps, dtype=np.int64)
    deltas = np.asarray(deltas, dtype=np.int64)[:, :top]
    live = np.arange(top)[None, :] < steps[:, None]
    walk = np.cumsum(np.where(live, deltas, 0), axis=1)  # cost after each step, relative to the start cost
    low_water = np.minimum.accumulate(np.minimum(walk, 0), axis=1)  # best-so-far (strict <: ties keep the earlier best)
    start_cost = costs - low_water[:, -1]
    return np.stack([start_cost + low_water[:, min(v, top) - 1] for v in budgets])


def run_repetitions(inst: Instance, cfg: SearchConfig, repetitions: int) -> list[MultiStartResult]:
    """The bench loop of cli.py:113-115: master seeds `cfg.master_seed + rep`, one launch."""
    if repetitions < 1:
        raise DomainError(f"repetitions must be >= 1, got {repetitions}")
    return run_multistart_many(inst, [replace(cfg, master_seed=cfg.master_seed + rep) for rep in range(repetitions)])


@dataclass(frozen=True)
class SweepPlan:
    axis: str
    values: tuple[int, ...]
    base: SearchConfig


def make_sweep(axis: str, values: list[int], base: SearchConfig) -> SweepPlan:
    """Validate a sweep over iteration count, start count or seed count (tuner.py:90-114)."""
    if axis not in SWEEP_AXES:
        raise DomainError(f"unknown sweep axis {axis!r}; expected one of {SWEEP_AXES}")
    if not values:
        raise DomainError("sweep values must be non-empty")
    if any(v <= 0 for v in values):
        raise DomainError("sweep values must be positive")
    if list(values) != sorted(set(values)):
        raise DomainError("sweep values must be strictly increasing")
    if axis == "instances":
        for v in values:
            if v & (v - 1) != 0:
                raise DomainError(f"instances axis requires powers of two, got {v}")
            if v > MAX_SWEEP_INSTANCES:
                raise DomainError(f"instances axis is bounded at {MAX_SWEEP_INSTANCES}, got {v}")
    return SweepPlan(axis=axis, values=tuple(values), base=base)


def expand(plan: SweepPlan, repetitions: int) -> Iterator[tuple[int, int, int]]:
    """(axis_value, repetition, master_seed) for every planned run (tuner.py:117-122)."""
    for value in plan.values:
        for rep in range(repetitions):
            yield value, rep, plan.base.master_seed + rep


def run_sweep(inst: Instance, plan: SweepPlan, repetitions: int) -> list[tuple[int, int, int]]:
    """Rows (axis_value, repetition, best_cost) of the reference's sweep command (cli.py:162-175):
    neighborhoods -> iterations = value (all budgets of a repetition from one traced run,
    `best_costs_at_budgets`); instances -> n_starts = value; seeds -> minimum over `value` master
    seeds `seed + 7919 * idx`.  The latter two go through `run_multistart_many`."""
    rows = list(expand(plan, repetitions))
    if plan.axis == "neighborhoods":
        # every budget of one repetition is a prefix of its longest run: one traced run per repetition
        table = {seed: best_costs_at_budgets(inst, replace(plan.base, master_seed=seed), list(plan.values))
                 for seed in sorted({seed for _v, _r, seed in rows})}
        return [(value, rep, int(table[seed][plan.values.index(value)].min())) for value, rep, seed in rows]
    configs: list[SearchConfig] = []
    spans: list[tuple[int, int]] = []
    for value, _rep, seed in rows:
        first = len(configs)
        if plan.axis == "neighborhoods":
            configs.append(replace(plan.base, iterations=value, master_seed=seed))
        elif plan.axis == "instances":
            configs.append(replace(plan.base, n_starts=value, master_seed=seed))
        else:
            configs.extend(replace(plan.base, master_seed=seed + SEED_STRIDE * idx) for idx in range(value))
        spans.append((first, len(configs)))
    results = run_multistart_many(inst, configs)
    return [(value, rep, min(results[k].best.cost for k in range(lo, hi)))
            for (value, rep, _seed), (lo, hi) in zip(rows, spans)]
