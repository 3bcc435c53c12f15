"""Batched multi-start: N independent searches, minimum-cost reduction.

Same public surface as /root/reference/pkg/src/qapsolve/multistart.py
(`SearchConfig`, `config_digest`, `MultiStartResult`, `run_start`,
`run_multistart`).  Where the reference maps starts over a process pool
(multistart.py:141-150), this module runs all starts of a rank in ONE persistent
kernel launch (device-side SplitMix64 -> shuffle -> tenure stream -> search) and,
under `torch.distributed`, shards the start indices contiguously over the ranks
(one rank per GPU) and picks the global winner with a single all-reduce(min) of a
packed (cost, index) key.  Start `index` always uses
`derive_seed(master_seed, index)` (multistart.py:88), so the result is a pure
function of (instance, config): any number of GPUs gives identical
`MultiStartResult`s -- the property the reference tests for worker counts.
"""

from __future__ import annotations

import hashlib
import json
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import tabu as tabu_mod
from . import two_opt as two_opt_mod
from .errors import DomainError, QapError
from .instance import Instance, SolutionRecord
from .rng import SplitMix64, derive_seed
from .tabu import TenureInterval, run_tabu
from .two_opt import run_two_opt

ALGORITHMS = ("2opt", "tabu")
_I64_MAX = np.iinfo(np.int64).max
_I64_MIN = np.iinfo(np.int64).min  # in-band "this rank failed" marker of the min-reduction


@dataclass(frozen=True)
class SearchConfig:
    algorithm: str = "tabu"
    n_starts: int = 6144
    iterations: int | None = None  # None: 4n (2opt) / 8n (tabu)
    tenure: TenureInterval | None = None
    master_seed: int = 0
    workers: int | str = "auto"  # accepted for compatibility; GPU sharding is by rank

    def __post_init__(self):
        if self.algorithm not in ALGORITHMS:
            raise DomainError(f"unknown algorithm {self.algorithm!r}")
        if self.n_starts < 1:
            raise DomainError(f"n_starts must be >= 1, got {self.n_starts}")
        if self.iterations is not None and self.iterations < 1:
            raise DomainError(f"iterations must be >= 1, got {self.iterations}")

    def resolved_iterations(self, n: int) -> int:
        if self.iterations is not None:
            return self.iterations
        return (tabu_mod if self.algorithm == "tabu" else two_opt_mod).default_iterations(n)

    def resolved_workers(self) -> int:
        if self.workers == "auto":
            return os.cpu_count() or 1
        count = int(self.workers)
        if count < 1:
            raise DomainError(f"workers must be >= 1, got {count}")
        return count

    def resolved_tenure(self, n: int) -> TenureInterval:
        return self.tenure or tabu_mod.tenure_bounds(n)


def config_digest(inst: Instance, cfg: SearchConfig) -> str:
    """16 hex digits over everything the result depends on -- same payload, key order
    and hash as multistart.py:63-74, so digests are interchangeable with the reference."""
    fields = {
        "instance": inst.name,
        "n": inst.n,
        "algorithm": cfg.algorithm,
        "n_starts": cfg.n_starts,
        "iterations": cfg.resolved_iterations(inst.n),
        "tenure": None if cfg.tenure is None else [cfg.tenure.low, cfg.tenure.high],
        "master_seed": cfg.master_seed,
    }
    blob = json.dumps(fields, sort_keys=True).encode()
    return hashlib.sha256(blob).hexdigest()[:16]


@dataclass
class MultiStartResult:
    best: SolutionRecord
    per_start_costs: np.ndarray
    wall_time: float
    config_digest: str
    best_start_index: int = field(default=0)


def run_start(inst: Instance, cfg: SearchConfig, index: int) -> SolutionRecord:
    """The single search owned by start `index` (multistart.py:86-93), through the
    single-start kernel entries with host-drawn inputs."""
    rng = SplitMix64(derive_seed(cfg.master_seed, index))
    iters = cfg.resolved_iterations(inst.n)
    if cfg.algorithm == "tabu":
        return run_tabu(inst, rng, iters, cfg.tenure)[0]
    return run_two_opt(inst, rng, iters)


def shard_bounds(n_starts: int, world_size: int, rank: int) -> tuple[int, int]:
    """Contiguous index range [lo, hi) of `rank`: floor(rank*N/G) .. floor((rank+1)*N/G)."""
    return rank * n_starts // world_size, (rank + 1) * n_starts // world_size


def _cuda_shard_runner(inst: Instance, cfg: SearchConfig, first_index: int, count: int):
    """Run starts [first_index, first_index+count) on this rank's GPU.

    Returns torch tensors on the device: costs[count], key[2] = (best cost, global
    index), perm[n]."""
    import torch

    from .backend import device_instance

    if not torch.cuda.is_available():
        raise QapError("no CUDA device: the multi-start path has no CPU fallback")
    dev = torch.cuda.current_device()
    device = torch.device("cuda", dev)
    # one device block [costs | key | perm]: a single read-back on the single-GPU path
    block = torch.empty(count + 2 + inst.n, dtype=torch.int64, device=device)
    costs, key, perm = block[:count], block[count:count + 2], block[count + 2:]
    if count == 0:
        key.fill_(_I64_MAX)
        perm.zero_()
    if count > 0:
        ten = cfg.resolved_tenure(inst.n)
        di = device_instance(inst.flow, inst.distance, dev)
        di.multistart_device(
            cfg.algorithm, cfg.master_seed, first_index, count, cfg.resolved_iterations(inst.n),
            ten.low, ten.high, costs.data_ptr(), key.data_ptr(), perm.data_ptr(),
            torch.cuda.current_stream(device).cuda_stream)
    return costs, key, perm


def _index_bits(n_starts: int) -> int:
    return max(1, (n_starts - 1).bit_length())


def _packable(inst: Instance, n_starts: int) -> bool:
    """True when every reachable cost is in [0, 2^(62-b)): then (cost, index) packs
    into one int64 whose min is the lexicographic min.  Decided from the instance
    alone so all ranks agree."""
    if int(inst.flow.min()) < 0 or int(inst.distance.min()) < 0:
        return False
    ub = int(np.abs(inst.flow).max()) * int(np.abs(inst.distance).max()) * inst.n * inst.n
    return ub < (1 << (62 - _index_bits(n_starts)))


def run_multistart(inst: Instance, cfg: SearchConfig, *, group=None, _shard_runner=None) -> MultiStartResult:
    """Run cfg.n_starts searches and reduce to (min cost, lowest index).

    With an initialised `torch.distributed` process group (one rank per GPU) the
    starts are sharded over the ranks and every rank returns the same result.
    `_shard_runner` exists for the CPU (gloo) tests of the sharding/reduction
    logic; production calls never pass it."""
    import torch
    import torch.distributed as dist

    t0 = time.perf_counter()
    world, rank = 1, 0
    grouped = dist.is_available() and dist.is_initialized()
    if grouped:
        world, rank = dist.get_world_size(group), dist.get_rank(group)
    # a one-rank group normally skips the collectives; QAPB_FORCE_COLLECTIVE=1 takes them anyway (how the
    # NCCL branch is exercised on a single-GPU box)
    collective = world > 1 or (grouped and os.environ.get("QAPB_FORCE_COLLECTIVE") == "1")
    lo, hi = shard_bounds(cfg.n_starts, world, rank)
    runner = _shard_runner or _cuda_shard_runner
    failure = None
    if not collective:
        costs, key, perm = runner(inst, cfg, lo, hi - lo)
    else:
        # The reference discards partial results when a worker fails (multistart.py:151-154: QapError).  Here a
        # rank-local failure must not leave the other ranks waiting in the all-reduce: the failing rank still
        # takes part, contributing the smallest int64 -- the min-reduction hands it to everyone and every rank
        # raises QapError.  (A CUDA fault that poisons the context also breaks NCCL on that rank; then the
        # others fail at the process group's timeout.)
        try:
            costs, key, perm = runner(inst, cfg, lo, hi - lo)
            if costs.is_cuda:
                torch.cuda.current_stream(costs.device).synchronize()  # surface asynchronous launch errors here
        except Exception as exc:  # noqa: BLE001 -- any failure of this rank's shard
            failure = exc
            dev = (torch.device("cuda", torch.cuda.current_device())
                   if _shard_runner is None and torch.cuda.is_available() else torch.device("cpu"))
            costs = torch.full((hi - lo,), _I64_MAX, dtype=torch.int64, device=dev)
            key = torch.full((2,), _I64_MIN, dtype=torch.int64, device=dev)
            perm = torch.zeros(inst.n, dtype=torch.int64, device=dev)

    if collective:
        bits = _index_bits(cfg.n_starts)
        if _packable(inst, cfg.n_starts):
            special = (key[0] == _I64_MAX) | (key[0] == _I64_MIN)  # empty shard / failed rank
            packed = torch.where(special, key[0], (key[0] << bits) | key[1]).reshape(1)
            dist.all_reduce(packed, op=dist.ReduceOp.MIN, group=group)  # the one data-path collective
            reduced = int(packed.item())
            best_cost, best_index = reduced >> bits, reduced & ((1 << bits) - 1)
            failed = reduced == _I64_MIN
        else:  # costs may be negative / huge: two-step lexicographic min
            c = key[0:1].clone()
            dist.all_reduce(c, op=dist.ReduceOp.MIN, group=group)
            failed = int(c.item()) == _I64_MIN  # (a true cost of -2^63 is impossible: |cost| <= n^2 2^60)
            mine = key[1:2] if int(key[0].item()) == int(c.item()) else torch.full_like(key[1:2], _I64_MAX)
            mine = mine.clone()
            dist.all_reduce(mine, op=dist.ReduceOp.MIN, group=group)
            best_cost, best_index = int(c.item()), int(mine.item())
        if failed:
            if failure is not None:
                raise QapError(f"multi-start shard [{lo}, {hi}) failed on rank {rank}: {failure}") from failure
            raise QapError("multi-start failed on another rank; partial results discarded")
        owner = next(r for r in range(world) if shard_bounds(cfg.n_starts, world, r)[0] <= best_index
                     < shard_bounds(cfg.n_starts, world, r)[1])
        src = owner if group is None else dist.get_global_rank(group, owner)
        dist.broadcast(perm, src=src, group=group)
        width = max(shard_bounds(cfg.n_starts, world, r)[1] - shard_bounds(cfg.n_starts, world, r)[0]
                    for r in range(world))
        padded = torch.full((width,), _I64_MAX, dtype=torch.int64, device=costs.device)
        padded[: hi - lo] = costs
        parts = [torch.empty_like(padded) for _ in range(world)]
        dist.all_gather(parts, padded, group=group)
        per_start = np.concatenate([
            parts[r][: shard_bounds(cfg.n_starts, world, r)[1] - shard_bounds(cfg.n_starts, world, r)[0]].cpu().numpy()
            for r in range(world)])
    else:
        base = costs._base
        if base is not None and base is key._base and base is perm._base and base.numel() == hi - lo + 2 + inst.n:
            host = base.cpu()  # [costs | key | perm] in one transfer
            costs, key, perm = host[:hi - lo], host[hi - lo:hi - lo + 2], host[hi - lo + 2:]
        key_h = key.cpu()
        best_cost, best_index = int(key_h[0]), int(key_h[1])
        per_start = costs.cpu().numpy()

    digest = config_digest(inst, cfg)
    best = SolutionRecord(
        instance_name=inst.name,
        permutation=perm.cpu().numpy().astype(np.int64),
        cost=best_cost,
        algorithm=cfg.algorithm,
        seed=derive_seed(cfg.master_seed, best_index),
        config_digest=digest,
    )
    return MultiStartResult(best=best, per_start_costs=per_start.astype(np.int64),
                            wall_time=time.perf_counter() - t0, config_digest=digest,
                            best_start_index=best_index)
