"""Accuracy of a batch of repetitions against a best-known cost.

Mirrors /root/reference/pkg/src/qapsolve/report.py:16-49: accuracy is the exact rational
(best cost over the repetitions - best known) / best known, taken on the MINIMUM over the
repetitions, and `bench_report` is the per-instance row of the reference's bench command
(cli.py:109-118) with its repetitions batched into one launch by `sweep.run_repetitions`.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from fractions import Fraction

from .errors import DomainError
from .instance import BestKnownRegistry, Instance
from .multistart import SearchConfig, config_digest


def accuracy(best_cost_from_runs: int, best_known: int) -> Fraction:
    """Exact gap to the best-known cost; 0 means it was matched (report.py:16-19)."""
    if best_known <= 0:
        raise DomainError(f"best_known must be positive, got {best_known}")
    return Fraction(int(best_cost_from_runs) - int(best_known), int(best_known))


def format_accuracy(value: Fraction) -> str:
    return f"{float(value):.6f}"


@dataclass
class RunReport:
    instance_name: str
    algorithm: str                       # "2opt" | "tabu"
    best_cost: int                       # minimum over the repetitions
    best_known: int | None               # registry entry, None if the instance has none
    per_run_costs: list[int] = field(default_factory=list)   # one per repetition (master_seed + rep)
    wall_times: list[float] = field(default_factory=list)    # one entry: the repetitions ran as one launch
    config_digest: str = ""              # digest of the base configuration (repetition 0)

    @property
    def accuracy(self) -> Fraction | None:
        if self.best_known is None:
            return None
        return accuracy(min(self.per_run_costs), self.best_known)

    def row(self) -> list:
        """[problem, algorithm, accuracy, best_cost, best_known, time_s] (cli.py:118,134)."""
        acc = self.accuracy
        return [self.instance_name, self.algorithm,
                format_accuracy(acc) if acc is not None else "no-best-known",
                self.best_cost, self.best_known if self.best_known else "", f"{sum(self.wall_times):.3f}"]


def bench_report(inst: Instance, cfg: SearchConfig, repetitions: int,
                 registry: BestKnownRegistry | None = None, *, _seed_runner=None) -> RunReport:
    """`repetitions` multi-start runs with master seeds `cfg.master_seed + rep` (cli.py:113-115),
    executed as one batched launch, summarised the way the reference's bench rows are."""
    from .sweep import run_multistart_many

    if repetitions < 1:
        raise DomainError(f"repetitions must be >= 1, got {repetitions}")
    from dataclasses import replace

    t0 = time.perf_counter()
    runs = run_multistart_many(inst, [replace(cfg, master_seed=cfg.master_seed + rep) for rep in range(repetitions)],
                               _seed_runner=_seed_runner)
    elapsed = time.perf_counter() - t0
    costs = [int(r.best.cost) for r in runs]
    known = registry.get(inst.name) if registry is not None else None
    return RunReport(instance_name=inst.name, algorithm=cfg.algorithm, best_cost=min(costs), best_known=known,
                     per_run_costs=costs, wall_times=[elapsed], config_digest=config_digest(inst, cfg))
