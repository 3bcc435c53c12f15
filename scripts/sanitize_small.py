"""Small runs of every kernel path for compute-sanitizer (memcheck / racecheck)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2307_11248_b200 as q
from paper_2307_11248_b200 import shapes
for name in ("rand12", "tai30a", "rand23"):
    inst = shapes.by_name(name)
    res = q.run_multistart(inst, q.SearchConfig(algorithm="tabu", n_starts=4, iterations=40, master_seed=1))
    res2 = q.run_multistart(inst, q.SearchConfig(algorithm="2opt", n_starts=4, iterations=20, master_seed=1))
    rec, trail = q.run_tabu(inst, 3, 30)
    q.all_deltas(inst, rec.permutation)
    print(name, res.best.cost, res2.best.cost, rec.cost)
import os
os.environ["QAPB_FORCE_GENERIC"] = "1"
from paper_2307_11248_b200.backend import clear_cache
clear_cache()
for name in ("rand12", "tai30a"):
    inst = shapes.by_name(name)
    res = q.run_multistart(inst, q.SearchConfig(algorithm="tabu", n_starts=4, iterations=40, master_seed=1))
    print("generic", name, res.best.cost)
