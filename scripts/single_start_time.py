"""Device time of one explicit-tenure tabu run / one 2opt run (the solver entry points' single-start path)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2307_11248_b200 as q
from paper_2307_11248_b200 import shapes
from paper_2307_11248_b200.backend import device_instance
for name, iters in (("nug12", 48), ("tai30a", 1000), ("tai64c", 512), ("tai100a", 800), ("tai256c", 2048)):
    inst = shapes.by_name(name)
    di = device_instance(inst.flow, inst.distance)
    rng = q.SplitMix64(3)
    perm = q.random_permutation(inst.n, rng)
    t = q.tenure_bounds(inst.n)
    ten = np.array([rng.randint(t.low, t.high) for _ in range(iters)], np.int64)
    best = {}
    for rep in range(5):
        di.tabu(perm, iters, ten)
        best["tabu"] = min(best.get("tabu", 1e9), di.last_kernel_ms())
        di.tabu(perm, iters, ten, cells=False, trail=False)
        best["tabu-norec"] = min(best.get("tabu-norec", 1e9), di.last_kernel_ms())
        di.two_opt(perm, iters)
        best["2opt"] = min(best.get("2opt", 1e9), di.last_kernel_ms())
    print(name, iters, " ".join(f"{k} {v*1e3:.1f} us ({v*1e3/iters:.2f} us/iter)" for k, v in best.items()))
