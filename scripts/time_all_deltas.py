"""Device time of the full evaluator (start + build + emit) for a batch of permutations (development aid)."""
import sys, json
sys.path.insert(0, ".")
import numpy as np
from paper_2307_11248_b200 import shapes
from paper_2307_11248_b200.backend import device_instance
for name in sys.argv[1:]:
    inst = shapes.by_name(name)
    di = device_instance(inst.flow, inst.distance)
    rs = np.random.default_rng(0)
    perms = np.stack([rs.permutation(inst.n) for _ in range(1024)]).astype(np.int64)
    best = None
    for _ in range(3):
        di.all_deltas(perms)
        ms = di.last_kernel_ms(); best = ms if best is None else min(best, ms)
    print(json.dumps({"shape": name, "batch": 1024, "ms": round(best, 4), "Gevals_s": round(1024 * inst.n * (inst.n - 1) / 2 / best / 1e6, 2)}))
