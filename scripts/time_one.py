import sys, json
sys.path.insert(0, ".")
import paper_2307_11248_b200 as q
from paper_2307_11248_b200 import shapes
from paper_2307_11248_b200.backend import device_instance
shape, algo, starts, iters = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
inst = shapes.by_name(shape)
di = device_instance(inst.flow, inst.distance)
t = q.tenure_bounds(inst.n)
best = None
for r in range(3):
    di.multistart(algo, r, 0, starts, iters, t.low, t.high)
    ms = di.last_kernel_ms(); best = ms if best is None else min(best, ms)
ev = starts * iters * inst.n * (inst.n - 1) // 2
print(json.dumps({"shape": shape, "algo": algo, "starts": starts, "iters": iters, "ms": round(best, 3), "Gevals_s": round(ev / best / 1e6, 1),
                  "threads": di.info["threads"], "upt": di.info["units_per_thread"], "storage": di.info["storage"], "ctas": di.info["ctas_per_sm"], "acc": di.info["acc_bits"]}))
