"""Development check of a single-instantiation build (QAPB_LIB=build/libqapb_dev*.so): multi-start
costs against the C oracle on the shape the preset serves, then device timing."""
import json, sys
sys.path.insert(0, ".")
import numpy as np
import oracle
import paper_2307_11248_b200 as q
from paper_2307_11248_b200 import shapes
from paper_2307_11248_b200.backend import device_instance

shape = sys.argv[1] if len(sys.argv) > 1 else "tai100a"
algo = sys.argv[2] if len(sys.argv) > 2 else "tabu"
starts = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 800
inst = shapes.by_name(shape)
di = device_instance(inst.flow, inst.distance)
t = q.tenure_bounds(inst.n)
chk_starts, chk_iters = 48, 3 * inst.n
got = di.multistart(algo, 5, 0, chk_starts, chk_iters, t.low, t.high)
want = oracle.multistart(inst.flow, inst.distance, algo, 5, chk_starts, chk_iters, threads=oracle.max_threads())
ok = bool(np.array_equal(got[0], want[0])) and got[1] == want[1] and got[2] == want[2] and bool(np.array_equal(got[3], want[3]))
best = None
for r in range(3):
    di.multistart(algo, r, 0, starts, iters, t.low, t.high)
    ms = di.last_kernel_ms(); best = ms if best is None else min(best, ms)
ev = starts * iters * inst.n * (inst.n - 1) // 2
print(json.dumps({"parity": ok, "shape": shape, "algo": algo, "starts": starts, "iters": iters, "ms": round(best, 3),
                  "Gevals_s": round(ev / best / 1e6, 1), "threads": di.info["threads"], "ctas": di.info["ctas_per_sm"],
                  "smem": di.info["smem_bytes"]}))
