import sys, json
sys.path.insert(0, ".")
import numpy as np
import paper_2307_11248_b200 as q
from paper_2307_11248_b200.backend import DeviceInstance
rs = np.random.default_rng(3)
for n, which in ((100, "dist"), (100, "flow"), (100, "none"), (160, "dist")):
    f = rs.integers(0, 100, (n, n)).astype(np.int64); d = rs.integers(0, 100, (n, n)).astype(np.int64)
    if which == "dist": d = d + d.T
    if which == "flow": f = f + f.T
    np.fill_diagonal(f, 0); np.fill_diagonal(d, 0)
    di = DeviceInstance(f, d)
    t = q.tenure_bounds(n)
    starts = 148 * 2 * max(1, di.info["ctas_per_sm"])
    best = None
    for r in range(3):
        di.multistart("tabu", r, 0, starts, 400, t.low, t.high)
        ms = di.last_kernel_ms(); best = ms if best is None else min(best, ms)
    print(n, which, "sym" , di.info["symmetric"], "threads", di.info["threads"], round(starts * 400 * n * (n - 1) / 2 / best / 1e6, 1), "G evals/s")
    di.close()
