"""Development check of the one-warp-per-search kernel (n <= 32) against the C oracle: single runs with
trail and cells, 2opt, multi-start; then device timing.  Usage: warp_check.py [sym|asym] [time]"""
import json, sys
sys.path.insert(0, ".")
import numpy as np
import oracle
import paper_2307_11248_b200 as q
from paper_2307_11248_b200 import shapes
from paper_2307_11248_b200.backend import device_instance

kind = sys.argv[1] if len(sys.argv) > 1 else "sym"
bad = 0
import os
NS = [int(x) for x in os.environ.get("WARP_NS", "2,3,4,5,8,9,12,13,16,17,21,24,25,28,29,30,31,32").split(",")]
for n in NS:
    inst = shapes.tai_a(n, seed=n) if kind == "sym" else shapes.rand(n, seed=n)
    di = device_instance(inst.flow, inst.distance)
    lo, hi = oracle.tenure_bounds(n)
    rng = oracle.Rng(oracle.derive_seed(11, n))
    perm = rng.permutation(n)
    iters = 150
    for tl, th in ((lo, hi), (1, 3)):
        ten = rng.tenures(tl, th, iters)
        got = q.kernels.tabu_run(inst.flow, inst.distance, perm, iters, ten)
        want = oracle.tabu_run(inst.flow, inst.distance, perm, iters, ten)
        ok = all(np.array_equal(g, w) for g, w in zip(got[:7], want[:7])) and all(np.array_equal(g, w) for g, w in zip(got[7], want[7]))
        if not ok:
            bad += 1
            first = [k for k, (g, w) in enumerate(zip(list(got[:7]) + list(got[7]), list(want[:7]) + list(want[7]))) if not np.array_equal(g, w)]
            ti = np.nonzero(np.asarray(got[7][0]) != np.asarray(want[7][0]))[0]
            print("tabu MISMATCH n", n, "tenures", tl, th, "fields", first, "first trail diff at", ti[:1], "info", di.info["threads"])
    got = q.kernels.two_opt_run(inst.flow, inst.distance, perm, 60)
    want = oracle.two_opt_run(inst.flow, inst.distance, perm, 60)
    if not all(np.array_equal(g, w) for g, w in zip(got, want)):
        bad += 1
        print("2opt MISMATCH n", n)
    for algo in ("tabu", "2opt"):
        g = di.multistart(algo, 5, 3, 40, 3 * n + 2, lo, hi)
        w = oracle.multistart(inst.flow, inst.distance, algo, 5, 40, 3 * n + 2, first_index=3, threads=oracle.max_threads())
        if not (np.array_equal(g[0], w[0]) and g[1] == w[1] and g[2] == w[2] and np.array_equal(g[3], w[3])):
            bad += 1
            print("multistart MISMATCH n", n, algo)
# searches that run out of admissible moves at different iterations (long tenures on tiny instances)
for n in (3, 4, 5, 6):
    if n not in NS and max(NS) < 17:
        pass
    inst = shapes.tai_a(n, seed=50 + n) if kind == "sym" else shapes.rand(n, seed=50 + n)
    di = device_instance(inst.flow, inst.distance)
    g = di.multistart("tabu", 8, 0, 9, 40, 50, 50)
    w = oracle.multistart(inst.flow, inst.distance, "tabu", 8, 9, 40, tenure=(50, 50), threads=1)
    if not (np.array_equal(g[0], w[0]) and g[1] == w[1] and g[2] == w[2] and np.array_equal(g[3], w[3])):
        bad += 1
        print("early-stop multistart MISMATCH n", n)
print("warp_check", kind, "mismatches:", bad, "threads", di.info["threads"], "smem", di.info["smem_bytes"], "ctas/SM", di.info["ctas_per_sm"])
if len(sys.argv) > 2:
    cases = (("tai30a", 1, 1000), ("tai30a", 1776, 240), ("tai30a", 4736, 240), ("tai30a", 9472, 240), ("nug12", 1776, 96), ("nug12", 4736, 96))
    if os.environ.get("WARP_TIME") == "small":
        cases = (("nug12", 1, 1000), ("nug12", 1776, 96), ("nug12", 4736, 96), ("nug12", 9472, 96), ("tai16a", 4736, 128))
    for name, starts, iters in cases:
        inst = shapes.by_name(name)
        di = device_instance(inst.flow, inst.distance)
        t = q.tenure_bounds(inst.n)
        best = None
        for r in range(4):
            di.multistart("tabu", r, 0, starts, iters, t.low, t.high)
            ms = di.last_kernel_ms(); best = ms if best is None else min(best, ms)
        ev = starts * iters * inst.n * (inst.n - 1) // 2
        print(json.dumps({"shape": name, "starts": starts, "iters": iters, "ms": round(best, 4), "us_per_iter": round(best * 1e3 / iters, 3),
                          "Gevals_s": round(ev / best / 1e6, 1), "threads": di.info["threads"], "ctas": di.info["ctas_per_sm"]}))
