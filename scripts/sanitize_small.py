"""Small runs of every kernel path for compute-sanitizer (memcheck / racecheck)."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2307_11248_b200 as q
from paper_2307_11248_b200 import shapes
from paper_2307_11248_b200.backend import clear_cache

def run(name, starts=3, iters=12):
    inst = shapes.by_name(name)
    res = q.run_multistart(inst, q.SearchConfig(algorithm="tabu", n_starts=starts, iterations=iters, master_seed=1))
    res2 = q.run_multistart(inst, q.SearchConfig(algorithm="2opt", n_starts=starts, iterations=iters, master_seed=1))
    rec, trail = q.run_tabu(inst, 3, iters)
    q.all_deltas(inst, rec.permutation)
    many = q.run_repetitions(inst, q.SearchConfig(algorithm="tabu", n_starts=2, iterations=iters, master_seed=1), 2)
    for algo in ("tabu", "2opt"):  # device RNG + recorded moves (qapb_multistart_trace)
        q.best_costs_at_budgets(inst, q.SearchConfig(algorithm=algo, n_starts=2, iterations=iters, master_seed=1), [3, iters])
    info = q.backend.device_instance(inst.flow, inst.distance).info
    print(name, res.best.cost, res2.best.cost, rec.cost, many[1].best.cost, "storage", info["storage"], "threads", info["threads"], "acc", info["acc_bits"])

# hybrid plans: one register unit (+ staging), asymmetric, two register units (n = 112), two CTAs with
# shared-memory units and diagonal blocks in shared memory (n = 132), one CTA (n = 200)
for name in ("rand12", "tai30a", "rand23", "tai112a", "rand132", "tai200a"):
    run(name)
# exactly one symmetric matrix (hybrid single-product update with combined vectors)
from paper_2307_11248_b200.instance import Instance
_rs = np.random.default_rng(5)
for _n, _which in ((23, "dist"), (40, "flow"), (132, "dist")):
    _f = _rs.integers(0, 60, (_n, _n)).astype(np.int64); _d = _rs.integers(0, 60, (_n, _n)).astype(np.int64)
    if _which == "dist": _d = _d + _d.T
    else: _f = _f + _f.T
    _inst = Instance(f"onesym{_n}{_which}", _n, _f, _d)
    _res = q.run_multistart(_inst, q.SearchConfig(algorithm="tabu", n_starts=3, iterations=12, master_seed=1))
    print(_inst.name, _res.best.cost, q.backend.device_instance(_f, _d).info["threads"])
# every candidate plan of a small and a mid-size instance (paired diagonal blocks, one-warp searches, ...)
from paper_2307_11248_b200.backend import device_instance as _di
for name in ("tai30a", "rand23", "tai100a"):
    inst = shapes.by_name(name)
    d = _di(inst.flow, inst.distance)
    for plan in d.plan_candidates():
        d.set_plan(plan)
        out = d.multistart("tabu", 1, 0, 3, 10, 1, 3)
        print(name, plan, out[1], "threads", d.info["threads"])
    clear_cache()
# tai*b shapes: unsigned 32-bit state with 64-bit deltas on the hybrid plans (n = 45: registers; n = 150: shared-memory units)
run("tai45b")
run("tai150b", starts=2, iters=6)
# generic kernel: int64 state (tai*b forced off the hybrid plans), forced int32, M in L2, masks in L2
os.environ["QAPB_FORCE_GENERIC"] = "1"
clear_cache()
run("tai45b")
run("tai30a")
for st in ("1", "2"):
    os.environ["QAPB_FORCE_STORAGE"] = st
    clear_cache()
    run("rand23")
