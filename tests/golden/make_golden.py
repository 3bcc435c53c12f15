#!/usr/bin/env python
"""Generate golden vectors by running the REFERENCE itself (in the build container).

    python tests/golden/make_golden.py

Imports /root/reference/pkg/src/qapsolve (drivers, RNG, multistart) and plugs in the
reference's own compiled kernel built into oracle/_ref (falls back to the pure
NumPy backend), runs the BASELINE.json configurations at CPU-affordable sizes and
writes tests/golden/golden_*.npz.  The instances come from
paper_2307_11248_b200.shapes (deterministic); their SHA-256 is stored so generator
drift is detected.  Neither the GPU box nor the tests read /root/reference.
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
os.environ.setdefault("QAPSOLVE_BACKEND", "python")
sys.path.insert(0, "/root/reference/pkg/src")

import qapsolve  # noqa: E402  the reference
import qapsolve.backend, qapsolve.core, qapsolve.tabu, qapsolve.two_opt  # noqa: E401,E402

import oracle  # noqa: E402

ref_kernels = oracle.load_ref_kernels()
if ref_kernels is not None:  # use the reference's compiled kernel (same results, much faster)
    for mod in (qapsolve.backend, qapsolve.core, qapsolve.tabu, qapsolve.two_opt):
        mod.kernels = ref_kernels

from paper_2307_11248_b200 import shapes  # noqa: E402


def digest(inst) -> str:
    return hashlib.sha256(inst.flow.tobytes() + inst.distance.tobytes()).hexdigest()


def ref_instance(inst):
    return qapsolve.Instance(inst.name, inst.n, inst.flow.copy(), inst.distance.copy())


def single(shape, algo, seed, iters):
    mine = shapes.by_name(shape)
    inst = ref_instance(mine)
    out = {"shape": shape, "algo": algo, "seed": seed, "iters": iters, "sha256": digest(mine)}
    rng = qapsolve.SplitMix64(seed)
    start = qapsolve.random_permutation(inst.n, rng)
    out["start"] = start
    out["start_cost"] = qapsolve.full_cost(inst, start)
    out["start_deltas"] = qapsolve.all_deltas(inst, start)
    if algo == "tabu":
        rec, trail = qapsolve.run_tabu(inst, seed, iters)
        out.update(best=rec.permutation, best_cost=rec.cost, move_i=trail.move_i, move_j=trail.move_j,
                   delta=trail.delta, tabu_flag=trail.tabu_flag, tenure=trail.tenure_drawn,
                   stopped_early=trail.stopped_early, final_tabu=trail.final_tabu)
    else:
        rec = qapsolve.run_two_opt(inst, seed, iters)
        k = qapsolve.backend.kernels.two_opt_run(inst.flow, inst.distance, start, iters)
        out.update(best=rec.permutation, best_cost=rec.cost, cur=k[2], cur_cost=k[3], move_i=k[4], move_j=k[5], delta=k[6])
    return out


def multi(shape, algo, starts, iters, master):
    mine = shapes.by_name(shape)
    inst = ref_instance(mine)
    res = qapsolve.run_multistart(inst, qapsolve.SearchConfig(algorithm=algo, n_starts=starts, iterations=iters,
                                                               master_seed=master, workers=os.cpu_count()))
    return {"shape": shape, "algo": algo, "starts": starts, "iters": iters, "master": master,
            "sha256": digest(mine), "per_start_costs": res.per_start_costs, "best_cost": res.best.cost,
            "best_index": res.best_start_index, "best_perm": res.best.permutation, "best_seed": res.best.seed,
            "digest": res.config_digest, "instance_name": inst.name}


def save(name, d):
    path = os.path.join(HERE, f"golden_{name}.npz")
    np.savez_compressed(path, **{k: np.asarray(v) for k, v in d.items()})
    print("wrote", path, os.path.getsize(path), "bytes")


def full_length():
    """Full-length single-start runs of the big BASELINE.json configurations (the lengths bench.py
    times): about three minutes of the reference's compiled kernel, one-off."""
    save("full_cfg2_tai100a_tabu", single("tai100a", "tabu", qapsolve.derive_seed(0, 0), 800))
    save("full_cfg4_tai150b_tabu", single("tai150b", "tabu", qapsolve.derive_seed(3, 1), 1200))
    save("full_cfg4_sko100_tabu", single("sko100", "tabu", qapsolve.derive_seed(3, 2), 800))
    save("full_cfg3_tai256c_2opt", single("tai256c", "2opt", 11, 1024))
    save("full_cfg3_tai256c_tabu", single("tai256c", "tabu", 11, 2048))
    # criterion-6 style audit at n >= 150 (test_acceptance.py:157-175): 6 starts x 8n iterations
    save("full_cfg4_tai150b_multi6", multi("tai150b", "tabu", 6, 1200, 7))


if __name__ == "__main__":
    print("reference backend:", qapsolve.backend.kernels.BACKEND_NAME)
    if "--full" in sys.argv:
        full_length()
        sys.exit(0)
    # BASELINE.json configs[0]: 2opt single start, nug12 shape, 4n iterations
    save("cfg0_nug12_2opt", single("nug12", "2opt", 3, 48))
    save("cfg0_nug12_tabu", single("nug12", "tabu", 3, 96))
    # configs[1]: robust tabu, tai30a shape, 1000 iterations, single start
    save("cfg1_tai30a_tabu", single("tai30a", "tabu", qapsolve.derive_seed(0, 0), 1000))
    save("cfg1_rand30_tabu", single("rand30", "tabu", qapsolve.derive_seed(0, 0), 1000))
    # configs[2]: tai100a shape, batched starts (16 of the 1024), 8n iterations
    save("cfg2_tai100a_multi", multi("tai100a", "tabu", 16, 800, 0))
    save("cfg2_tai100a_single", single("tai100a", "tabu", qapsolve.derive_seed(0, 5), 300))
    # configs[3]: tai256c shape, 2opt + tabu (short: the reference is O(n^3) per iteration)
    save("cfg3_tai256c_2opt", single("tai256c", "2opt", 11, 24))
    save("cfg3_tai256c_tabu", single("tai256c", "tabu", 11, 40))
    # configs[4]: sko100 / tai150b multi-start
    save("cfg4_sko100_multi", multi("sko100", "tabu", 16, 200, 3))
    save("cfg4_tai150b_multi", multi("tai150b", "tabu", 8, 100, 3))
    save("cfg4_tai150b_2opt_multi", multi("tai150b", "2opt", 8, 60, 3))
    # reference's own generator, survey KAT
    save("kat30_multi_tabu", multi("rand30", "tabu", 64, 240, 0))
    save("kat30_multi_2opt", multi("rand30", "2opt", 64, 120, 0))
