"""Quick device timing of the multistart kernel (development aid)."""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
import __graft_entry__ as e
import paper_2307_11248_b200 as q
from paper_2307_11248_b200 import shapes
from paper_2307_11248_b200.backend import device_instance

def run(shape, algo, starts, iters, reps=3):
    inst = shapes.by_name(shape)
    di = device_instance(inst.flow, inst.distance)
    lo, hi = q.tenure_bounds(inst.n).low, q.tenure_bounds(inst.n).high
    best = None
    for r in range(reps):
        di.multistart(algo, r, 0, starts, iters, lo, hi)
        ms = di.last_kernel_ms()
        best = ms if best is None else min(best, ms)
    evals = starts * iters * inst.n * (inst.n - 1) // 2
    print(json.dumps({"shape": shape, "algo": algo, "starts": starts, "iters": iters, "ms": round(best, 3),
                      "Gevals_s": round(evals / best / 1e6, 2), "info": di.info}))

if __name__ == "__main__":
    run("tai30a", "tabu", 1, 1000)
    run("tai30a", "tabu", 1024, 1000)
    run("tai100a", "tabu", 148, 800)
    run("tai100a", "tabu", 296, 800)
    run("tai100a", "tabu", 1024, 800)
    run("tai100a", "2opt", 1024, 400)
    run("sko100", "tabu", 1024, 800)
    run("tai150b", "tabu", 148, 400)
    run("tai256c", "tabu", 148, 256)
