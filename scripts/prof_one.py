"""One short multistart launch for ncu captures (development aid)."""
import sys
sys.path.insert(0, ".")
import paper_2307_11248_b200 as q
from paper_2307_11248_b200 import shapes
from paper_2307_11248_b200.backend import device_instance

shape = sys.argv[1] if len(sys.argv) > 1 else "tai100a"
starts = int(sys.argv[2]) if len(sys.argv) > 2 else 296
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 200
algo = sys.argv[4] if len(sys.argv) > 4 else "tabu"
inst = shapes.by_name(shape)
di = device_instance(inst.flow, inst.distance)
t = q.tenure_bounds(inst.n)
for r in range(2):
    di.multistart(algo, r, 0, starts, iters, t.low, t.high)
    print(di.last_kernel_ms())
