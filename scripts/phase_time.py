"""Per-phase cycle counters of CTA 0 of the hybrid search kernel (development aid).

Needs a library built with the counters compiled in:
    NVCC_EXTRA=-DQAPB_PHASE_TIMING QAPB_FORCE_BUILD=1 python -c "import __graft_entry__ as g; g.build()"
(the production build leaves them out: they cost ~6 % of the search loop)."""
import ctypes, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2307_11248_b200 as q
from paper_2307_11248_b200 import shapes, _lib
from paper_2307_11248_b200.backend import device_instance
shape = sys.argv[1] if len(sys.argv) > 1 else "tai100a"
starts = int(sys.argv[2]) if len(sys.argv) > 2 else 296
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 400
algo = sys.argv[4] if len(sys.argv) > 4 else "tabu"
inst = shapes.by_name(shape)
di = device_instance(inst.flow, inst.distance)
t = q.tenure_bounds(inst.n)
L = _lib.lib()
L.qapb_debug_phase_cycles.argtypes = [ctypes.c_void_p]
buf = np.zeros(18, np.int64)
di.multistart(algo, 0, 0, starts, iters, t.low, t.high)
L.qapb_debug_phase_cycles(buf.ctypes.data)   # enable
di.multistart(algo, 1, 0, starts, iters, t.low, t.high)
ms = di.last_kernel_ms()
L.qapb_debug_phase_cycles(buf.ctypes.data)   # read
names = ["pass", "reduce+bar1+book", "vector", "winner", "publish+expire", "bar2"]
print(f"{shape} starts={starts} iters={iters} {algo}: {ms:.3f} ms  ({ms*1e3/iters:.2f} us/iter)")
for slot, who in enumerate(["thread0 (owner+vector)", "thread128 (owner)", "diag lane0"]):
    v = buf[slot*6:(slot+1)*6] / iters
    print(f"  {who:24s} " + "  ".join(f"{n}={x:6.0f}" for n, x in zip(names, v)) + f"   total={v.sum():.0f} clk/iter")
