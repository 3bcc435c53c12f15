"""all_deltas (kernels.all_deltas batched) timing + check against the oracle (development aid)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import oracle
from paper_2307_11248_b200 import shapes, _lib
from paper_2307_11248_b200.backend import device_instance
for name, batch in (("tai100a", 1024), ("rand100", 1024), ("tai64c", 1024), ("nug12", 1024), ("tai30a", 1024), ("rand30", 64)):
    inst = shapes.by_name(name); n = inst.n
    di = device_instance(inst.flow, inst.distance)
    rs = np.random.default_rng(1)
    perms = np.stack([rs.permutation(n) for _ in range(batch)]).astype(np.int64)
    got = di.all_deltas(perms[:8])
    ok = all(np.array_equal(got[k], oracle.all_deltas(inst.flow, inst.distance, perms[k])) for k in range(8))
    pm = torch.from_numpy(perms).cuda(); od = torch.empty((batch, n * (n - 1) // 2), dtype=torch.int64, device="cuda")
    best = None
    for _ in range(5):
        _lib.check(_lib.lib().qapb_all_deltas(di.handle, pm.data_ptr(), batch, od.data_ptr(), None))
        ms = di.last_kernel_ms(); best = ms if best is None else min(best, ms)
    print(name, "parity", ok, "ms", round(best, 4), "G evals/s", round(batch * n * (n - 1) / 2 / best / 1e6, 2))
