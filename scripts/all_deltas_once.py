import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2307_11248_b200 import shapes, _lib
from paper_2307_11248_b200.backend import device_instance
inst = shapes.by_name("tai100a"); n = inst.n; batch = 1024
di = device_instance(inst.flow, inst.distance)
rs = np.random.default_rng(1)
perms = np.stack([rs.permutation(n) for _ in range(batch)]).astype(np.int64)
pm = torch.from_numpy(perms).cuda(); od = torch.empty((batch, n * (n - 1) // 2), dtype=torch.int64, device="cuda")
for _ in range(3):
    _lib.check(_lib.lib().qapb_all_deltas(di.handle, pm.data_ptr(), batch, od.data_ptr(), None))
torch.cuda.synchronize()
