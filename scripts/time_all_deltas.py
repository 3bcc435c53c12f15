import sys, json, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2307_11248_b200 as q
from paper_2307_11248_b200 import shapes, _lib
from paper_2307_11248_b200.backend import device_instance
for shape, B in (("tai100a", 1024), ("tai256c", 148), ("rand100", 1024), ("tai30a", 4096)):
    inst = shapes.by_name(shape); n = inst.n
    di = device_instance(inst.flow, inst.distance)
    perms = torch.stack([torch.randperm(n) for _ in range(B)]).to(torch.int64).cuda()
    out = torch.empty((B, n * (n - 1) // 2), dtype=torch.int64, device="cuda")
    best = None
    for r in range(4):
        _lib.check(_lib.lib().qapb_all_deltas(di.handle, perms.data_ptr(), B, out.data_ptr(), None))
        ms = di.last_kernel_ms(); best = ms if best is None else min(best, ms)
    ev = B * n * (n - 1) // 2
    kterms = ev * (n - 2)
    print(json.dumps({"shape": shape, "batch": B, "ms": round(best, 3), "Gevals_s": round(ev / best / 1e6, 2), "Tkterms_s": round(kterms / best / 1e9, 3)}))
