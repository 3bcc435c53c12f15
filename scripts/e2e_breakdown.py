"""Where the end-to-end time of run_multistart goes beyond the kernels (development aid)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2307_11248_b200 as q
from paper_2307_11248_b200 import shapes
from paper_2307_11248_b200.backend import DeviceInstance, clear_cache, device_instance, _mat
import hashlib
inst = shapes.by_name("tai100a")
cfg = lambda m: q.SearchConfig(algorithm="tabu", n_starts=1024, iterations=800, master_seed=m)
q.run_multistart(inst, cfg(0))
def T(f, reps=20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3
print("hash ms", T(lambda: hashlib.blake2b(_mat(inst.flow).tobytes() + _mat(inst.distance).tobytes(), digest_size=16).digest()))
def create():
    d = DeviceInstance(inst.flow, inst.distance); d.close()
print("create+destroy ms", T(create))
def full_fresh():
    clear_cache(); q.run_multistart(inst, cfg(1))
def full_res():
    q.run_multistart(inst, cfg(1))
print("run_multistart fresh ms", T(full_fresh, 10))
print("run_multistart resident ms", T(full_res, 10))
di = device_instance(inst.flow, inst.distance)
t = q.tenure_bounds(100)
def host_call():
    di.multistart("tabu", 1, 0, 1024, 800, t.low, t.high)
print("di.multistart (host buffers) ms", T(host_call, 10), "kernel ms", di.last_kernel_ms())
