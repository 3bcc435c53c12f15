"""The NCCL branch of run_multistart on real hardware.

A single-GPU box can still execute it: a one-rank NCCL group with QAPB_FORCE_COLLECTIVE=1 runs the packed
all-reduce(min), the winner broadcast and the per-start-cost all-gather through NCCL kernels.  With two or
more GPUs the 1-vs-N invariance of the reference (test_acceptance.py:141-153: identical best permutation,
cost, per_start_costs and digest for every worker count) is checked with real ranks."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_RANK_SCRIPT = r"""
import json, os, sys
sys.path.insert(0, os.environ["QAPB_ROOT"])
import numpy as np, torch, torch.distributed as dist
import paper_2307_11248_b200 as q
from paper_2307_11248_b200 import shapes
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
out = {}
for name, algo, starts, iters in (("rand30", "tabu", 37, 120), ("tai100a", "tabu", 24, 100), ("tai150b", "tabu", 5, 40),
                                  ("nug12", "2opt", 9, 30)):
    inst = shapes.by_name(name)
    res = q.run_multistart(inst, q.SearchConfig(algorithm=algo, n_starts=starts, iterations=iters, master_seed=11))
    out[name] = {"costs": res.per_start_costs.tolist(), "cost": int(res.best.cost), "index": int(res.best_start_index),
                 "perm": res.best.permutation.tolist(), "digest": res.config_digest, "seed": int(res.best.seed)}
if dist.get_rank() == 0:
    print("RESULT " + json.dumps({"world": dist.get_world_size(), "backend": dist.get_backend(), "out": out}))
dist.barrier()
dist.destroy_process_group()
"""


def _run(world: int, extra_env=None):
    env = dict(os.environ, QAPB_ROOT=ROOT, **(extra_env or {}))
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        env.pop(k, None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 2000 + world), "-c", _RANK_SCRIPT]
    # torch.distributed.run has no -c: go through a temp file
    import tempfile

    with tempfile.NamedTemporaryFile("w", suffix=".py", delete=False) as fh:
        fh.write(_RANK_SCRIPT)
        path = fh.name
    cmd = cmd[:-2] + [path]
    try:
        proc = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    finally:
        os.unlink(path)
    assert proc.returncode == 0, proc.stderr[-3000:]
    line = next(ln for ln in proc.stdout.splitlines() if ln.startswith("RESULT "))
    return json.loads(line[len("RESULT "):])


def _single_process_results():
    import paper_2307_11248_b200 as q
    from paper_2307_11248_b200 import shapes

    out = {}
    for name, algo, starts, iters in (("rand30", "tabu", 37, 120), ("tai100a", "tabu", 24, 100), ("tai150b", "tabu", 5, 40),
                                      ("nug12", "2opt", 9, 30)):
        inst = shapes.by_name(name)
        res = q.run_multistart(inst, q.SearchConfig(algorithm=algo, n_starts=starts, iterations=iters, master_seed=11))
        out[name] = {"costs": res.per_start_costs.tolist(), "cost": int(res.best.cost), "index": int(res.best_start_index),
                     "perm": res.best.permutation.tolist(), "digest": res.config_digest, "seed": int(res.best.seed)}
    return out


def test_one_rank_nccl_group_runs_the_collective_branch(built):
    got = _run(1, {"QAPB_FORCE_COLLECTIVE": "1"})
    assert got["world"] == 1 and got["backend"] == "nccl"
    assert got["out"] == _single_process_results()


def test_rank_count_invariance_on_gpus(built):
    import torch

    have = torch.cuda.device_count()
    if have < 2:
        pytest.skip(f"needs >= 2 GPUs, {have} visible")
    want = _single_process_results()
    for world in sorted({2, min(have, 4), min(have, 8)}):
        got = _run(world)
        assert got["world"] == world and got["backend"] == "nccl"
        assert got["out"] == want, world


def test_bench_under_torchrun_one_rank(built):
    """bench.py as the driver launches it for N ranks (here N = 1): NCCL group, all-reduce inside the timed
    step, the configs[4] section, one JSON line."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1", "--master-addr", "127.0.0.1",
           "--master-port", str(31500 + os.getpid() % 2000), os.path.join(ROOT, "bench.py"), "--gpus", "1", "--steps", "2",
           "--warmup", "3", "--no-cpu-baseline", "--no-time-to-gap", "--no-shapes"]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert proc.returncode == 0, proc.stderr[-3000:]
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["value"] > 1e11 and d["result_check"] is True
    assert d["config"]["steps_done_per_step"] == 1024 * 800
    assert 0 < d["roofline"]["frac"] < 1 and 0 < d["roofline"]["smem"]["frac"] < 1
    mg = d["multi_gpu"]
    assert mg["world"] == 1 and mg["allreduce_min_8B_us"] > 0
    assert {(r["shape"], r["scaling"]) for r in mg["runs"]} == {("sko100", "weak"), ("sko100", "strong"),
                                                               ("tai150b", "weak"), ("tai150b", "strong")}
    assert all(r["evals_per_s"] > 1e10 for r in mg["runs"])
