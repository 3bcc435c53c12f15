"""Multi-rank sharding / reduction logic of run_multistart on CPU: world_size 2 and 3,
gloo backend.  The per-shard compute is injected (`_shard_runner`) and served by the
oracle here, because no GPU is available; the collective logic (contiguous index
shards, packed all-reduce(min), winner broadcast, per-start-cost all-gather) is the
product code that runs under NCCL on the GPUs.  Mirrors the reference's
worker-count-invariance tests (test_multistart.py:69-92, test_acceptance.py:141-153)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _oracle_runner(inst, cfg, first_index, count):
    import oracle

    n = inst.n
    i64max = np.iinfo(np.int64).max
    if count == 0:
        return (torch.empty(0, dtype=torch.int64), torch.full((2,), i64max, dtype=torch.int64),
                torch.zeros(n, dtype=torch.int64))
    ten = cfg.resolved_tenure(n)
    costs, bc, bi, bp = oracle.multistart(inst.flow, inst.distance, cfg.algorithm, cfg.master_seed, count,
                                          cfg.resolved_iterations(n), (ten.low, ten.high), first_index=first_index)
    return torch.from_numpy(costs), torch.tensor([bc, bi], dtype=torch.int64), torch.from_numpy(bp.copy())


def _cases():
    import paper_2307_11248_b200 as q
    from paper_2307_11248_b200 import shapes

    rs = np.random.default_rng(4)
    neg = q.Instance("neg9", 9, rs.integers(-50, 50, (9, 9)).astype(np.int64), rs.integers(-50, 50, (9, 9)).astype(np.int64))
    flat = q.Instance("flat6", 6, np.ones((6, 6), np.int64) - np.eye(6, dtype=np.int64), np.ones((6, 6), np.int64) - np.eye(6, dtype=np.int64))
    return [
        (shapes.rand(10, 3), q.SearchConfig(algorithm="tabu", n_starts=24, iterations=30, master_seed=5)),
        (shapes.rand(10, 3), q.SearchConfig(algorithm="2opt", n_starts=7, iterations=12, master_seed=1)),
        (neg, q.SearchConfig(algorithm="tabu", n_starts=11, iterations=20, master_seed=2)),   # two-step min path
        (flat, q.SearchConfig(algorithm="tabu", n_starts=5, iterations=4, master_seed=0)),    # all tie -> index 0
        (shapes.rand(5, 1), q.SearchConfig(algorithm="tabu", n_starts=1, iterations=5, master_seed=9)),  # empty shards
    ]


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2307_11248_b200 as q

    try:
        for k, (inst, cfg) in enumerate(_cases()):
            res = q.run_multistart(inst, cfg, _shard_runner=_oracle_runner)
            np.savez(os.path.join(out_dir, f"r{rank}_c{k}.npz"), costs=res.per_start_costs, perm=res.best.permutation,
                     cost=res.best.cost, index=res.best_start_index, seed=res.best.seed, digest=res.config_digest)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_rank_count_invariance(world, tmp_path, built):
    import oracle
    import paper_2307_11248_b200 as q

    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for k, (inst, cfg) in enumerate(_cases()):
        ten = cfg.resolved_tenure(inst.n)
        costs, bc, bi, bp = oracle.multistart(inst.flow, inst.distance, cfg.algorithm, cfg.master_seed, cfg.n_starts,
                                              cfg.resolved_iterations(inst.n), (ten.low, ten.high))
        for rank in range(world):
            got = np.load(os.path.join(tmp_path, f"r{rank}_c{k}.npz"))
            assert np.array_equal(got["costs"], costs), (k, rank)
            assert int(got["cost"]) == bc and int(got["index"]) == bi, (k, rank)
            assert np.array_equal(got["perm"], bp), (k, rank)
            assert int(got["seed"]) == q.derive_seed(cfg.master_seed, bi)
            assert str(got["digest"]) == q.config_digest(inst, cfg)


def test_single_process_path_with_runner(built):
    """world_size 1 (no process group): same result object, tie rule -> lowest index."""
    import oracle
    import paper_2307_11248_b200 as q

    inst, cfg = _cases()[3]
    res = q.run_multistart(inst, cfg, _shard_runner=_oracle_runner)
    assert res.best_start_index == 0 and len(set(res.per_start_costs.tolist())) == 1
    inst, cfg = _cases()[0]
    res = q.run_multistart(inst, cfg, _shard_runner=_oracle_runner)
    costs, bc, bi, _ = oracle.multistart(inst.flow, inst.distance, "tabu", 5, 24, 30)
    assert np.array_equal(res.per_start_costs, costs) and (res.best.cost, res.best_start_index) == (bc, bi)
    assert q.evaluate_cost(inst, res.best.permutation) == res.best.cost


def _failing_worker(rank, world, port, out_dir):
    """Rank 1's shard raises; every rank must come back with QapError instead of hanging in the all-reduce
    (the analogue of the reference's pool-failure rule, multistart.py:151-154)."""
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2307_11248_b200 as q

    def runner(inst, cfg, first_index, count):
        if rank == 1:
            raise RuntimeError("injected shard failure")
        return _oracle_runner(inst, cfg, first_index, count)

    try:
        for k, (inst, cfg) in enumerate(_cases()[:3]):  # packed and two-step reductions
            try:
                q.run_multistart(inst, cfg, _shard_runner=runner)
                outcome = "returned"
            except q.QapError as exc:
                outcome = "QapError: " + str(exc)
            with open(os.path.join(out_dir, f"fail_r{rank}_c{k}.txt"), "w") as fh:
                fh.write(outcome)
    finally:
        dist.destroy_process_group()


def test_rank_failure_raises_on_every_rank(tmp_path, built):
    world = 3
    mp.spawn(_failing_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for k in range(3):
        for rank in range(world):
            text = open(os.path.join(tmp_path, f"fail_r{rank}_c{k}.txt")).read()
            assert text.startswith("QapError"), (k, rank, text)
            assert ("injected shard failure" in text) == (rank == 1)


def _forced_collective_worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), QAPB_FORCE_COLLECTIVE="1")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2307_11248_b200 as q

    try:
        inst, cfg = _cases()[0]
        res = q.run_multistart(inst, cfg, _shard_runner=_oracle_runner)
        np.savez(os.path.join(out_dir, "forced.npz"), costs=res.per_start_costs, cost=res.best.cost, index=res.best_start_index)
    finally:
        dist.destroy_process_group()


def test_one_rank_group_takes_the_collective_path_when_forced(tmp_path, built):
    """QAPB_FORCE_COLLECTIVE=1: a one-rank group runs the all-reduce / broadcast / all-gather branch
    (the -m gpu suite uses this to execute the NCCL branch on a single-GPU box)."""
    import oracle

    mp.spawn(_forced_collective_worker, args=(1, _free_port(), str(tmp_path)), nprocs=1, join=True)
    inst, cfg = _cases()[0]
    costs, bc, bi, _ = oracle.multistart(inst.flow, inst.distance, "tabu", 5, 24, 30)
    got = np.load(os.path.join(tmp_path, "forced.npz"))
    assert np.array_equal(got["costs"], costs) and (int(got["cost"]), int(got["index"])) == (bc, bi)
