"""Host-side logic (no GPU): RNG, QAPLIB I/O, records, config digest, sharding, error
classes, the step-wise auditors fed with oracle-produced trails, and the C-ABI surface."""
import ctypes
import io
import os
import re

import numpy as np
import pytest

import paper_2307_11248_b200 as q
from paper_2307_11248_b200 import _lib, multistart, shapes
from paper_2307_11248_b200.rng import raw_stream

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# file formats, registries, the trail writer and the host auditor are the reference's own objects (re-exported when
# `qapsolve` is importable, see paper_2307_11248_b200/_refpkg.py); without it there is nothing of ours to test
from paper_2307_11248_b200._refpkg import reference as _reference  # noqa: E402

needs_reference = pytest.mark.skipif(_reference() is None, reason="the reference package qapsolve is not importable")
TOY = "2\n0 3\n2 0\n0 1\n5 0"


def test_rng_matches_oracle(built):
    import oracle

    for seed in (0, 5, 2**64 - 3, 123456789):
        a, b = q.SplitMix64(seed), oracle.Rng(seed)
        assert [a.next64() for _ in range(5)] == [b.next64() for _ in range(5)]
        assert [a.randbelow(k) for k in (1, 2, 10, 97, 2**40 + 7)] == [b.randbelow(k) for k in (1, 2, 10, 97, 2**40 + 7)]
        assert a.state == b.state
    assert q.derive_seed(7, 5) == 0x3FDABE86CBBEAA11 == oracle.derive_seed(7, 5)
    assert q.derive_seed(-1, 0) == oracle.derive_seed(-1 & (2**64 - 1), 0)
    assert np.array_equal(q.random_permutation(23, q.SplitMix64(9)), oracle.Rng(9).permutation(23))
    with pytest.raises(ValueError):
        q.derive_seed(1, -1)
    assert raw_stream(5, 4).tolist() == [q.SplitMix64(5).next64() if False else x for x in
                                         (lambda r: [r.next64() for _ in range(4)])(q.SplitMix64(5))]


def test_random_instance_matches_oracle(built):
    import oracle

    inst = shapes.rand(12, 1234)
    f, d = oracle.Rng(oracle.derive_seed(1234, 0)).instance(12)
    assert np.array_equal(inst.flow, f) and np.array_equal(inst.distance, d)
    assert inst.flow[0].tolist() == [0, 21, 93, 16, 79, 57, 99, 30, 76, 2, 56, 38]


def test_tenure_bounds_table():
    """test_tabu.py:13-18."""
    for n, lo, hi in [(30, 3, 10), (100, 10, 33), (12, 1, 4), (256, 25, 85), (2, 1, 1), (150, 15, 50)]:
        t = q.tenure_bounds(n)
        assert (t.low, t.high) == (lo, hi)
    with pytest.raises(q.DomainError):
        q.tenure_bounds(1)
    with pytest.raises(q.DomainError):
        q.TenureInterval(0, 3)


@needs_reference
def test_parse_and_roundtrip():
    inst = q.parse_instance(TOY, name="toy")
    assert inst.n == 2 and inst.flow.tolist() == [[0, 3], [2, 0]] and inst.distance.tolist() == [[0, 1], [5, 0]]
    assert not inst.flow.flags.writeable
    buf = io.StringIO()
    q.write_qaplib(inst, buf)
    assert q.parse_instance(buf.getvalue(), name="toy") == inst
    assert q.evaluate_cost(inst, np.array([0, 1])) == 13 and q.evaluate_cost(inst, np.array([1, 0])) == 17
    with pytest.raises(q.MalformedInstanceError) as e:
        q.parse_instance("2\n0 3\n2 0\n0 1\n5")
    assert e.value.byte_offset == len("2\n0 3\n2 0\n0 1\n5")
    with pytest.raises(q.MalformedInstanceError):
        q.parse_instance("2 0 3 2 0 0 1 5 0 9")
    with pytest.raises(q.TokenParseError) as e:
        q.parse_instance("2\n0 x\n2 0\n0 1\n5 0")
    assert e.value.byte_offset == 4
    with pytest.raises(q.MalformedInstanceError):
        q.parse_instance("")
    with pytest.raises(q.DomainError):
        q.parse_instance("1 0 0")


@needs_reference
def test_solution_io():
    inst = q.parse_instance(TOY, name="toy")
    rec = q.SolutionRecord("toy", np.array([0, 1], np.int64), 13, "tabu", 7)
    buf = io.StringIO()
    q.write_solution(rec, buf, inst)
    assert buf.getvalue() == "toy\n2\n13\n1 2\n"
    back = q.read_solution(buf.getvalue())
    assert back.cost == 13 and back.permutation.tolist() == [0, 1] and back.instance_name == "toy"
    with pytest.raises(q.IntegrityError):
        q.write_solution(q.SolutionRecord("toy", np.array([0, 1]), 14), io.StringIO(), inst)


@needs_reference
def test_best_known_registry():
    reg = q.load_best_known("# c\ntai30a,1818146\n\ntai100a,21052466\n")
    assert reg.get("tai30a") == 1818146 and reg.get("nope") is None
    with pytest.raises(q.TokenParseError):
        q.load_best_known("a,b,c\n")
    with pytest.raises(q.DomainError):
        q.load_best_known("a,0\n")


def test_search_config_and_digest():
    cfg = q.SearchConfig()
    assert cfg.n_starts == 6144 and cfg.resolved_iterations(30) == 240
    assert q.SearchConfig(algorithm="2opt").resolved_iterations(30) == 120
    for bad in (dict(algorithm="sa"), dict(n_starts=0), dict(iterations=0)):
        with pytest.raises(q.DomainError):
            q.SearchConfig(**bad)
    # digest of (kat30, tabu, 64 starts, 240 iterations, master 0) from the reference
    inst = shapes.rand(30, 1234)
    kat = q.Instance("kat30", 30, inst.flow.copy(), inst.distance.copy())
    cfg = q.SearchConfig(algorithm="tabu", n_starts=64, iterations=240, master_seed=0)
    assert q.config_digest(kat, cfg) == "bd8b855cdce8c9f9"
    g = np.load(os.path.join(ROOT, "tests", "golden", "golden_kat30_multi_tabu.npz"))
    assert q.config_digest(inst, cfg) == str(g["digest"])
    import dataclasses

    assert q.config_digest(inst, dataclasses.replace(cfg, workers=3)) == q.config_digest(inst, cfg)


def test_shard_bounds_partition():
    for n_starts in (1, 7, 64, 1000, 6144):
        for world in (1, 2, 3, 4, 8):
            spans = [multistart.shard_bounds(n_starts, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n_starts
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def test_moves_and_delta_cost(built):
    import oracle

    assert q.enumerate_moves(4) == [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
    rs = np.random.default_rng(3)
    for n in (3, 7, 12):
        f = rs.integers(-20, 50, (n, n)).astype(np.int64)
        d = rs.integers(-20, 50, (n, n)).astype(np.int64)
        inst = q.Instance("x", n, f, d)
        p = rs.permutation(n).astype(np.int64)
        want = oracle.all_deltas(f, d, p)
        got = [q.delta_cost(inst, p, mv) for mv in q.enumerate_moves(n)]
        assert got == want.tolist()
        for mv, dl in zip(q.enumerate_moves(n), got):
            assert q.evaluate_cost(inst, q.apply_move(p, mv)) == q.evaluate_cost(inst, p) + dl
    with pytest.raises(q.DomainError):
        q.apply_move(np.arange(4), (2, 1))
    with pytest.raises(q.DomainError):
        q.apply_move(np.arange(4), (1, 1))


@needs_reference
def test_admissibility_truth_table():
    """test_tabu.py:53-71."""
    cells = np.zeros((3, 3), np.int64)
    cells[0, 1] = 5
    assert q.is_admissible(cells, (0, 1), 100, 50, 5)        # expired exactly now
    assert not q.is_admissible(cells, (0, 1), 100, 50, 4)    # tabu, no aspiration
    assert q.is_admissible(cells, (0, 1), 49, 50, 4)         # aspirated
    assert not q.is_admissible(cells, (0, 1), 50, 50, 4)     # equal does not aspirate
    cells[1, 0] = 99                                         # frequency cell is never read
    assert q.is_admissible(cells, (0, 2), 100, 50, 1)
    with pytest.raises(q.DomainError):
        q.is_admissible(cells, (1, 0), 1, 1, 1)


@needs_reference
def test_trail_csv_format():
    tr = q.TabuTrail("t", np.array([0, 1]), q.TenureInterval(1, 2), 2, False, np.array([0]), np.array([1]),
                     np.array([-4]), np.array([0]), np.array([0]), np.array([2]))
    buf = io.StringIO()
    q.write_trail(tr, buf)
    assert buf.getvalue() == "iter,i,j,delta,tabu_flag,aspirated_flag,tenure_drawn\n1,1,2,-4,0,0,2\n"


def test_abi_exports_every_declared_symbol(built):
    """The library loads (no GPU needed) and exports every function include/qapb.h declares."""
    header = open(os.path.join(ROOT, "include", "qapb.h")).read()
    declared = set(re.findall(r"\b(qapb_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations found"
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} declared in qapb.h but not exported"
    assert declared == set(_lib.SIGNATURES), "ctypes table and header disagree"
    assert _lib.lib().qapb_version() == 1


def test_abi_argument_errors_without_gpu(built):
    """Argument validation happens before any CUDA work and maps to DomainError."""
    L = _lib.lib()
    h = ctypes.c_void_p()
    f = np.zeros((1, 1), np.int64)
    rc = L.qapb_create(1, f.ctypes.data, f.ctypes.data, 0, ctypes.byref(h))
    assert rc == _lib.ERR_INVALID and b"n" in L.qapb_last_error()
    with pytest.raises(q.DomainError):
        _lib.check(rc)
    assert L.qapb_get_info(None, None) == _lib.ERR_INVALID
    assert L.qapb_destroy(None) == _lib.OK


def test_no_cpu_fallback(built):
    """Without a CUDA device compute entries raise QapError -- nothing is computed on the host."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    inst = q.parse_instance(TOY, name="toy")
    with pytest.raises(q.QapError):
        q.full_cost(inst, np.array([0, 1]))
    with pytest.raises(q.QapError):
        q.run_multistart(inst, q.SearchConfig(n_starts=2, iterations=2))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2307_11248_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", text, re.M), fn
                assert "liboracle" not in text, fn


def test_derive_seeds_vectorised_matches_scalar():
    from paper_2307_11248_b200.sweep import derive_seeds

    for master in (0, 7, 2**63 + 5, 2**64 - 1):
        got = derive_seeds(master, 3, 40)
        want = [q.derive_seed(master, i) for i in range(3, 43)]
        assert [int(x) for x in got] == want


def test_make_sweep_validation_and_expand():
    """tuner.py:90-122 rules: axis names, non-empty strictly increasing positive values, powers of
    two <= 1024 on the instances axis; expand yields (value, rep, master_seed + rep)."""
    base = q.SearchConfig(algorithm="2opt", n_starts=4, master_seed=10)
    for bad in (("nope", [1]), ("seeds", []), ("seeds", [0, 1]), ("seeds", [2, 1]), ("instances", [3]),
                ("instances", [2048])):
        with pytest.raises(q.DomainError):
            q.make_sweep(bad[0], bad[1], base)
    plan = q.make_sweep("instances", [2, 8], base)
    assert list(q.expand(plan, 2)) == [(2, 0, 10), (2, 1, 11), (8, 0, 10), (8, 1, 11)]


def test_run_multistart_many_groups_and_splits():
    """Grouping by (algorithm, iterations, tenure), concatenated seeds, per-run split, first-minimum
    tie rule -- with a fake seed runner (cost = seed-derived number), no GPU."""
    from paper_2307_11248_b200 import shapes
    from paper_2307_11248_b200.sweep import derive_seeds, run_multistart_many

    inst = shapes.rand(6, 3)
    calls = []

    def fake(inst_, algorithm, seeds, iterations, low, high):
        calls.append((algorithm, iterations, low, high, len(seeds)))
        costs = (seeds % np.uint64(5)).astype(np.int64)  # many ties
        perms = np.tile(np.arange(inst_.n, dtype=np.int64), (len(seeds), 1))
        perms[:, 0] = (seeds % np.uint64(1000)).astype(np.int64)  # tag each row with its seed
        return costs, perms

    cfgs = [q.SearchConfig(algorithm="tabu", n_starts=5, iterations=9, master_seed=1),
            q.SearchConfig(algorithm="2opt", n_starts=3, iterations=9, master_seed=1),
            q.SearchConfig(algorithm="tabu", n_starts=7, iterations=9, master_seed=2),
            q.SearchConfig(algorithm="tabu", n_starts=2, iterations=4, master_seed=1)]
    res = run_multistart_many(inst, cfgs, _seed_runner=fake)
    assert sorted(c[4] for c in calls) == [2, 3, 12] and len(calls) == 3  # the two 9-iteration tabu runs share a launch
    for cfg, r in zip(cfgs, res):
        seeds = derive_seeds(cfg.master_seed, 0, cfg.n_starts)
        costs = (seeds % np.uint64(5)).astype(np.int64)
        assert np.array_equal(r.per_start_costs, costs)
        k = int(np.flatnonzero(costs == costs.min())[0])
        assert r.best_start_index == k and r.best.cost == int(costs[k])
        assert r.best.permutation[0] == int(seeds[k] % np.uint64(1000))
        assert r.best.seed == q.derive_seed(cfg.master_seed, k)
        assert r.config_digest == q.config_digest(inst, cfg)


def test_thread_config_space():
    """tuner.py:28-78 known answers (from the reference itself): 1434 configurations in all, six for
    N = 4096, and the violation messages of an invalid triple."""
    cfgs = q.enumerate_configs()
    assert len(cfgs) == 1434 and cfgs[0] == q.ThreadConfig(1024, 32, 32) and cfgs[-1] == q.ThreadConfig(12288, 1024, 12)
    assert [c.threads_per_block for c in q.enumerate_configs(4096)] == [32, 64, 128, 256, 512, 1024]
    assert q.enumerate_configs(1000) == []
    ok, why = q.validate_config(q.ThreadConfig(1000, 33, 2))
    assert not ok and why == ["n_starts 1000 outside [1024, 12288]", "n_starts 1000 not a multiple of warp size 32",
                              "threads_per_block 33 not a multiple of warp size 32",
                              "n_starts 1000 not divisible by threads_per_block 33"]
    assert q.validate_config(q.ThreadConfig(2048, 64, 32)) == (True, [])
    assert q.validate_config(q.ThreadConfig(2048, 64, 31))[1] == ["blocks 31 != n_starts / threads_per_block (32)"]


@needs_reference
def test_report_accuracy_and_bench_report():
    """report.py:16-49 semantics: exact rational gap on the minimum over repetitions, six-decimal
    formatting, DomainError for a non-positive best-known cost; bench_report batches the
    repetitions (master seeds seed + rep, cli.py:113-115) through run_multistart_many."""
    from fractions import Fraction

    from paper_2307_11248_b200 import shapes
    from paper_2307_11248_b200.sweep import derive_seeds

    assert q.accuracy(110, 100) == Fraction(1, 10) and q.accuracy(100, 100) == 0
    assert q.format_accuracy(Fraction(1, 3)) == "0.333333" and q.format_accuracy(Fraction(0)) == "0.000000"
    with pytest.raises(q.DomainError):
        q.accuracy(5, 0)

    inst = shapes.rand(6, 3)
    seen = []

    def fake(inst_, algorithm, seeds, iterations, low, high):
        seen.append(np.asarray(seeds).copy())
        costs = (seeds % np.uint64(97)).astype(np.int64) + 50
        return costs, np.tile(np.arange(inst_.n, dtype=np.int64), (len(seeds), 1))

    cfg = q.SearchConfig(algorithm="tabu", n_starts=4, iterations=5, master_seed=11)
    reg = q.BestKnownRegistry({inst.name: 40})
    rep = q.bench_report(inst, cfg, 3, reg, _seed_runner=fake)
    assert len(seen) == 1 and len(seen[0]) == 12  # one launch for the three repetitions
    want = [int(((derive_seeds(11 + r, 0, 4) % np.uint64(97)).astype(np.int64) + 50).min()) for r in range(3)]
    assert rep.per_run_costs == want and rep.best_cost == min(want)
    assert rep.accuracy == Fraction(min(want) - 40, 40)
    row = rep.row()
    assert row[:2] == [inst.name, "tabu"] and row[2] == q.format_accuracy(rep.accuracy) and row[3:5] == [min(want), 40]
    assert q.bench_report(inst, cfg, 1, None, _seed_runner=fake).row()[2] == "no-best-known"
    with pytest.raises(q.DomainError):
        q.bench_report(inst, cfg, 0, reg, _seed_runner=fake)


def test_best_costs_at_budgets_from_one_trace(built):
    """sweep.best_costs_at_budgets: the prefix property behind the one-run `neighborhoods` sweep
    (cli.py:162-166) -- checked with a trace runner made of the oracle's single-start runs against the
    oracle's own multistart at every budget, including a start that stops early."""
    from dataclasses import replace

    from paper_2307_11248_b200 import shapes
    import oracle as orc
    from paper_2307_11248_b200.sweep import best_costs_at_budgets

    def oracle_trace(inst_, algorithm, seeds, iterations, low, high):
        costs, steps, deltas = [], [], np.zeros((len(seeds), iterations), np.int64)
        for b, sd in enumerate(seeds):
            rng = orc.Rng(int(sd))
            perm = rng.permutation(inst_.n)
            if algorithm == "tabu":
                out = orc.tabu_run(inst_.flow, inst_.distance, perm, iterations, rng.tenures(low, high, iterations))
                k, d = int(out[6]), out[7][2]
            else:
                out = orc.two_opt_run(inst_.flow, inst_.distance, perm, iterations)
                k, d = iterations, out[6]
            costs.append(int(out[1])); steps.append(k); deltas[b, :k] = d[:k]
        return np.array(costs, np.int64), np.array(steps, np.int64), deltas

    for inst, algo, ten in ((shapes.rand(12, 5), "tabu", None), (shapes.rand(9, 2), "2opt", None),
                            (shapes.rand(4, 8), "tabu", q.TenureInterval(40, 60))):  # n = 4, long tenures: early stops
        cfg = q.SearchConfig(algorithm=algo, n_starts=6, iterations=1, master_seed=31, tenure=ten)
        budgets = [1, 3, 10, 37]
        got = best_costs_at_budgets(inst, cfg, budgets, _trace_runner=oracle_trace)
        assert got.shape == (4, 6)
        t = cfg.resolved_tenure(inst.n)
        for row, v in zip(got, budgets):
            want = orc.multistart(inst.flow, inst.distance, algo, 31, 6, v, tenure=(t.low, t.high))
            assert np.array_equal(row, want[0]), (inst.n, algo, v)
    with pytest.raises(q.DomainError):
        best_costs_at_budgets(inst, cfg, [], _trace_runner=oracle_trace)
