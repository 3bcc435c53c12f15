"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit-exact.

Modelled on the reference's backend-equivalence suite
(/root/reference/pkg/tests/test_backends.py:24-71): every returned array of
full_cost / all_deltas / two_opt_run / tabu_run is compared element for element,
on the reference's own generator (`random_instance`) and on the QAPLIB-shaped
synthetic instances of BASELINE.json.  Sizes are chosen so the oracle finishes in
seconds; full-size runs are covered by size-independent properties in
test_properties_gpu.py.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q(built):
    import paper_2307_11248_b200 as pkg

    return pkg


@pytest.fixture(scope="module")
def orc(built):
    import oracle

    return oracle


def _fuzz_instance(n, seed, symmetric=False, diag=True, lo=-40, hi=90):
    rng = np.random.default_rng(seed)
    f = rng.integers(lo, hi, (n, n)).astype(np.int64)
    d = rng.integers(lo, hi, (n, n)).astype(np.int64)
    if symmetric:
        f, d = f + f.T, d + d.T
    if not diag:
        np.fill_diagonal(f, 0)
        np.fill_diagonal(d, 0)
    return f, d


def _cases():
    from paper_2307_11248_b200 import shapes

    out = []
    for n in (2, 3, 5, 12, 23, 30):
        inst = shapes.rand(n, 1000 + n)
        out.append((f"rand{n}", inst.flow, inst.distance))
    for n in (4, 5, 12, 23, 30):
        out.append((f"fuzz-asym-diag{n}",) + _fuzz_instance(n, n))
        out.append((f"fuzz-sym-diag{n}",) + _fuzz_instance(n, 100 + n, symmetric=True))
    for name in ("nug12", "tai30a", "sko49", "tai64c"):
        inst = shapes.by_name(name)
        out.append((name, inst.flow, inst.distance))
    # kernel-plan coverage: |delta| >= 2^27 (unpacked argmin keys), entries > 32767 (no int16 staging),
    # both symmetric and asymmetric
    out.append(("fuzz-unpacked-asym30",) + _fuzz_instance(30, 7, lo=0, hi=1000))
    out.append(("fuzz-unpacked-sym23",) + _fuzz_instance(23, 8, symmetric=True, diag=False, lo=0, hi=800))
    big = _fuzz_instance(30, 9, lo=0, hi=6)
    out.append(("fuzz-nostage-asym30", big[0] * 9000, big[1]))
    # exactly one symmetric matrix: single-product update with combined vectors (hybrid SYMM = 2)
    for n, which in ((23, "dist"), (30, "flow"), (12, "dist")):
        f, d = _fuzz_instance(n, 40 + n, lo=0, hi=70)
        if which == "dist":
            d = d + d.T
        else:
            f = f + f.T
        out.append((f"fuzz-one-sym-{which}{n}", f, d))
    return out


CASES = _cases()


@pytest.mark.parametrize("name,flow,dist", CASES, ids=[c[0] for c in CASES])
def test_kernels_match_oracle(q, orc, name, flow, dist):
    n = flow.shape[0]
    rng = orc.Rng(77 + n)
    perm = rng.permutation(n)
    lo, hi = orc.tenure_bounds(n)
    iters = 60
    ten = rng.tenures(lo, hi, iters)
    k = q.kernels

    assert k.full_cost(flow, dist, perm) == orc.full_cost(flow, dist, perm)
    assert np.array_equal(k.all_deltas(flow, dist, perm), orc.all_deltas(flow, dist, perm))

    got = k.two_opt_run(flow, dist, perm, iters)
    want = orc.two_opt_run(flow, dist, perm, iters)
    for idx, (g, w) in enumerate(zip(got, want)):
        assert np.array_equal(g, w), f"two_opt_run output {idx}"

    got = k.tabu_run(flow, dist, perm, iters, ten)
    want = orc.tabu_run(flow, dist, perm, iters, ten)
    for idx, (g, w) in enumerate(zip(got[:7], want[:7])):
        assert np.array_equal(g, w), f"tabu_run output {idx}"
    for idx, (g, w) in enumerate(zip(got[7], want[7])):
        assert np.array_equal(g, w), f"tabu trail array {idx}"


def test_inputs_not_mutated(q):
    from paper_2307_11248_b200 import shapes

    inst = shapes.rand(12, 5)
    perm = np.arange(12, dtype=np.int64)[::-1].copy()
    snap = perm.copy()
    q.kernels.two_opt_run(inst.flow, inst.distance, perm, 10)
    q.kernels.tabu_run(inst.flow, inst.distance, perm, 10, np.full(10, 2, np.int64))
    assert np.array_equal(perm, snap)


def test_toy2_known_answers(q):
    """conftest.py:12-18 / test_core.py:31-33,55-56: costs 13 and 17, delta +4."""
    inst = q.parse_instance("2\n0 3\n2 0\n0 1\n5 0", name="toy")
    ident, swapped = np.array([0, 1], np.int64), np.array([1, 0], np.int64)
    assert q.full_cost(inst, ident) == 13
    assert q.full_cost(inst, swapped) == 17
    assert q.all_deltas(inst, ident).tolist() == [4]


def test_premature_stop(q, orc):
    """test_tabu.py:96-105: on n=2 the only move becomes tabu and nothing aspirates."""
    inst = q.parse_instance("2\n0 3\n2 0\n0 1\n5 0", name="toy")
    perm = np.array([0, 1], np.int64)
    ten = np.full(6, 3, np.int64)
    got = q.kernels.tabu_run(inst.flow, inst.distance, perm, 6, ten)
    want = orc.tabu_run(inst.flow, inst.distance, perm, 6, ten)
    assert want[5] is True and got[5] is True
    assert got[6] == want[6]
    for g, w in zip(got[:5], want[:5]):
        assert np.array_equal(g, w)
    for g, w in zip(got[7], want[7]):
        assert np.array_equal(g, w)


def test_batched_runs_match_single(q, orc):
    from paper_2307_11248_b200 import shapes

    inst = shapes.rand(23, 9)
    n, iters, B = 23, 40, 9
    lo, hi = orc.tenure_bounds(n)
    perms, tens = [], []
    for b in range(B):
        r = orc.Rng(orc.derive_seed(3, b))
        perms.append(r.permutation(n))
        tens.append(r.tenures(lo, hi, iters))
    perms, tens = np.stack(perms), np.stack(tens)
    best, bc, cur, cc, cells, stop, steps, tr = q.kernels.tabu_run_batch(inst.flow, inst.distance, perms, iters, tens)
    deltas = q.kernels.all_deltas_batch(inst.flow, inst.distance, perms)
    costs = q.kernels.full_cost_batch(inst.flow, inst.distance, perms)
    for b in range(B):
        want = orc.tabu_run(inst.flow, inst.distance, perms[b], iters, tens[b])
        assert np.array_equal(best[b], want[0]) and bc[b] == want[1]
        assert np.array_equal(cur[b], want[2]) and cc[b] == want[3]
        assert np.array_equal(cells[b], want[4])
        assert steps[b] == want[6]
        assert np.array_equal(tr[0][b, : want[6]], want[7][0])
        assert np.array_equal(tr[2][b, : want[6]], want[7][2])
        assert np.array_equal(deltas[b], orc.all_deltas(inst.flow, inst.distance, perms[b]))
        assert costs[b] == orc.full_cost(inst.flow, inst.distance, perms[b])


@pytest.mark.parametrize("shape,iters,starts", [("tai100a", 40, 3), ("sko100", 40, 2), ("rand100", 30, 2), ("tai128a", 24, 2),
                                                ("rand160", 16, 2), ("tai150b", 24, 2), ("tai256c", 8, 2)])
def test_large_shapes_short_runs(q, orc, shape, iters, starts):
    """BASELINE.json configs 3-5 at oracle-affordable iteration counts, one case per kernel plan:
    register-only (n=100 symmetric / asymmetric, n=128), registers + shared memory (n=160
    asymmetric, n=256), int64 state in the generic kernel (tai150b)."""
    from paper_2307_11248_b200 import shapes
    from paper_2307_11248_b200.backend import device_instance

    inst = shapes.by_name(shape)
    n = inst.n
    info = device_instance(inst.flow, inst.distance).info
    if shape == "tai150b":
        assert info["acc_bits"] == 64
    lo, hi = orc.tenure_bounds(n)
    for b in range(starts):
        r = orc.Rng(orc.derive_seed(11, b))
        perm = r.permutation(n)
        ten = r.tenures(lo, hi, iters)
        assert np.array_equal(q.kernels.all_deltas(inst.flow, inst.distance, perm),
                              orc.all_deltas(inst.flow, inst.distance, perm))
        got = q.kernels.tabu_run(inst.flow, inst.distance, perm, iters, ten)
        want = orc.tabu_run(inst.flow, inst.distance, perm, iters, ten)
        for idx, (g, w) in enumerate(zip(got[:7], want[:7])):
            assert np.array_equal(g, w), f"{shape} tabu output {idx}"
        for idx, (g, w) in enumerate(zip(got[7], want[7])):
            assert np.array_equal(g, w), f"{shape} trail {idx}"
        got2 = q.kernels.two_opt_run(inst.flow, inst.distance, perm, iters)
        want2 = orc.two_opt_run(inst.flow, inst.distance, perm, iters)
        for idx, (g, w) in enumerate(zip(got2, want2)):
            assert np.array_equal(g, w), f"{shape} 2opt output {idx}"


@pytest.mark.parametrize("algo", ["tabu", "2opt"])
@pytest.mark.parametrize("shape,starts,iters", [("rand30", 64, 240), ("nug12", 40, 48), ("tai100a", 8, 60), ("rand5", 33, 20)])
def test_multistart_matches_oracle(q, orc, algo, shape, starts, iters):
    """Device-side RNG + batched search + reduce == reference run_multistart semantics
    (multistart.py:86-172): per-start cost vector, winner, tie rule."""
    from paper_2307_11248_b200 import shapes

    inst = shapes.by_name(shape)
    res = q.run_multistart(inst, q.SearchConfig(algorithm=algo, n_starts=starts, iterations=iters, master_seed=5))
    costs, bc, bi, bp = orc.multistart(inst.flow, inst.distance, algo, 5, starts, iters, threads=orc.max_threads())
    assert np.array_equal(res.per_start_costs, costs)
    assert res.best.cost == bc and res.best_start_index == bi
    assert np.array_equal(res.best.permutation, bp)
    assert res.best.seed == orc.derive_seed(5, bi)
    assert q.evaluate_cost(inst, res.best.permutation) == res.best.cost


def test_multistart_golden_kat30(q):
    """SURVEY.md 8c known answers generated from the reference itself: kat30,
    64 starts x 240 iterations, master seed 0."""
    from paper_2307_11248_b200 import shapes

    inst = shapes.rand(30, 1234)
    res = q.run_multistart(inst, q.SearchConfig(algorithm="tabu", n_starts=64, iterations=240, master_seed=0))
    assert (res.best.cost, res.best_start_index, int(res.per_start_costs.sum())) == (1776990, 23, 115222749)
    res = q.run_multistart(inst, q.SearchConfig(algorithm="2opt", n_starts=64, iterations=120, master_seed=0))
    assert (res.best.cost, res.best_start_index, int(res.per_start_costs.sum())) == (1809350, 36, 117877671)


def test_sequential_rng_path_is_identical(q):
    """The rejection-exact sequential RNG path (taken when a draw would be rejected)
    must give the same starts as the parallel fast path."""
    from paper_2307_11248_b200 import _lib, shapes
    from paper_2307_11248_b200.backend import DeviceInstance

    inst = shapes.rand(23, 2)
    di = DeviceInstance(inst.flow, inst.distance)
    fast = di.multistart("tabu", 9, 0, 16, 30, 2, 8)
    _lib.check(_lib.lib().qapb_debug_force_seq_rng(di.handle, 1))
    slow = di.multistart("tabu", 9, 0, 16, 30, 2, 8)
    assert np.array_equal(fast[0], slow[0]) and fast[1:3] == slow[1:3] and np.array_equal(fast[3], slow[3])
    di.close()


def test_first_index_offsets_are_consistent(q):
    """Sharding invariant used for multi-GPU: starts [8,16) run alone equal the same
    slice of a [0,16) run."""
    from paper_2307_11248_b200 import shapes
    from paper_2307_11248_b200.backend import device_instance

    inst = shapes.rand(12, 4)
    di = device_instance(inst.flow, inst.distance)
    whole = di.multistart("tabu", 3, 0, 16, 40, 1, 4)
    part = di.multistart("tabu", 3, 8, 8, 40, 1, 4)
    assert np.array_equal(whole[0][8:], part[0])


def test_error_mapping(q):
    from paper_2307_11248_b200 import shapes

    inst = shapes.rand(5, 1)
    with pytest.raises(q.DomainError):
        q.kernels.two_opt_run(inst.flow, inst.distance, np.arange(5), -1)
    with pytest.raises(q.DomainError):
        q.run_two_opt(inst, 1, 0)  # the solver entry point refuses an empty budget (two_opt.py:62-63)
    with pytest.raises(q.DomainError):
        q.full_cost(inst, np.arange(4))


def test_randomized_sweep(q, orc):
    """Property sweep in the spirit of test_core.py:76-89 / test_acceptance.py:54-69: random sizes,
    value ranges, symmetry and diagonals; deltas == oracle, run trajectories == oracle."""
    rs = np.random.default_rng(20240824)
    for case in range(40):
        n = int(rs.integers(2, 41))
        hi = int(rs.choice([3, 50, 400, 5000]))
        f = rs.integers(-hi if case % 4 == 0 else 0, hi + 1, (n, n)).astype(np.int64)
        d = rs.integers(0, hi + 1, (n, n)).astype(np.int64)
        if case % 3 == 0:
            f, d = f + f.T, d + d.T
        if case % 2 == 0:
            np.fill_diagonal(f, 0)
            np.fill_diagonal(d, 0)
        rng = orc.Rng(1000 + case)
        perm = rng.permutation(n)
        iters = 25
        lo, hi_t = orc.tenure_bounds(n)
        ten = rng.tenures(lo, hi_t, iters)
        assert np.array_equal(q.kernels.all_deltas(f, d, perm), orc.all_deltas(f, d, perm)), case
        got, want = q.kernels.tabu_run(f, d, perm, iters, ten), orc.tabu_run(f, d, perm, iters, ten)
        for g, w in zip(got[:7], want[:7]):
            assert np.array_equal(g, w), case
        for g, w in zip(got[7], want[7]):
            assert np.array_equal(g, w), case
        got, want = q.kernels.two_opt_run(f, d, perm, iters), orc.two_opt_run(f, d, perm, iters)
        for g, w in zip(got, want):
            assert np.array_equal(g, w), case


def test_exhaustive_solve_small(q, orc):
    """core.exhaustive_solve (core.py:90-108) with GPU-batched costs == brute force with the oracle."""
    import itertools

    from paper_2307_11248_b200 import shapes

    inst = shapes.rand(6, 21)
    perm, cost = q.exhaustive_solve(inst)
    best = min((orc.full_cost(inst.flow, inst.distance, np.array(p)), p) for p in itertools.permutations(range(6)))
    assert cost == best[0] and tuple(perm.tolist()) == best[1]
    # oracle-quality check of test_acceptance.py:73-91: tabu multi-start reaches the optimum on n=6
    res = q.run_multistart(inst, q.SearchConfig(algorithm="tabu", n_starts=32, iterations=48, master_seed=2))
    assert res.best.cost == cost


def test_tabu_not_worse_than_two_opt_and_dominance(q):
    """test_acceptance.py:123-137,194-202: more starts never hurt (subset dominance) and the
    per-start vector of a larger run extends the smaller one."""
    from paper_2307_11248_b200 import shapes

    inst = shapes.rand(20, 5)
    small = q.run_multistart(inst, q.SearchConfig(algorithm="tabu", n_starts=16, iterations=80, master_seed=4))
    large = q.run_multistart(inst, q.SearchConfig(algorithm="tabu", n_starts=64, iterations=80, master_seed=4))
    assert large.best.cost <= small.best.cost
    assert np.array_equal(large.per_start_costs[:16], small.per_start_costs)


@pytest.mark.parametrize("storage", ["0", "1", "2"])
@pytest.mark.parametrize("shape", ["rand23", "tai30a", "tai45b"])
def test_generic_kernel_storage_modes(q, orc, monkeypatch, shape, storage):
    """Every placement of the generic kernel's state (M in shared memory / M in L2 / M and the tabu
    masks in L2), int32 (rand, tai*a) and int64 (tai*b) state."""
    from paper_2307_11248_b200 import shapes
    from paper_2307_11248_b200.backend import DeviceInstance

    monkeypatch.setenv("QAPB_FORCE_GENERIC", "1")
    if storage != "0":
        monkeypatch.setenv("QAPB_FORCE_STORAGE", storage)
    inst = shapes.by_name(shape)
    n, iters = inst.n, 50
    di = DeviceInstance(inst.flow, inst.distance)
    try:
        assert di.info["storage"] == int(storage)
        assert di.info["acc_bits"] == (64 if shape.endswith("b") else 32)
        lo, hi = orc.tenure_bounds(n)
        perms, tens = [], []
        for b in range(3):
            r = orc.Rng(orc.derive_seed(17, b))
            perms.append(r.permutation(n))
            tens.append(r.tenures(lo, hi, iters))
        perms, tens = np.stack(perms), np.stack(tens)
        best, bc, cur, cc, cz, stop, steps, tr, _ = di.tabu(perms, iters, tens)
        b2, bc2, cur2, cc2, mi, mj, md = di.two_opt(perms, iters)
        deltas = di.all_deltas(perms)
        for b in range(3):
            want = orc.tabu_run(inst.flow, inst.distance, perms[b], iters, tens[b])
            assert np.array_equal(best[b], want[0]) and bc[b] == want[1]
            assert np.array_equal(cur[b], want[2]) and cc[b] == want[3]
            assert np.array_equal(cz[b], want[4]) and steps[b] == want[6]
            for a in range(4):
                assert np.array_equal(tr[a][b, : want[6]], want[7][a])
            w2 = orc.two_opt_run(inst.flow, inst.distance, perms[b], iters)
            for g, w in zip((b2[b], bc2[b], cur2[b], cc2[b], mi[b], mj[b], md[b]), w2):
                assert np.array_equal(g, w)
            assert np.array_equal(deltas[b], orc.all_deltas(inst.flow, inst.distance, perms[b]))
        costs, kbest, kidx, kperm = di.multistart("tabu", 21, 0, 6, iters, lo, hi)
        wc, wbc, wbi, wbp = orc.multistart(inst.flow, inst.distance, "tabu", 21, 6, iters, threads=orc.max_threads())
        assert np.array_equal(costs, wc) and (kbest, kidx) == (wbc, wbi) and np.array_equal(kperm, wbp)
    finally:
        di.close()


def test_batched_runs_equal_separate_calls(q):
    """sweep.run_multistart_many / run_repetitions / run_sweep: one launch per (algorithm, iterations,
    tenure) group gives the MultiStartResult of separate run_multistart calls (cli.py:109-116,162-175)."""
    from dataclasses import replace

    from paper_2307_11248_b200 import shapes

    inst = shapes.rand(23, 6)
    base = q.SearchConfig(algorithm="tabu", n_starts=12, iterations=40, master_seed=3)
    cfgs = [base, replace(base, master_seed=4), replace(base, algorithm="2opt", iterations=25),
            replace(base, n_starts=5, master_seed=3 + 7919), replace(base, iterations=17)]
    many = q.run_multistart_many(inst, cfgs)
    for cfg, got in zip(cfgs, many):
        want = q.run_multistart(inst, cfg)
        assert np.array_equal(got.per_start_costs, want.per_start_costs)
        assert (got.best.cost, got.best_start_index, got.best.seed) == (want.best.cost, want.best_start_index, want.best.seed)
        assert np.array_equal(got.best.permutation, want.best.permutation)
        assert got.config_digest == want.config_digest
    reps = q.run_repetitions(inst, base, 3)
    assert [r.best.cost for r in reps] == [q.run_multistart(inst, replace(base, master_seed=3 + k)).best.cost for k in range(3)]
    rows = q.run_sweep(inst, q.make_sweep("seeds", [1, 3], base), 2)
    for value, rep, cost in rows:
        want = min(q.run_multistart(inst, replace(base, master_seed=3 + rep + 7919 * idx)).best.cost for idx in range(value))
        assert cost == want
    rows = q.run_sweep(inst, q.make_sweep("neighborhoods", [10, 30], base), 1)
    assert [c for _, _, c in rows] == [q.run_multistart(inst, replace(base, iterations=v)).best.cost for v in (10, 30)]
    from paper_2307_11248_b200._refpkg import reference

    if reference() is not None:  # the best-known registry is the reference's object
        rep = q.bench_report(inst, base, 3, q.BestKnownRegistry({inst.name: 1000}))
        assert rep.per_run_costs == [r.best.cost for r in reps] and rep.best_cost == min(rep.per_run_costs)
        assert rep.accuracy == q.accuracy(rep.best_cost, 1000) and rep.config_digest == q.config_digest(inst, base)


@pytest.mark.parametrize("n,iters", [(257, 6), (400, 4), (1020, 2)])
def test_sizes_beyond_the_hybrid_plans(q, orc, n, iters):
    """n > 256 runs in the generic kernel with M in the L2-resident workspace; n = 1020 is the largest
    supported size.  Few iterations: the oracle is O(n^3) per iteration."""
    from paper_2307_11248_b200 import shapes
    from paper_2307_11248_b200.backend import device_instance

    inst = shapes.rand(n, 77)
    info = device_instance(inst.flow, inst.distance).info
    assert info["storage"] == (2 if n > 700 else 1) and info["acc_bits"] == 32
    rng = orc.Rng(orc.derive_seed(5, n))
    perm = rng.permutation(n)
    lo, hi = orc.tenure_bounds(n)
    ten = rng.tenures(lo, hi, iters)
    assert np.array_equal(q.kernels.all_deltas(inst.flow, inst.distance, perm), orc.all_deltas(inst.flow, inst.distance, perm))
    got = q.kernels.tabu_run(inst.flow, inst.distance, perm, iters, ten)
    want = orc.tabu_run(inst.flow, inst.distance, perm, iters, ten)
    for idx, (g, w) in enumerate(zip(got[:7], want[:7])):
        assert np.array_equal(g, w), f"n={n} tabu output {idx}"
    for idx, (g, w) in enumerate(zip(got[7], want[7])):
        assert np.array_equal(g, w), f"n={n} trail {idx}"


def test_unsupported_sizes_and_values(q):
    """n > 1020 and |entry| >= 2^30 are refused with QapError (status QAPB_ERR_UNSUPPORTED), not computed wrongly."""
    from paper_2307_11248_b200.backend import DeviceInstance

    big = np.zeros((1021, 1021), np.int64)
    with pytest.raises(q.QapError):
        DeviceInstance(big, big)
    f = np.zeros((4, 4), np.int64)
    f[0, 1] = 1 << 30
    with pytest.raises(q.QapError):
        DeviceInstance(f, np.ones((4, 4), np.int64))
    with pytest.raises(q.DomainError):
        DeviceInstance(np.zeros((1, 1), np.int64), np.zeros((1, 1), np.int64))


@pytest.mark.parametrize("which,scale", [("dist", 1), ("flow", 1), ("dist", 40000), ("flow", 40000)])
def test_generic_kernel_one_symmetric_matrix(q, orc, monkeypatch, which, scale):
    """One symmetric matrix lets the generic kernel's rank-2 update use a single product per entry
    (a == c or b == e); int32 state (scale 1) and int64 state (large entries)."""
    from paper_2307_11248_b200.backend import DeviceInstance

    monkeypatch.setenv("QAPB_FORCE_GENERIC", "1")
    rs = np.random.default_rng(31 + scale)
    n, iters = 27, 40
    f = rs.integers(0, 60, (n, n)).astype(np.int64)
    d = rs.integers(0, 60, (n, n)).astype(np.int64)
    if which == "dist":
        d = d + d.T
        f = f * scale
    else:
        f = f + f.T
        d = d * scale
    np.fill_diagonal(f, rs.integers(0, 9, n))  # non-zero diagonals too
    di = DeviceInstance(f, d)
    try:
        assert di.info["storage"] == 0 and di.info["symmetric"] == 0
        assert di.info["acc_bits"] == (32 if scale == 1 else 64)
        lo, hi = orc.tenure_bounds(n)
        rng = orc.Rng(orc.derive_seed(9, scale))
        perm = rng.permutation(n)
        ten = rng.tenures(lo, hi, iters)
        best, bc, cur, cc, cz, stop, steps, tr, _ = di.tabu(perm, iters, ten)
        want = orc.tabu_run(f, d, perm, iters, ten)
        assert np.array_equal(best[0], want[0]) and bc[0] == want[1] and np.array_equal(cur[0], want[2]) and cc[0] == want[3]
        assert np.array_equal(cz[0], want[4]) and steps[0] == want[6]
        for a in range(4):
            assert np.array_equal(tr[a][0, : want[6]], want[7][a])
        b2 = di.two_opt(perm, iters)
        for g, w in zip([x[0] for x in b2], orc.two_opt_run(f, d, perm, iters)):
            assert np.array_equal(g, w)
    finally:
        di.close()


@pytest.mark.parametrize("shape,iters", [("rand30", 40), ("tai112a", 16), ("rand132", 12), ("tai200a", 8)])
def test_every_launch_plan_gives_identical_results(q, orc, shape, iters):
    """tuner: results do not depend on the launch plan (one / two register units, shared-memory units,
    diagonal blocks in registers or shared memory, one or two searches per SM)."""
    from paper_2307_11248_b200 import shapes
    from paper_2307_11248_b200.backend import DeviceInstance

    inst = shapes.by_name(shape)
    lo, hi = orc.tenure_bounds(inst.n)
    want = orc.multistart(inst.flow, inst.distance, "tabu", 13, 5, iters, threads=orc.max_threads())
    di = DeviceInstance(inst.flow, inst.distance)
    try:
        plans = di.plan_candidates()
        assert len(plans) >= 2 and di.info["storage"] in (3, 4)
        for plan in plans:
            di.set_plan(plan)
            costs, bc, bi, bp = di.multistart("tabu", 13, 0, 5, iters, lo, hi)
            assert np.array_equal(costs, want[0]) and (bc, bi) == (want[1], want[2]) and np.array_equal(bp, want[3]), plan
        with pytest.raises(q.DomainError):
            di.set_plan((1, 32, 0, 0) if inst.n > 64 else (2, 4096, 0, 0))
    finally:
        di.close()
    # instances of the generic kernel have a single configuration (n > 256 here; tai*b shapes run on the
    # register / shared-memory plans with 64-bit deltas since round 2)
    big = shapes.by_name("tai300a")
    assert DeviceInstance(big.flow, big.distance).plan_candidates() == []
    wide = DeviceInstance(shapes.by_name("tai45b").flow, shapes.by_name("tai45b").distance)
    assert wide.info["storage"] == 3 and wide.info["acc_bits"] == 64 and len(wide.plan_candidates()) >= 1


def test_autotune_installs_the_fastest_plan(q):
    from paper_2307_11248_b200 import shapes
    from paper_2307_11248_b200.backend import device_instance

    inst = shapes.by_name("tai64c")
    timings = q.autotune(inst, iterations=40)
    assert timings and all(a.evals_per_second >= b.evals_per_second for a, b in zip(timings, timings[1:]))
    di = device_instance(inst.flow, inst.distance)
    assert di.info["threads"] == timings[0].threads
    assert q.autotune(shapes.by_name("tai300a"), iterations=8, n_starts=8) == []  # generic kernel: one configuration


@pytest.mark.parametrize("n", [5, 12, 30, 100, 130])
def test_explicit_tenures_at_the_edges(q, orc, n):
    """Caller-provided tenures outside the sampled interval (`tabu_run` takes any int64 array,
    _kernels.pyx:121,176): zero and negative tenures (the cell is never tabu), a mix, and tenures so
    long that every move becomes tabu and the search stops early (_kernels.pyx:168-170)."""
    from paper_2307_11248_b200 import shapes

    inst = shapes.rand(n, 300 + n)
    rng = orc.Rng(5 + n)
    perm = rng.permutation(n)
    iters = 40 if n <= 30 else 12
    gen = np.random.default_rng(n)
    patterns = {
        "zero": np.zeros(iters, np.int64),
        "negative": np.full(iters, -3, np.int64),
        "mixed": gen.integers(-2, 6, iters).astype(np.int64),
        "long": np.full(iters, 1_000_000, np.int64),
        "alternating": np.where(np.arange(iters) % 2 == 0, 1_000_000, 0).astype(np.int64),
    }
    # n = 30 also with entries that force the int64 generic kernel
    variants = [(inst.flow, inst.distance)] + ([(inst.flow * 40000, inst.distance * 9000)] if n == 30 else [])
    for flow, dist in variants:
        for label, ten in patterns.items():
            got = q.kernels.tabu_run(flow, dist, perm, iters, ten)
            want = orc.tabu_run(flow, dist, perm, iters, ten)
            for idx, (g, w) in enumerate(zip(got[:7], want[:7])):
                assert np.array_equal(g, w), f"{label}: tabu_run output {idx}"
            for idx, (g, w) in enumerate(zip(got[7], want[7])):
                assert np.array_equal(g, w), f"{label}: trail array {idx}"


def test_tenure_beyond_int32_is_refused(q):
    """Expiry iterations are kept in int32 on the device: a tenure that would overflow is an error,
    not a silent wrap."""
    from paper_2307_11248_b200 import shapes

    inst = shapes.rand(12, 1)
    perm = np.arange(12, dtype=np.int64)
    with pytest.raises(q.QapError):
        q.kernels.tabu_run(inst.flow, inst.distance, perm, 4, np.array([1, 2**31, 1, 1], np.int64))
    with pytest.raises(q.QapError):
        q.kernels.tabu_run(inst.flow, inst.distance, perm, 4, np.array([1, 1, -2**31 - 9, 1], np.int64))


def test_zero_iterations_return_the_start(q, orc):
    """kernels.two_opt_run / tabu_run with an empty budget (the loops of _kernels.pyx:94,153 do not
    run): best = current = start, empty move arrays, zero cells -- as the reference returns."""
    from paper_2307_11248_b200 import shapes

    inst = shapes.rand(12, 9)
    perm = orc.Rng(4).permutation(12)
    cost = orc.full_cost(inst.flow, inst.distance, perm)
    got = q.kernels.two_opt_run(inst.flow, inst.distance, perm, 0)
    assert np.array_equal(got[0], perm) and np.array_equal(got[2], perm) and got[1] == cost == got[3]
    assert all(a.shape == (0,) and a.dtype == np.int64 for a in got[4:])
    got = q.kernels.tabu_run(inst.flow, inst.distance, perm, 0, np.zeros(0, np.int64))
    assert np.array_equal(got[0], perm) and got[1] == cost and np.array_equal(got[2], perm) and got[3] == cost
    assert not got[4].any() and got[4].shape == (12, 12) and got[5] is False and got[6] == 0
    assert len(got[7]) == 6 and all(a.shape == (0,) for a in got[7])
    assert got[0] is not perm


def test_instance_cache_never_serves_stale_matrices(q, orc):
    """The kernels interface takes (flow, dist) on every call (backend.py:16-29) and the shim caches
    the uploaded instance: by identity only for frozen arrays that own their data, by content
    otherwise -- an in-place edit of a caller's array (or of the base of a read-only view) must be seen."""
    from paper_2307_11248_b200 import shapes
    from paper_2307_11248_b200.backend import device_instance

    inst = shapes.rand(12, 77)
    assert device_instance(inst.flow, inst.distance) is device_instance(inst.flow, inst.distance)
    perm = np.arange(12, dtype=np.int64)

    f = inst.flow.copy()
    d = inst.distance.copy()
    assert q.kernels.full_cost(f, d, perm) == orc.full_cost(f, d, perm)
    f[0, 1] += 5
    assert q.kernels.full_cost(f, d, perm) == orc.full_cost(f, d, perm)
    assert np.array_equal(q.kernels.all_deltas(f, d, perm), orc.all_deltas(f, d, perm))

    view = f.view()
    view.setflags(write=False)
    before = q.kernels.full_cost(view, d, perm)
    f[0, 1] += 7  # the base changes under the read-only view
    after = q.kernels.full_cost(view, d, perm)
    assert after == orc.full_cost(f, d, perm) and after != before


@pytest.mark.parametrize("shape,algo,starts,budgets", [("rand23", "tabu", 9, [1, 5, 23, 60]), ("rand30", "2opt", 7, [2, 40]),
                                                       ("tai100a", "tabu", 40, [50, 100, 400]),
                                                       ("tai150b", "tabu", 6, [10, 60])])
def test_budget_sweep_from_one_traced_run(q, orc, shape, algo, starts, budgets):
    """qapb_multistart_trace + sweep.best_costs_at_budgets: one run at the largest budget reproduces
    `run_multistart(...).per_start_costs` of every shorter budget (the neighborhoods axis of
    cli.py:162-166); the recorded trajectories equal the oracle's, and run_sweep uses it."""
    from dataclasses import replace

    from paper_2307_11248_b200 import shapes
    from paper_2307_11248_b200.backend import device_instance
    from paper_2307_11248_b200.sweep import derive_seeds

    inst = shapes.by_name(shape)
    cfg = q.SearchConfig(algorithm=algo, n_starts=starts, iterations=budgets[-1], master_seed=77)
    table = q.best_costs_at_budgets(inst, cfg, budgets)
    for row, v in zip(table, budgets):
        assert np.array_equal(row, q.run_multistart(inst, replace(cfg, iterations=v)).per_start_costs), v
    # trajectories of the traced run against the oracle (first starts; the oracle is O(n^3) per iteration)
    ten = q.tenure_bounds(inst.n)
    top = budgets[-1] if inst.n <= 30 else budgets[0]
    seeds = derive_seeds(77, 0, starts)
    costs, perms, steps, mi, mj, md = device_instance(inst.flow, inst.distance).multistart_trace(algo, seeds, top, ten.low, ten.high)
    for b in range(min(starts, 3)):
        rng = orc.Rng(int(seeds[b]))
        perm = rng.permutation(inst.n)
        if algo == "tabu":
            want = orc.tabu_run(inst.flow, inst.distance, perm, top, rng.tenures(ten.low, ten.high, top))
            k, wi, wj, wd = int(want[6]), want[7][0], want[7][1], want[7][2]
        else:
            want = orc.two_opt_run(inst.flow, inst.distance, perm, top)
            k, wi, wj, wd = top, want[4], want[5], want[6]
        assert int(steps[b]) == k and int(costs[b]) == int(want[1]) and np.array_equal(perms[b], want[0])
        assert np.array_equal(mi[b, :k], wi[:k]) and np.array_equal(mj[b, :k], wj[:k]) and np.array_equal(md[b, :k], wd[:k])
    if inst.n <= 30:
        rows = q.run_sweep(inst, q.make_sweep("neighborhoods", budgets, cfg), 2)
        for value, rep, cost in rows:
            assert cost == q.run_multistart(inst, replace(cfg, iterations=value, master_seed=77 + rep)).best.cost


@pytest.mark.parametrize("n,kind,scale", [(27, 0, 23000), (27, 1, 6000), (27, 2, 12000), (100, 2, 3800), (100, 0, 6600),
                                          (150, 2, 2600), (150, 1, 1500), (150, 0, 4800), (130, 3, 2900)])
def test_unsigned_state_with_64_bit_deltas(q, orc, n, kind, scale):
    """Non-negative instances whose bound exceeds int32 but not 2^32 (tai*b shapes) keep unsigned 32-bit state on the
    register / shared-memory plans; only deltas, threshold and argmin are 64-bit.  Every plan, every symmetry class
    (kind 0: none, 1: both, 2: distance only, 3: flow only), tabu with trail and cells, 2opt, all_deltas, multi-start."""
    from paper_2307_11248_b200.backend import DeviceInstance

    rs = np.random.default_rng(7 * n + kind)
    f = (rs.integers(0, 60, (n, n)) * scale).astype(np.int64)
    d = rs.integers(0, 60, (n, n)).astype(np.int64)
    f[rs.random((n, n)) < 0.4] = 0
    if kind in (1, 2):
        d = d + d.T
    if kind in (1, 3):
        f = f + f.T
    np.fill_diagonal(f, rs.integers(0, 9, n))
    np.fill_diagonal(d, rs.integers(0, 5, n))
    di = DeviceInstance(f, d)
    try:
        assert di.info["storage"] == 3 and di.info["acc_bits"] == 64, di.info
        iters = 40 if n > 100 else 90
        rng = orc.Rng(orc.derive_seed(n, kind))
        perm = rng.permutation(n)
        ten = rng.tenures(1, 4, iters)
        want = orc.tabu_run(f, d, perm, iters, ten)
        assert abs(int(np.abs(want[7][2]).max())) > 2 ** 27, "deltas too small to exercise the wide path"
        for plan in di.plan_candidates() or [None]:
            if plan is not None:
                di.set_plan(plan)
            best, bc, cur, cc, cz, stop, steps, tr, _ = di.tabu(perm, iters, ten)
            assert np.array_equal(best[0], want[0]) and bc[0] == want[1] and np.array_equal(cur[0], want[2]) and cc[0] == want[3], plan
            assert np.array_equal(cz[0], want[4]) and steps[0] == want[6] and bool(stop[0]) == want[5], plan
            for a in range(4):
                assert np.array_equal(tr[a][0, : want[6]], want[7][a]), (plan, a)
            for g, w in zip([x[0] for x in di.two_opt(perm, iters)], orc.two_opt_run(f, d, perm, iters)):
                assert np.array_equal(g, w), plan
        assert np.array_equal(di.all_deltas(perm)[0], orc.all_deltas(f, d, perm))
        lo, hi = orc.tenure_bounds(n)
        got = di.multistart("tabu", 3, 0, 5, iters, lo, hi)
        w2 = orc.multistart(f, d, "tabu", 3, 5, iters, threads=orc.max_threads())
        assert np.array_equal(got[0], w2[0]) and got[1:3] == (w2[1], w2[2]) and np.array_equal(got[3], w2[3])
    finally:
        di.close()


def test_multistart_runs_in_waves_under_a_memory_budget(q, orc, monkeypatch):
    """qapb_multistart splits a batch whose per-start workspace exceeds the memory budget into waves (the reference's
    default of 6144 starts on a large instance would otherwise ask for tens of GB); the result is the same."""
    from paper_2307_11248_b200 import shapes
    from paper_2307_11248_b200.backend import DeviceInstance

    for name, starts, iters, budget in (("tai30a", 64, 40, 100_000), ("tai45b", 23, 30, 120_000), ("tai300a", 7, 3, 3_000_000)):
        inst = shapes.by_name(name)
        lo, hi = orc.tenure_bounds(inst.n)
        want = orc.multistart(inst.flow, inst.distance, "tabu", 9, starts, iters, threads=orc.max_threads())
        monkeypatch.setenv("QAPB_WAVE_BYTES", str(budget))
        di = DeviceInstance(inst.flow, inst.distance)
        try:
            got = di.multistart("tabu", 9, 0, starts, iters, lo, hi)
            assert np.array_equal(got[0], want[0]) and got[1:3] == (want[1], want[2]) and np.array_equal(got[3], want[3]), name
            assert di.last_total_steps() == starts * iters
            # a shard that does not start at index 0
            got = di.multistart("tabu", 9, 5, starts - 5, iters, lo, hi)
            assert np.array_equal(got[0], want[0][5:]), name
        finally:
            di.close()
        monkeypatch.delenv("QAPB_WAVE_BYTES")
