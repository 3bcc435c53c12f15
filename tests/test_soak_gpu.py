"""Differential soak inside the driver-run suite: GPU vs the C oracle on random instances at the sizes
whose launch plans keep part of a search in shared memory / L2 (n = 129 .. 256) and at the small sizes,
with SHORT tenures ([1, 3]) and enough iterations that tabu bits expire and re-arm many times on every
plan's expiry path (register units, shared-memory units, shared-memory diagonal blocks, L2 expiries).
Every launch plan of each instance must reproduce the oracle bit for bit.  (tests/soak_gpu.py is the
open-ended version of the same loop.)"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _instance(rs, n, kind, hi):
    f = rs.integers(0, hi + 1, (n, n)).astype(np.int64)
    d = rs.integers(0, hi + 1, (n, n)).astype(np.int64)
    if kind in (1, 3):
        d = d + d.T
    if kind in (2, 3):
        f = f + f.T
    if kind != 0:
        np.fill_diagonal(f, 0)
        np.fill_diagonal(d, 0)
    return f, d


def _check_single(di, oracle, f, d, perm, iters, ten, tag):
    g = di.tabu(perm, iters, ten)
    w = oracle.tabu_run(f, d, perm, iters, ten)
    assert np.array_equal(g[0][0], w[0]) and g[1][0] == w[1], tag
    assert np.array_equal(g[2][0], w[2]) and g[3][0] == w[3], tag
    assert np.array_equal(g[4][0], w[4]), tag                      # final tabu memory `cells`
    assert bool(g[5][0]) == w[5] and g[6][0] == w[6], tag          # stopped_early, steps_done
    for a in range(4):                                             # trail: i, j, delta, tabu flag
        assert np.array_equal(g[7][a][0, : w[6]], w[7][a]), (tag, a)
    return w


@pytest.mark.parametrize("n,kind,hi", [(129, 3, 60), (160, 3, 99), (160, 1, 30), (200, 3, 99), (200, 0, 20),
                                       (256, 3, 99), (256, 2, 12), (144, 3, 3000), (164, 3, 50), (176, 3, 99), (100, 3, 99), (100, 0, 99),
                                       (64, 3, 99), (33, 1, 1000), (30, 3, 99), (12, 0, 50)])
def test_short_tenures_every_plan(built, n, kind, hi):
    import oracle
    from paper_2307_11248_b200.backend import DeviceInstance

    rs = np.random.default_rng(1000 * n + 10 * kind + 1)
    f, d = _instance(rs, n, kind, hi)
    iters = 64 if n > 128 else 150
    rng = oracle.Rng(oracle.derive_seed(n, kind))
    ten = rng.tenures(1, 3, iters)
    di = DeviceInstance(f, d)
    try:
        # start next to a local optimum (the current permutation of a long 2opt run; any permutation is a valid
        # input, the oracle checks the tabu run from it): the search then moves uphill, its reverse moves are
        # tabu, expire after 1-3 iterations and are taken again -- every expiry path is hit many times
        perm = di.two_opt(rng.permutation(n), 3 * n, moves=False)[2][0]
        plans = di.plan_candidates() or [None]
        want = None
        for plan in plans:
            if plan is not None:
                di.set_plan(plan)
            want = _check_single(di, oracle, f, d, perm, iters, ten, (n, kind, plan))
        pairs = list(zip(want[7][0].tolist(), want[7][1].tolist()))
        assert len(set(pairs)) < len(pairs), "no pair was ever taken twice: the case does not exercise expiry"
        # batched device-RNG path with a short tenure interval: compare against single-start runs drawn on the host
        for plan in plans[:2]:
            if plan is not None:
                di.set_plan(plan)
            costs = di.multistart("tabu", 77, 0, 3, iters, 1, 3)[0]
            for idx in range(3):
                r2 = oracle.Rng(oracle.derive_seed(77, idx))
                p2 = r2.permutation(n)
                t2 = r2.tenures(1, 3, iters)
                assert int(costs[idx]) == int(oracle.tabu_run(f, d, p2, iters, t2)[1]), (n, kind, plan, idx)
    finally:
        di.close()


@pytest.mark.parametrize("n,hi", [(160, 99), (256, 40)])
def test_two_opt_every_plan(built, n, hi):
    import oracle
    from paper_2307_11248_b200.backend import DeviceInstance

    rs = np.random.default_rng(n)
    f, d = _instance(rs, n, 3, hi)
    perm = oracle.Rng(5).permutation(n)
    w = oracle.two_opt_run(f, d, perm, 48)
    di = DeviceInstance(f, d)
    try:
        for plan in di.plan_candidates() or [None]:
            if plan is not None:
                di.set_plan(plan)
            g = di.two_opt(perm, 48)
            assert all(np.array_equal(a[0], b) for a, b in zip(g, w)), (n, plan)
    finally:
        di.close()


@pytest.mark.parametrize("n,hi", [(130, 99), (152, 60), (164, 99), (176, 40)])
def test_register_only_plan_above_128(built, n, hi):
    """n = 129..176 with two symmetric matrices and packed keys run by default on the register-only kernel of
    n <= 128 in layout size class 256 (one search per SM on noff + 64 threads; 72 registers up to n = 164, 64 above):
    the recording, the multi-start tabu and the multi-start 2opt instantiations against the oracle."""
    import oracle
    from paper_2307_11248_b200.backend import DeviceInstance

    rs = np.random.default_rng(7 * n)
    f, d = _instance(rs, n, 3, hi)
    nb = (n + 3) // 4
    noff = nb * (nb - 1) // 2
    di = DeviceInstance(f, d)
    try:
        info = di.info
        assert info["storage"] == 3 and info["units_per_thread"] == 1 and info["ctas_per_sm"] == 1, info
        assert info["threads"] == (noff + 31) // 32 * 32 + 64, info
        iters = 80
        rng = oracle.Rng(oracle.derive_seed(n, 1))
        perm = di.two_opt(rng.permutation(n), 3 * n, moves=False)[2][0]
        _check_single(di, oracle, f, d, perm, iters, rng.tenures(1, 3, iters), (n, "short tenures"))
        lo, hi_t = oracle.tenure_bounds(n)
        for algo in ("tabu", "2opt"):
            got = di.multistart(algo, 11, 0, 5, iters, lo, hi_t)
            want = oracle.multistart(f, d, algo, 11, 5, iters, threads=oracle.max_threads())
            assert np.array_equal(got[0], want[0]) and got[1:3] == (want[1], want[2]), (n, algo)
            assert np.array_equal(got[3], want[3]), (n, algo)
    finally:
        di.close()


def test_wide_plan_follows_the_batch_size(built):
    """64-bit deltas at n > 128 (the tai150b shape): a batch of at most one search per SM runs on the register-only
    plan, a larger one on the default plan with two searches per SM (qapb_handle::have_alt); qapb_set_plan pins the
    plan.  Results equal the oracle's either way."""
    import oracle
    from paper_2307_11248_b200 import shapes
    from paper_2307_11248_b200.backend import DeviceInstance

    inst = shapes.by_name("tai150b")
    f, d = np.asarray(inst.flow), np.asarray(inst.distance)
    n = inst.n
    nb = (n + 3) // 4
    tro = (nb * (nb - 1) // 2 + 31) // 32 * 32
    lo, hi = oracle.tenure_bounds(n)
    di = DeviceInstance(f, d)
    try:
        assert di.info["acc_bits"] == 64 and di.info["storage"] == 3
        default_threads = di.info["threads"]
        sm = di.info["sm_count"]
        got = di.multistart("tabu", 3, 0, 6, 48, lo, hi)
        di._refresh_info()  # (the cached dict is refreshed by set_plan only)
        assert di.info["threads"] == tro + 64 and di.info["ctas_per_sm"] == 1, di.info
        want = oracle.multistart(f, d, "tabu", 3, 6, 48, threads=oracle.max_threads())
        assert np.array_equal(got[0], want[0]) and got[1:3] == (want[1], want[2]) and np.array_equal(got[3], want[3])
        big = di.multistart("tabu", 3, 0, sm + 8, 6, lo, hi)
        di._refresh_info()
        assert di.info["threads"] == default_threads, di.info
        want_big = oracle.multistart(f, d, "tabu", 3, sm + 8, 6, threads=oracle.max_threads())
        assert np.array_equal(big[0], want_big[0]) and big[1:3] == (want_big[1], want_big[2])
        # a caller's own choice stands
        plan = [p for p in di.plan_candidates() if p[2] > 0][0]
        di.set_plan(plan)
        pinned = di.info["threads"]
        again = di.multistart("tabu", 3, 0, 6, 48, lo, hi)
        di._refresh_info()
        assert di.info["threads"] == pinned and np.array_equal(again[0], want[0])
    finally:
        di.close()
