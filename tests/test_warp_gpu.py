"""The one-warp-per-search kernel (csrc/search_warp.cuh, n <= 32; two searches per warp at n <= 16) against the
C oracle: every size from 2 to 32 (every count of off-diagonal units, diagonal pairs and pad locations),
symmetric / asymmetric / non-zero diagonals / negative entries, full trails and tabu memory, short tenures
(expiry and re-arming of unit bits and of diagonal pairs), the exact sequential tenure replay, batches that
do not fill a warp or a CTA, and a start-index offset (_kernels.pyx:73-197, multistart.py:86-118)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _instance(n, kind, seed):
    rs = np.random.default_rng(seed)
    lo = -30 if kind == 4 else 0
    f = rs.integers(lo, 100, (n, n)).astype(np.int64)
    d = rs.integers(lo, 100, (n, n)).astype(np.int64)
    if kind in (1, 3):
        d = d + d.T
    if kind in (2, 3):
        f = f + f.T
    if kind in (1, 2, 3):
        np.fill_diagonal(f, 0)
        np.fill_diagonal(d, 0)
    return f, d


def _same_single(got, want, tag):
    for k in range(4):
        assert np.array_equal(np.asarray(got[k]).reshape(-1), np.asarray(want[k]).reshape(-1)), (tag, k)
    assert np.array_equal(got[4][0], want[4]), (tag, "cells")
    assert bool(got[5][0]) == want[5] and got[6][0] == want[6], (tag, "stop")
    for a in range(4):
        assert np.array_equal(got[7][a][0, : want[6]], want[7][a]), (tag, "trail", a)


@pytest.mark.parametrize("n", list(range(2, 33)))
def test_every_size_single_runs(built, n):
    import oracle
    from paper_2307_11248_b200.backend import DeviceInstance

    for kind in (3, 0, 4):
        f, d = _instance(n, kind, 100 * n + kind)
        di = DeviceInstance(f, d)
        try:
            plan = di.plan_candidates()[0]
            assert plan[0] == 0 and di.info["threads"] % 32 == 0, "the warp plan is the default at n <= 32"
            rng = oracle.Rng(oracle.derive_seed(n, kind))
            perm = rng.permutation(n)
            iters = 90
            for tl, th in (oracle.tenure_bounds(n), (1, 3)):
                ten = rng.tenures(tl, th, iters)
                _same_single(di.tabu(perm, iters, ten), oracle.tabu_run(f, d, perm, iters, ten), (n, kind, tl, th))
            g = di.two_opt(perm, 40)
            w = oracle.two_opt_run(f, d, perm, 40)
            assert all(np.array_equal(a[0], b) for a, b in zip(g, w)), (n, kind, "2opt")
        finally:
            di.close()


@pytest.mark.parametrize("n,kind", [(5, 3), (12, 3), (13, 0), (16, 3), (17, 3), (24, 0), (30, 3), (32, 3), (32, 0)])
def test_multistart_batches(built, n, kind):
    """Device-drawn starts and tenures: batches of 1, 3 (half a warp's worth at n <= 16 plus one), 37 and 301
    searches (partial warps and CTAs), a start-index offset, both algorithms, and the sequential RNG path."""
    import oracle
    from paper_2307_11248_b200 import _lib
    from paper_2307_11248_b200.backend import DeviceInstance

    f, d = _instance(n, kind, 7 * n + kind)
    lo, hi = oracle.tenure_bounds(n)
    di = DeviceInstance(f, d)
    try:
        for algo in ("tabu", "2opt"):
            iters = 2 * n + 3
            want = oracle.multistart(f, d, algo, 21, 301, iters, first_index=4, threads=oracle.max_threads())
            for count in (1, 3, 37, 301):
                got = di.multistart(algo, 21, 4, count, iters, lo, hi)
                assert np.array_equal(got[0], want[0][:count]), (n, kind, algo, count)
                k = int(np.argmin(want[0][:count]))
                assert got[1] == int(want[0][k]) and got[2] == 4 + k, (n, kind, algo, count)
        # short tenure interval on the device stream, fast and exact-sequential draws
        fast = di.multistart("tabu", 9, 0, 33, 60, 1, 3)
        for idx in (0, 1, 32):
            r2 = oracle.Rng(oracle.derive_seed(9, idx))
            p2 = r2.permutation(n)
            t2 = r2.tenures(1, 3, 60)
            assert int(fast[0][idx]) == int(oracle.tabu_run(f, d, p2, 60, t2)[1]), (n, kind, idx)
        _lib.check(_lib.lib().qapb_debug_force_seq_rng(di.handle, 1))
        slow = di.multistart("tabu", 9, 0, 33, 60, 1, 3)
        assert np.array_equal(fast[0], slow[0]) and fast[1:3] == slow[1:3] and np.array_equal(fast[3], slow[3])
    finally:
        di.close()


def test_traced_multistart_and_early_stop(built):
    """Recorded trajectories of several starts in one launch, and a search that runs out of admissible moves
    (n = 3 with long tenures: three pairs, all tabu after three moves unless one aspirates)."""
    import oracle
    from paper_2307_11248_b200.backend import DeviceInstance

    f, d = _instance(14, 3, 5)
    di = DeviceInstance(f, d)
    try:
        seeds = np.array([oracle.derive_seed(3, k) for k in range(9)], np.uint64)
        costs, perms, steps, mi, mj, md = di.multistart_trace("tabu", seeds, 50, 2, 5)
        for k in range(9):
            r = oracle.Rng(int(seeds[k]))
            p = r.permutation(14)
            t = r.tenures(2, 5, 50)
            w = oracle.tabu_run(f, d, p, 50, t)
            assert costs[k] == w[1] and np.array_equal(perms[k], w[0]) and steps[k] == w[6]
            assert np.array_equal(mi[k, : w[6]], w[7][0]) and np.array_equal(md[k, : w[6]], w[7][2])
    finally:
        di.close()
    f, d = _instance(3, 3, 11)
    di = DeviceInstance(f, d)
    try:
        perm = np.array([2, 0, 1], np.int64)
        ten = np.full(40, 1000, np.int64)
        g = di.tabu(perm, 40, ten)
        w = oracle.tabu_run(f, d, perm, 40, ten)
        _same_single(g, w, "n=3 long tenures")
    finally:
        di.close()


@pytest.mark.parametrize("n,kind", [(3, 3), (4, 0), (5, 3), (6, 4), (18, 3)])
def test_searches_of_one_warp_stop_at_different_iterations(built, n, kind):
    """Long tenures on tiny instances: every pair turns tabu and the searches run out of admissible moves after a
    different number of steps each -- at n <= 16 two searches share a warp and its reductions, so a stopped
    search must not disturb its partner (nor the clone that fills an odd batch)."""
    import oracle
    from paper_2307_11248_b200.backend import DeviceInstance

    f, d = _instance(n, kind, 900 + n)
    di = DeviceInstance(f, d)
    try:
        ten = (400, 400)
        for count in (1, 2, 9):
            got = di.multistart("tabu", 8, 0, count, 60, *ten)
            want = oracle.multistart(f, d, "tabu", 8, count, 60, tenure=ten, threads=1)
            assert np.array_equal(got[0], want[0]) and got[1] == want[1] and got[2] == want[2], (n, kind, count)
            assert np.array_equal(got[3], want[3]), (n, kind, count)
        seeds = np.array([oracle.derive_seed(8, k) for k in range(5)], np.uint64)
        costs, perms, steps, mi, mj, md = di.multistart_trace("tabu", seeds, 60, *ten)
        for k in range(5):
            r = oracle.Rng(int(seeds[k]))
            p = r.permutation(n)
            t = r.tenures(ten[0], ten[1], 60)
            w = oracle.tabu_run(f, d, p, 60, t)
            assert steps[k] == w[6] and costs[k] == w[1] and np.array_equal(mi[k, : w[6]], w[7][0]), (n, kind, k)
        assert n > 6 or int(steps.min()) < 60, "no search stopped early: the case does not exercise the inert path"
    finally:
        di.close()
