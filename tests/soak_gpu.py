"""Randomised differential soak: GPU multistart / tabu_run / two_opt_run vs the C oracle on random
instances (sizes, value ranges, symmetry, diagonals), every launch plan of each instance.
Usage: python tests/soak_gpu.py [seconds] [seed]   (development aid; the oracle is the checker)
SOAK_SMALL=1 restricts the sizes to n = 2 .. 32 (the one-warp-per-search kernel) with batches of up to 70 starts."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np
import __graft_entry__ as e
e.build()
import oracle
import paper_2307_11248_b200 as q
from paper_2307_11248_b200.backend import DeviceInstance

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rs = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
t0 = time.time(); cases = 0; plans_run = 0
while time.time() - t0 < budget:
    n = int(rs.choice([2, 3, 4, 5, 7, 8, 9, 12, 16, 17, 23, 31, 32, 33, 40, 48, 63, 64, 65, 80, 100, 129, 140]))
    small = os.environ.get("SOAK_SMALL") == "1"
    if small:
        n = int(rs.integers(2, 33))
    hi = int(rs.choice([2, 10, 100, 1000, 40000, 3000000]))
    lo = -hi if rs.random() < 0.2 else 0
    f = rs.integers(lo, hi + 1, (n, n)).astype(np.int64)
    d = rs.integers(0, hi + 1, (n, n)).astype(np.int64)
    kind = rs.integers(0, 4)
    if kind in (1, 3): d = d + d.T
    if kind in (2, 3): f = f + f.T
    if rs.random() < 0.5:
        np.fill_diagonal(f, 0); np.fill_diagonal(d, 0)
    if rs.random() < 0.3:
        f[rs.random((n, n)) < 0.6] = 0
    iters = int(rs.integers(1, 3 * n + 8)) if n <= 64 else int(rs.integers(1, 40))
    if n <= 33 and rs.random() < 0.08:
        iters = int(rs.integers(250, 700))  # across the 256-iteration tenure chunk boundaries
    starts = int(rs.integers(1, 71 if small else 7))
    algo = "tabu" if rs.random() < 0.7 else "2opt"
    master = int(rs.integers(0, 2**62))
    lo_t, hi_t = oracle.tenure_bounds(n)
    if rs.random() < 0.3:
        lo_t, hi_t = 1, int(rs.integers(1, 4))  # short tenures: frequent expiries and early stops
    want = oracle.multistart(f, d, algo, master, starts, iters, threads=oracle.max_threads()) if (lo_t, hi_t) == oracle.tenure_bounds(n) else None
    di = DeviceInstance(f, d)
    try:
        plans = di.plan_candidates() or [None]
        for plan in plans:
            if plan is not None:
                di.set_plan(plan)
            if want is not None:
                got = di.multistart(algo, master, 0, starts, iters, lo_t, hi_t)
                assert np.array_equal(got[0], want[0]) and got[1:3] == (want[1], want[2]) and np.array_equal(got[3], want[3]), (n, hi, kind, algo, plan, "multistart")
            # host-drawn single start with explicit tenures (any tenure interval)
            rng = oracle.Rng(oracle.derive_seed(master, 0))
            perm = rng.permutation(n)
            ten = rng.tenures(lo_t, hi_t, iters)
            if algo == "tabu":
                g = di.tabu(perm, iters, ten)
                w = oracle.tabu_run(f, d, perm, iters, ten)
                ok = np.array_equal(g[0][0], w[0]) and g[1][0] == w[1] and np.array_equal(g[2][0], w[2]) and g[3][0] == w[3] \
                    and np.array_equal(g[4][0], w[4]) and bool(g[5][0]) == w[5] and g[6][0] == w[6] \
                    and all(np.array_equal(g[7][a][0, : w[6]], w[7][a]) for a in range(4))
            else:
                g = di.two_opt(perm, iters)
                w = oracle.two_opt_run(f, d, perm, iters)
                ok = all(np.array_equal(a[0], b) for a, b in zip(g, w))
            assert ok, (n, hi, kind, algo, plan, "single")
            plans_run += 1
    finally:
        di.close()
    cases += 1
print(f"soak ok: {cases} instances, {plans_run} (instance, plan) runs in {time.time() - t0:.0f} s")
