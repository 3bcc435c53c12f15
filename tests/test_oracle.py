"""Pin the CPU oracle: reference literal known answers, golden vectors produced by the
reference itself (tests/golden/make_golden.py), and -- when built -- the reference's own
compiled kernel in oracle/_ref.  CPU only."""
import glob
import hashlib
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def orc():
    import oracle

    oracle.build()
    return oracle


def golden(name):
    return np.load(os.path.join(HERE, "golden", f"golden_{name}.npz"))


def _instance(g):
    from paper_2307_11248_b200 import shapes

    inst = shapes.by_name(str(g["shape"]))
    assert hashlib.sha256(inst.flow.tobytes() + inst.distance.tobytes()).hexdigest() == str(g["sha256"])
    return inst


def test_rng_known_answers(orc):
    """SURVEY.md 8c (generated from the reference): SplitMix64/derive_seed/randbelow/shuffle."""
    r = orc.Rng(0)
    assert [r.next64() for _ in range(3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    assert [orc.derive_seed(0, k) for k in range(3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    assert orc.mix64(1) == 0x5692161D100B05E5
    assert orc.derive_seed(7, 5) == 0x3FDABE86CBBEAA11
    r = orc.Rng(5)
    assert [r.randbelow(10) for _ in range(5)] == [8, 4, 3, 9, 1]
    assert orc.Rng(orc.derive_seed(0, 0)).permutation(12).tolist() == [4, 10, 5, 9, 7, 6, 2, 11, 0, 1, 8, 3]


def test_tenure_table(orc):
    """test_tabu.py:13-18 literal table n -> [lo, hi]."""
    assert orc.tenure_bounds(30) == (3, 10)
    assert orc.tenure_bounds(100) == (10, 33)
    assert orc.tenure_bounds(12) == (1, 4)
    assert orc.tenure_bounds(256) == (25, 85)
    assert orc.tenure_bounds(2) == (1, 1)


def test_toy2_literals(orc):
    """conftest.py:12-18, test_core.py:31-33,55-56: costs 13 / 17, delta +4."""
    f = np.array([[0, 3], [2, 0]], np.int64)
    d = np.array([[0, 1], [5, 0]], np.int64)
    assert orc.full_cost(f, d, [0, 1]) == 13 and orc.full_cost(f, d, [1, 0]) == 17
    assert orc.all_deltas(f, d, [0, 1]).tolist() == [4]
    out = orc.tabu_run(f, d, np.array([0, 1]), 6, np.full(6, 3))
    assert out[5] is True and out[6] == 1  # premature stop (test_tabu.py:96-105)


def test_kat12(orc):
    """kat12 instance rows, start cost, first 2opt moves, final results."""
    f, d = orc.Rng(orc.derive_seed(1234, 0)).instance(12)
    assert f[0].tolist() == [0, 21, 93, 16, 79, 57, 99, 30, 76, 2, 56, 38]
    assert d[0].tolist() == [0, 85, 75, 19, 60, 96, 23, 86, 13, 62, 86, 53]
    rng = orc.Rng(3)
    p = rng.permutation(12)
    assert orc.full_cost(f, d, p) == 333188
    out = orc.two_opt_run(f, d, p, 48)
    moves = list(zip(out[4][:8].tolist(), out[5][:8].tolist(), out[6][:8].tolist()))
    assert moves == [(7, 8, -23626), (2, 5, -16046), (10, 11, -9480), (4, 6, -7191), (7, 9, -2339),
                     (1, 5, 688), (6, 7, -4985), (3, 6, -357)]
    assert out[1] == 265122 and out[0].tolist() == [0, 4, 7, 10, 1, 3, 2, 8, 6, 5, 9, 11]
    ten = rng.tenures(1, 4, 96)
    assert ten[:8].tolist() == [4, 1, 4, 1, 3, 3, 2, 1]
    t = orc.tabu_run(f, d, p, 96, ten)
    assert t[1] == 262131 and t[0].tolist() == [0, 4, 3, 5, 1, 7, 11, 10, 6, 2, 9, 8] and not t[5]


SINGLES = ["cfg0_nug12_2opt", "cfg0_nug12_tabu", "cfg1_tai30a_tabu", "cfg1_rand30_tabu",
           "cfg2_tai100a_single", "cfg3_tai256c_2opt", "cfg3_tai256c_tabu"]


@pytest.mark.parametrize("name", SINGLES)
def test_single_start_goldens(orc, name):
    g = golden(name)
    inst = _instance(g)
    n, iters, seed = inst.n, int(g["iters"]), int(g["seed"])
    if n > 200:
        iters = min(iters, 12)  # the O(n^3)-per-iteration oracle: keep the CPU suite short
    rng = orc.Rng(seed)
    start = rng.permutation(n)
    assert np.array_equal(start, g["start"])
    assert orc.full_cost(inst.flow, inst.distance, start) == int(g["start_cost"])
    assert np.array_equal(orc.all_deltas(inst.flow, inst.distance, start), g["start_deltas"])
    if str(g["algo"]) == "tabu":
        lo, hi = orc.tenure_bounds(n)
        ten = rng.tenures(lo, hi, int(g["iters"]))
        out = orc.tabu_run(inst.flow, inst.distance, start, iters, ten[:iters])
        k = out[6]
        assert np.array_equal(out[7][0], g["move_i"][:k]) and np.array_equal(out[7][1], g["move_j"][:k])
        assert np.array_equal(out[7][2], g["delta"][:k]) and np.array_equal(out[7][3], g["tabu_flag"][:k])
        assert np.array_equal(out[7][5], g["tenure"][:k])
        if iters == int(g["iters"]):
            assert out[1] == int(g["best_cost"]) and np.array_equal(out[0], g["best"])
            assert np.array_equal(out[4], g["final_tabu"]) and out[5] == bool(g["stopped_early"])
    else:
        out = orc.two_opt_run(inst.flow, inst.distance, start, iters)
        assert np.array_equal(out[4], g["move_i"][:iters]) and np.array_equal(out[6], g["delta"][:iters])
        if iters == int(g["iters"]):
            assert out[1] == int(g["best_cost"]) and np.array_equal(out[0], g["best"])
            assert out[3] == int(g["cur_cost"]) and np.array_equal(out[2], g["cur"])


@pytest.mark.parametrize("name,limit", [("kat30_multi_tabu", 64), ("kat30_multi_2opt", 64),
                                        ("cfg2_tai100a_multi", 3), ("cfg4_sko100_multi", 6),
                                        ("cfg4_tai150b_multi", 3), ("cfg4_tai150b_2opt_multi", 3)])
def test_multistart_goldens(orc, name, limit):
    """per_start_costs of the reference's run_multistart; `limit` starts are recomputed."""
    g = golden(name)
    inst = _instance(g)
    starts = min(limit, int(g["starts"]))
    costs, bc, bi, bp = orc.multistart(inst.flow, inst.distance, str(g["algo"]), int(g["master"]), starts,
                                       int(g["iters"]), threads=min(8, orc.max_threads()))
    assert np.array_equal(costs, g["per_start_costs"][:starts])
    if starts == int(g["starts"]):
        assert (bc, bi) == (int(g["best_cost"]), int(g["best_index"])) and np.array_equal(bp, g["best_perm"])


def test_survey_multistart_kat(orc):
    g = golden("kat30_multi_tabu")
    assert (int(g["best_cost"]), int(g["best_index"]), int(g["per_start_costs"].sum())) == (1776990, 23, 115222749)
    g = golden("kat30_multi_2opt")
    assert (int(g["best_cost"]), int(g["best_index"]), int(g["per_start_costs"].sum())) == (1809350, 36, 117877671)


def test_against_reference_compiled_kernel(orc):
    """When oracle/_ref holds the reference's own compiled kernel, compare directly
    (the pattern of the reference's tests/test_backends.py:24-63)."""
    ref = orc.load_ref_kernels()
    if ref is None:
        pytest.skip("oracle/_ref not built (reference sources absent)")
    rs = np.random.default_rng(0)
    for n in (2, 5, 12, 23):
        f = rs.integers(-30, 99, (n, n)).astype(np.int64)
        d = rs.integers(-30, 99, (n, n)).astype(np.int64)
        rng = orc.Rng(1000 + n)
        p = rng.permutation(n)
        ten = rng.tenures(*orc.tenure_bounds(n), 50)
        assert orc.full_cost(f, d, p) == ref.full_cost(f, d, p)
        assert np.array_equal(orc.all_deltas(f, d, p), ref.all_deltas(f, d, p))
        for a, b in zip(orc.two_opt_run(f, d, p, 30), ref.two_opt_run(f, d, p, 30)):
            assert np.array_equal(a, b)
        a, b = orc.tabu_run(f, d, p, 50, ten), ref.tabu_run(f, d, p, 50, ten)
        for x, y in zip(a[:7], b[:7]):
            assert np.array_equal(x, y)
        for x, y in zip(a[7], b[7]):
            assert np.array_equal(x, y)


def test_golden_files_present():
    assert len(glob.glob(os.path.join(HERE, "golden", "golden_*.npz"))) >= 13
