"""GPU vs golden vectors produced by the reference itself (tests/golden/make_golden.py),
at the full iteration counts of the BASELINE.json configurations, plus size-independent
properties at sizes the CPU oracle cannot reach in seconds."""
import hashlib
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
from paper_2307_11248_b200._refpkg import reference as _reference  # noqa: E402

HAVE_REFERENCE = _reference() is not None


@pytest.fixture(scope="module")
def q(built):
    import paper_2307_11248_b200 as pkg

    return pkg


def golden(name):
    return np.load(os.path.join(HERE, "golden", f"golden_{name}.npz"))


def _instance(g):
    from paper_2307_11248_b200 import shapes

    inst = shapes.by_name(str(g["shape"]))
    assert hashlib.sha256(inst.flow.tobytes() + inst.distance.tobytes()).hexdigest() == str(g["sha256"])
    return inst


@pytest.mark.parametrize("name", ["cfg0_nug12_2opt", "cfg0_nug12_tabu", "cfg1_tai30a_tabu", "cfg1_rand30_tabu",
                                  "cfg2_tai100a_single", "cfg3_tai256c_2opt", "cfg3_tai256c_tabu",
                                  # full length: the iteration counts bench.py times, from the reference's kernel
                                  "full_cfg2_tai100a_tabu", "full_cfg4_tai150b_tabu", "full_cfg4_sko100_tabu",
                                  "full_cfg3_tai256c_2opt", "full_cfg3_tai256c_tabu"])
def test_single_start_trajectories(q, name):
    """Drivers run_two_opt / run_tabu (host RNG -> kernel) against the reference's per-iteration
    trajectory: moves, deltas, tabu flags, tenures, final tabu matrix, best permutation."""
    g = golden(name)
    inst = _instance(g)
    seed, iters = int(g["seed"]), int(g["iters"])
    start = q.random_permutation(inst.n, q.SplitMix64(seed))
    assert np.array_equal(start, g["start"])
    assert q.full_cost(inst, start) == int(g["start_cost"])
    assert np.array_equal(q.all_deltas(inst, start), g["start_deltas"])
    if str(g["algo"]) == "tabu":
        rec, trail = q.run_tabu(inst, seed, iters)
        assert rec.cost == int(g["best_cost"]) and np.array_equal(rec.permutation, g["best"])
        assert rec.seed == seed and rec.algorithm == "tabu"
        assert np.array_equal(trail.move_i, g["move_i"]) and np.array_equal(trail.move_j, g["move_j"])
        assert np.array_equal(trail.delta, g["delta"]) and np.array_equal(trail.tabu_flag, g["tabu_flag"])
        assert np.array_equal(trail.aspirated_flag, g["tabu_flag"]) and np.array_equal(trail.tenure_drawn, g["tenure"])
        assert np.array_equal(trail.final_tabu, g["final_tabu"]) and trail.stopped_early == bool(g["stopped_early"])
        if HAVE_REFERENCE:  # the reference's own auditor (tabu.py:236-283), unchanged, accepts the GPU trail
            assert q.replay_and_audit(inst, trail).cost == rec.cost
    else:
        rec = q.run_two_opt(inst, seed, iters)
        assert rec.cost == int(g["best_cost"]) and np.array_equal(rec.permutation, g["best"])
        out = q.kernels.two_opt_run(inst.flow, inst.distance, start, iters)
        assert np.array_equal(out[2], g["cur"]) and out[3] == int(g["cur_cost"])
        assert np.array_equal(out[4], g["move_i"]) and np.array_equal(out[5], g["move_j"]) and np.array_equal(out[6], g["delta"])


@pytest.mark.parametrize("name", ["kat30_multi_tabu", "kat30_multi_2opt", "cfg2_tai100a_multi", "cfg4_sko100_multi",
                                  "cfg4_tai150b_multi", "cfg4_tai150b_2opt_multi", "full_cfg4_tai150b_multi6"])
def test_multistart_results(q, name):
    g = golden(name)
    inst = _instance(g)
    cfg = q.SearchConfig(algorithm=str(g["algo"]), n_starts=int(g["starts"]), iterations=int(g["iters"]),
                         master_seed=int(g["master"]))
    res = q.run_multistart(inst, cfg)
    assert np.array_equal(res.per_start_costs, g["per_start_costs"])
    assert res.best.cost == int(g["best_cost"]) and res.best_start_index == int(g["best_index"])
    assert np.array_equal(res.best.permutation, g["best_perm"]) and res.best.seed == int(g["best_seed"])
    assert res.config_digest == str(g["digest"])
    # run_start (single-start kernel entries, host RNG) agrees with the batched device-RNG path
    for idx in (0, int(g["best_index"])):
        assert q.run_start(inst, cfg, idx).cost == int(g["per_start_costs"][idx])


def test_stepwise_references_agree(q):
    """Kernel runs == step-wise host references (test_two_opt.py:79-87, test_tabu.py:130-145)."""
    from paper_2307_11248_b200 import shapes, tabu, two_opt

    inst = shapes.rand(12, 77)
    start = q.random_permutation(12, q.SplitMix64(4))
    st = two_opt.initial_state(inst, start)
    for _ in range(20):
        st = q.two_opt_step(inst, st)
    out = q.kernels.two_opt_run(inst.flow, inst.distance, start, 20)
    assert np.array_equal(out[0], st.best) and out[1] == st.best_cost and np.array_equal(out[2], st.current)
    rng = q.SplitMix64(4)
    start = q.random_permutation(12, rng)
    state, rng2 = tabu.initial_tabu_state(inst, start), q.SplitMix64(rng.state)
    for _ in range(30):
        state = q.tabu_step(inst, state, rng2)
    rec, trail = q.run_tabu(inst, 4, 30)
    assert rec.cost == state.best_cost and np.array_equal(rec.permutation, state.best)
    assert np.array_equal(trail.final_tabu, state.tabu)


@pytest.mark.parametrize("shape,algo,starts,iters", [("tai100a", "tabu", 1024, 800), ("tai256c", "tabu", 64, 512),
                                                     ("tai256c", "2opt", 32, 256), ("tai150b", "tabu", 128, 400),
                                                     ("sko100", "2opt", 512, 400)])
def test_full_size_properties(q, shape, algo, starts, iters):
    """BASELINE.json full sizes (beyond what the O(n^3)/iteration oracle can check in seconds):
    every reported best cost equals an independent recompute of the returned permutation, the
    winner is the (cost, index) minimum, results are idempotent across launches, and a start
    run alone through the single-start entry reproduces its batched cost."""
    from paper_2307_11248_b200 import shapes
    from paper_2307_11248_b200.backend import device_instance

    inst = shapes.by_name(shape)
    cfg = q.SearchConfig(algorithm=algo, n_starts=starts, iterations=iters, master_seed=42)
    res = q.run_multistart(inst, cfg)
    again = q.run_multistart(inst, cfg)
    assert np.array_equal(res.per_start_costs, again.per_start_costs) and res.best.cost == again.best.cost
    k = int(np.argmin(res.per_start_costs))
    assert res.best_start_index == k and res.best.cost == int(res.per_start_costs[k])
    assert sorted(res.best.permutation.tolist()) == list(range(inst.n))
    assert q.evaluate_cost(inst, res.best.permutation) == res.best.cost
    for idx in (0, starts - 1):
        assert q.run_start(inst, cfg, idx).cost == int(res.per_start_costs[idx])
    # trajectory self-consistency on one start: cost + sum(deltas) == recomputed current cost
    rng = q.SplitMix64(q.derive_seed(42, 1))
    start = q.random_permutation(inst.n, rng)
    di = device_instance(inst.flow, inst.distance)
    if algo == "tabu":
        t = q.tenure_bounds(inst.n)
        ten = np.array([rng.randint(t.low, t.high) for _ in range(iters)], np.int64)
        best, bc, cur, cc, cells, stop, steps, tr, _ = di.tabu(start, iters, ten)
        deltas = tr[2][0, : int(steps[0])]
    else:
        best, bc, cur, cc, mi, mj, md = di.two_opt(start, iters)
        deltas = md[0]
    c0 = q.evaluate_cost(inst, start)
    assert c0 + int(deltas.sum()) == int(cc[0]) == q.evaluate_cost(inst, cur[0])
    if algo == "tabu" and inst.n <= 150:
        # the solve command's --trail flow (cli.py:99-103, criterion 6 of test_acceptance.py:157-175): re-run
        # the winning start with its trail and let the host auditor replay every move of it
        rec, trail = q.run_tabu(inst, q.SplitMix64(q.derive_seed(42, k)), iters)
        assert rec.cost == res.best.cost and np.array_equal(rec.permutation, res.best.permutation)
        if HAVE_REFERENCE:
            audited = q.replay_and_audit(inst, trail)
            assert audited.cost == rec.cost and np.array_equal(audited.permutation, rec.permutation)
    assert int(bc[0]) == q.evaluate_cost(inst, best[0]) == c0 + int(np.minimum.accumulate(np.concatenate([[0], np.cumsum(deltas)])).min())
