"""bench.py contract (CPU part): the reference arm runs the reference's own compiled kernel (or the C
port) on the host cores and prints ONE JSON line with the keys the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line(built):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0", "--no-time-to-gap"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "swap_move_evals_per_sec" and d["unit"] == "evals/s"
    assert d["higher_is_better"] is True and d["value"] > 1e6 and d["steps"] == 1
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"] == d["e2e"]["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "tai100a" in d["config"]["workload"]


def test_survey_ops_model():
    """n = 100 -> 46.9 int-ops per eval for the incremental evaluator, 796 for the full one."""
    sys.path.insert(0, ROOT)
    import bench

    assert abs(bench.survey_ops_per_eval(100) - 46.88) < 0.01
    assert 8 * (100 - 2) + 12 == 796


def test_gpus_n_spawns_n_ranks():
    """`python bench.py --gpus 2` outside torchrun re-launches itself with two ranks (checked on CPU with the
    launch-plumbing-only flag: gloo, no CUDA)."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--spawn-check"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d == {"spawned": 2, "n_gpus": 2, "rank_sum": 3}


def test_gpus_mismatch_is_refused():
    """A rank count that differs from --gpus is an error, not a silent one-rank run."""
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1", MASTER_PORT="29999")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"], capture_output=True, text=True,
                         timeout=300, cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE=1" in (out.stderr + out.stdout)


def test_time_to_gap_ladder_fixture():
    with open(os.path.join(ROOT, "tests", "golden", "time_to_gap_tai100a.json")) as fh:
        d = json.load(fh)
    gaps = [r["gap_pct"] for r in d["runs"]]
    assert gaps == sorted(gaps, reverse=True) and gaps[-1] == 0.0 and d["starts"] == 1024
