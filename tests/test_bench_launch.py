"""bench.py --gpus N started as a plain process re-launches itself under
torchrun with N ranks: checked on CPU with the gloo backend
through the kernel-free `launchcheck` workload."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True,
                       text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_gpus2_spawns_two_ranks():
    out = _run(["--gpus", "2", "--workload", "launchcheck"], {"MIMW_BENCH_BACKEND": "gloo"})
    assert out["n_gpus"] == 2
    assert out["rank_sum"] == 1  # ranks 0 + 1 met in the collective
    assert out["backend"] == "gloo"


def test_gpus1_runs_in_process():
    out = _run(["--gpus", "1", "--workload", "launchcheck"])
    assert out["n_gpus"] == 1


def test_world_size_mismatch_is_an_error():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload",
                        "launchcheck"], capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert r.returncode != 0
    assert "WORLD_SIZE" in (r.stderr + r.stdout)
