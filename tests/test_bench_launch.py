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


def test_reference_arm_runs_requested_steps(monkeypatch, capsys):
    """`bench.py --impl reference` times exactly --steps bounded samples after
    --warmup untimed ones and reports both (the driver's reference arm); the
    samplers are stubbed, so no oracle work runs here."""
    sys.path.insert(0, ROOT)
    import bench
    calls = []

    def fake_gemm(seconds_target=12.0, single=True):
        calls.append((seconds_target, single))
        return {"value": 1e-3 * len(calls), "unit": "TFLOPS", "cores": 2, "kind": "reference",
                "sample": "stub"}

    monkeypatch.setattr(bench, "cpu_gemm_sample", fake_gemm)
    monkeypatch.setattr(bench, "cpu_attention_sample",
                        lambda *a, **k: {"value": 2e-3, "unit": "TFLOPS", "cores": 2, "kind": "reference"})
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--steps", "7", "--warmup", "4"])
    monkeypatch.delenv("RANK", raising=False)
    bench.main()
    out = json.loads([ln for ln in capsys.readouterr().out.splitlines() if ln.startswith("{")][-1])
    assert out["impl"] == "reference" and out["steps"] == 7 and out["warmup"] == 4
    assert len(calls) == 11 and sum(single for _, single in calls) == 1  # one single-thread probe
    assert all(1.0 <= t <= 12.0 for t, _ in calls)
    assert out["value"] == out["cpu_baseline"]["value"] == out["e2e"]["value"]
    assert out["e2e"]["h2d_bytes_per_step"] == 0 and out["e2e"]["d2h_bytes_per_step"] == 0
    assert abs(out["value"] - 1e-3 * 8) < 1e-12  # median of the 7 timed samples (5..11)
