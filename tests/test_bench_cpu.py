"""bench.py's contract pieces that run without a GPU: the reference arm
(the oracle port on the host cores) prints one JSON line with the same
config as our arm, N simulated ranks for --gpus N, and the driver's keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                       timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1 and lines[0].startswith("{"), r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_same_config_and_keys():
    d = _run("--impl", "reference", "--config", "tiny", "--gpus", "2", "--steps", "1", "--warmup", "1")
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    for k in ("metric", "value", "unit", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in d
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert "2 simulated rank" in d["cpu_baseline"]["sample"]
    assert d["cpu_baseline"]["host"]["cpu_count"] == os.cpu_count()
    sys.path.insert(0, ROOT)
    import bench
    argv, sys.argv = sys.argv, ["bench.py", "--config", "tiny", "--gpus", "2"]
    try:
        ours = bench.step_config(bench.parse(), 2)
    finally:
        sys.argv = argv
    assert ours == d["config"]
