"""CLI (the reference's cli.py run/verify/dump-plan, driving the GPU runtime)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cli(*args, timeout=600):
    return subprocess.run([sys.executable, "-m", "paper_2304_11277_b200", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=timeout)


def test_dump_plan_matches_reference_golden(golden):
    _, meta = golden
    for f in ("1", "2", "8"):
        r = _cli("dump-plan", "--model", "tiny", "--shard-factor", f)
        assert r.returncode == 0, r.stderr
        assert r.stdout.strip().splitlines() == meta["tiny_gpt"][f]["dump"]


@pytest.mark.gpu
def test_run_and_verify_world1():
    r = _cli("run", "--model", "tiny", "--steps", "2", "--micro", "2")
    assert r.returncode == 0, r.stderr[-3000:]
    recs = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert [x["step"] for x in recs] == [0, 1] and all(x["loss"] > 0 for x in recs)
    v = _cli("verify", "--steps", "2")
    assert v.returncode == 0, v.stdout + v.stderr[-3000:]
    assert json.loads(v.stdout.strip().splitlines()[-1])["verify"] == "PASS"
