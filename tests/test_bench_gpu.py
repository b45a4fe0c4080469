"""bench.py's multi-rank path on whatever GPUs the box has (ranks share a GPU
when there are fewer GPUs than ranks): the self-launch, the one JSON line,
and the size-independent replica property of HYBRID_SHARD (ranks r, r + F
end bit-identical in master and Adam state, collectives.py:63-72, :377-397)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("world,F", [(4, 2), (2, 1)])
def test_bench_hybrid_replicas(world, F):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    strategy = ["--strategy", "HYBRID_SHARD", "--hybrid-shard-size", str(F)] if F > 1 else \
        ["--strategy", "NO_SHARD"]
    r = subprocess.run([sys.executable, "bench.py", "--gpus", str(world), "--config", "tiny", "--micro", "1",
                        *strategy, "--steps", "2", "--warmup", "3", "--no-exposed", "--no-cpu-baseline",
                        "--check-replicas"], cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == world and d["gpu_launches"] > 0
    rc = d["replica_check"]
    assert rc["identical_within_groups"], rc
    assert len(rc["replica_groups"]) == F and all(len(g) == world // F for g in rc["replica_groups"])
    if F > 1:
        assert rc["shards_differ_across_positions"], rc
