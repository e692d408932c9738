"""bench.py's multi-GPU path driven end to end on CPU: `bench.py --gpus 2` spawns its own two
ranks (torch.distributed.run, gloo in --dry-run), deals the tenant set with
sharding.shard_streams, runs each shard through the native serving loop (decisions only) and
checks every shard's completion times against the oracle engine on that sub-workload
(SURVEY §8(e)); rank 0 prints whole-box numbers."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], capture_output=True,
                         text=True, timeout=300, env=env, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_spawns_two_ranks_weak_scaling():
    line = _run("--gpus", "2", "--dry-run", "--steps", "4", "--warmup", "3")
    assert line["n_gpus"] == 2 and line["scaling"] == "weak" and line["tenants"] == 32
    assert line["comm"]["backend"] == "gloo"
    assert line["shard_parity"] is True
    shards = [r["tenants"] for r in sorted(line["ranks"], key=lambda r: r["rank"])]
    assert shards[0] == [f"t{i:02d}" for i in range(0, 32, 2)]
    assert shards[1] == [f"t{i:02d}" for i in range(1, 32, 2)]
    # whole-box value = sum of the ranks' work over the slowest rank's time
    want = sum(r["flops"] for r in line["ranks"]) / max(r["host_seconds"] for r in line["ranks"]) / 1e12
    assert abs(line["value"] - want) <= 1e-6 * max(1.0, want)


def test_bench_partitions_a_fixed_tenant_set():
    line = _run("--gpus", "2", "--dry-run", "--steps", "2", "--warmup", "3", "--tenants", "48")
    assert line["scaling"] == "strong" and line["tenants"] == 48
    assert line["shard_parity"] is True
    got = sorted(t for r in line["ranks"] for t in r["tenants"])
    assert got == [f"t{i:02d}" for i in range(48)]
    assert all(len(r["tenants"]) == 24 for r in line["ranks"])


def test_rank_core_pools_are_disjoint():
    """Node-local ranks pin their serving loops to disjoint cores (bench.pin_serving_thread)."""
    import bench
    pool = list(range(1, 16))
    for lw in (1, 2, 4, 8):
        pools = [set(bench.rank_core_pool(pool, r, lw)) for r in range(lw)]
        assert set().union(*pools) == set(pool)
        for i in range(lw):
            assert pools[i]
            for j in range(i):
                assert not pools[i] & pools[j]
