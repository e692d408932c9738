"""Multi-GPU path on CPU: tenant sharding with world_size-2 gloo process groups.

Each rank runs the native Scheduler over its tenant shard through the
restated engine loop; every shard's trace must equal the oracle engine run
alone on that sub-workload (per-shard parity), the shards must partition the
requests, and the whole-job throughput reduction is sum(work) / max(time).
"""

import json
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1901_10008_b200 import sharding

from .conftest import GOLDEN, REPO


def test_shard_streams_partition_round_robin():
    shards = sharding.shard_streams([f"s{i}" for i in (5, 1, 3, 0, 4, 2)], 4)
    assert shards == [["s0", "s4"], ["s1", "s5"], ["s2"], ["s3"]]
    assert sorted(sum(shards, [])) == [f"s{i}" for i in range(6)]
    with pytest.raises(ValueError):
        sharding.shard_streams(["a"], 0)


def test_whole_job_throughput_is_sum_over_max():
    assert sharding.whole_job_throughput([10.0, 30.0], [1.0, 2.0]) == 20.0
    assert sharding.whole_job_throughput([1.0], [0.0]) == 0.0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import hashlib

        from oracle import decisions as od
        from oracle import sim
        from tests.test_core_parity import product_factory

        with open(os.path.join(GOLDEN, "traces.json")) as fh:
            traces = json.load(fh)
        with open(os.path.join(GOLDEN, "models.json")) as fh:
            lib = json.load(fh)
        with open(os.path.join(GOLDEN, "profiles.json")) as fh:
            prof = od.Prof(**json.load(fh)["b200"])
        wl = traces["workloads"]["c4_poisson64"]
        sub = sharding.shard_workload(wl, rank, world)
        trace, metrics, _, _ = sim.simulate(sub, lib, prof, "ooo", factory=product_factory)
        ref_trace, ref_metrics, _, _ = sim.simulate(sub, lib, prof, "ooo")
        g = json.loads(metrics)["global"]
        stats = {"rank": rank, "streams": [s["stream_id"] for s in sub["streams"]],
                 "parity": trace == ref_trace and metrics == ref_metrics,
                 "requests": g["requests"], "completed": g["completed"],
                 "useful": g["throughput_flops"] * 1.0,
                 "trace_sha": hashlib.sha256(trace.encode()).hexdigest()}
        gathered = sharding.gather_rank_stats(stats)
        if rank == 0:
            with open(os.path.join(out_dir, "gathered.json"), "w") as fh:
                json.dump(gathered, fh)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_shards_match_reference_engine(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    gathered = json.loads((tmp_path / "gathered.json").read_text())
    assert [g["rank"] for g in gathered] == [0, 1]
    assert all(g["parity"] for g in gathered)
    streams = sum((g["streams"] for g in gathered), [])
    assert len(streams) == len(set(streams)) == 64
    with open(os.path.join(GOLDEN, "traces.json")) as fh:
        wl = json.load(fh)["workloads"]["c4_poisson64"]
    assert sorted(streams) == sorted(s["stream_id"] for s in wl["streams"])
    from oracle import sim
    with open(os.path.join(GOLDEN, "models.json")) as fh:
        lib = json.load(fh)
    assert sum(g["requests"] for g in gathered) == len(sim.materialize(wl, lib, 0))
    assert all(g["completed"] > 0 for g in gathered)
