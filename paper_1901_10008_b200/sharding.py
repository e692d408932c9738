"""Tenant sharding across GPUs: replicas of the scheduler, no hot-path collective.

Tenants (streams) are independent and the reference scheduler is per device
("No cross-GPU scheduling"), so G GPUs run G independent
Scheduler+executor replicas over disjoint tenant shards. Streams are sorted
and dealt round-robin; each shard's decisions equal the reference engine run
on that sub-workload (the per-shard `tenancy`, scheduler.py:418, is the
shard's). The only collectives are end-of-run gathers of small per-rank
numbers (torch.distributed: NCCL on GPUs, gloo in CPU tests).
"""

from __future__ import annotations

import copy


def shard_streams(stream_ids, world_size: int) -> list:
    """Sorted stream ids dealt round-robin into `world_size` shards."""
    if world_size < 1:
        raise ValueError("world_size must be >= 1")
    ordered = sorted(stream_ids)
    return [ordered[r::world_size] for r in range(world_size)]


def shard_workload(workload: dict, rank: int, world_size: int) -> dict:
    """The sub-workload (reference JSON workload format) of one rank."""
    mine = set(shard_streams([s["stream_id"] for s in workload["streams"]], world_size)[rank])
    sub = copy.deepcopy(workload)
    sub["streams"] = [s for s in sub["streams"] if s["stream_id"] in mine]
    return sub


def whole_job_throughput(useful_flops_per_rank, seconds_per_rank) -> float:
    """Whole-box throughput: all ranks' useful FLOPs over the slowest rank's time."""
    t = max(seconds_per_rank)
    return sum(useful_flops_per_rank) / t if t > 0 else 0.0


def gather_rank_stats(stats: dict, group=None) -> list:
    """all_gather_object of a small per-rank dict (after the run; never on the hot path)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return [stats]
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, stats, group=group)
    return out
