"""Hardware autotuner: a MEASURED replacement for the reference's analytical
`tune` grid (gpumux/tuning.py:90-135) that writes the same TuningTable JSON
(tuning.py:162-191), so the reference scheduler, this package's scheduler and the executor all
consume it.

For every cluster key K and co-tenancy t in 1..T, t identical members of K (one per tenant)
are registered on the executor and run as ONE coalesced step for each candidate output tile
(UMMA M = 128 rows; UMMA N in {64, 128}); the step's mean device time is measured over a CUDA
graph of back-to-back launches rotating over operand replicas. The stored entry for (K, t) is
the candidate with the best aggregate throughput at that tenancy — at t = 1 the solo ("greedy")
best, at t > 1 the tile that serves t co-running tenants best, which can differ (the paper's
collaborative choice, PAPER.md 358-380):

  tile_m = 128, tile_n = chosen UMMA N
      the executor uses tile_n as the problem's tile (gmx_problem_desc.tile_n), and the decision
      model's block_count (kernels.py:202-213) then counts the real output tiles;
  sm_footprint = CTAs the step's plan occupied / #SMs;
  efficiency_factor = the factor f in (0, 1] for which the reference cost model
      (device.py:130-150: eff = min(1, blocks / capacity) * f, duration = max(compute, bytes))
      predicts the measured time wherever the compute term can reach it, i.e.
      f = min(1, t * flops / (peak * occupancy * T_measured)); if even f = 1 keeps the byte term
      above the measurement, f = 1.

GEMV / elementwise keys have no tile choice: they get the reference default tiles and the
measured factor.
"""

from __future__ import annotations


import time

import torch

from .device import DeviceProfile
from .kernels import block_count, bytes_moved, flop_count
from .tuning import ClusterKey, TuningConfig, TuningTable

UMMA_M = 128
TILE_N_CANDIDATES = (64, 128)


def _time_step(ex, slot_sets, launches=48):
    """Mean device seconds of one coalesced launch (CUDA graph, events on its stream)."""
    s = torch.cuda.Stream(device=ex.device)
    with torch.cuda.stream(s):
        for sl in slot_sets:   # plans built + uploaded outside the graph
            ex.launch(sl, s, independent=True)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for j in range(launches):
                ex.launch(slot_sets[j % len(slot_sets)], s, independent=True)
        g.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
        s.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / (reps * launches)


def measure(ex, key: ClusterKey, tenancy: int, tile_n: int = 0, replicas: int = 3, seed: int = 0):
    """(seconds per coalesced step of `tenancy` members of `key`, CTAs used) on executor `ex`."""
    from .executor import OperandSet
    sets = []
    for r in range(replicas):
        row = []
        for t in range(tenancy):
            o = OperandSet(key.op_kind, key.dims, dtype=key.dtype, seed=seed + 97 * r + t, on_device=True)
            row.append((o, o.register(ex, tile_n=tile_n) if key.op_kind == "gemm" else o.register(ex)))
        sets.append(row)
    try:
        sec = _time_step(ex, [[sl for _, sl in row] for row in sets])
        grid = ex.last_plan()["grid"]
    finally:
        for row in sets:
            for _, sl in row:
                ex.unregister(sl)
    return sec, grid


def calibrated_factor(key: ClusterKey, tenancy: int, tile_m: int, tile_n: int, seconds: float,
                      profile: DeviceProfile) -> float:
    """efficiency_factor for which the reference cost model predicts `seconds` (see module doc)."""
    flops = tenancy * flop_count(key.op_kind, key.dims)
    blocks = tenancy * block_count(key.op_kind, key.dims, tile_m, tile_n)
    occupancy = min(1.0, blocks / profile.block_capacity)
    peak = profile.peak("dense" if key.dtype == "fp16" else "scalar")
    f = flops / (peak * occupancy * seconds) if seconds > 0 else 1.0
    return float(min(1.0, max(f, 1e-6)))


def autotune(ex, keys, max_tenancy: int, profile: DeviceProfile, log=None) -> TuningTable:
    """Measure every key at tenancy 1..max_tenancy; return the table (with provenance)."""
    table = TuningTable(provenance={
        "tuner": "measured (paper_1901_10008_b200.autotune)", "device": torch.cuda.get_device_name(ex.device),
        "profile": profile.name, "max_tenancy": max_tenancy, "tile_m": UMMA_M,
        "tile_n_candidates": list(TILE_N_CANDIDATES), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
        "measurements": {},
    })
    for key in keys:
        for t in range(1, max_tenancy + 1):
            cands = TILE_N_CANDIDATES if key.op_kind == "gemm" else (0,)
            results = []
            for tn in cands:
                sec, grid = measure(ex, key, t, tn)
                results.append((sec, tn, grid))
                if log:
                    log(f"{key.as_string()} t={t} tile_n={tn}: {sec * 1e6:.2f} us (grid {grid})")
            sec, tn, grid = min(results)
            if key.op_kind == "gemm":
                tile_m, tile_n = UMMA_M, tn
            else:
                tile_m, tile_n = 64, 64   # DEFAULT_CONFIG tiles (tuning.py:48-49)
            cfg = TuningConfig(tile_m=tile_m, tile_n=tile_n,
                               sm_footprint=min(1.0, max(grid, 1) / ex.num_sms),
                               efficiency_factor=calibrated_factor(key, t, tile_m, tile_n, sec, profile))
            table.put(key, t, cfg)
            table.provenance["measurements"][f"{key.as_string()}@{t}"] = {
                "us": {str(tn_): round(s_ * 1e6, 3) for s_, tn_, _ in results},
                "aggregate_gbps": round(t * bytes_moved(key.op_kind, key.dims, key.dtype) / sec / 1e9, 1),
            }
    return table


def tile_n_for(table: TuningTable, key: ClusterKey, tenancy: int = 1) -> int:
    """Executor tile for a member of `key` per a measured table (0 = automatic)."""
    cfg = table.lookup(key, tenancy)
    if cfg is None or key.op_kind != "gemm" or cfg.tile_n not in TILE_N_CANDIDATES:
        return 0
    return cfg.tile_n


__all__ = ["autotune", "measure", "calibrated_factor", "tile_n_for", "TILE_N_CANDIDATES", "UMMA_M"]

