"""Split-K granularity vs (a) a lone C2 step (CUDA events around one launch, device idle
around it), (b) a held resident batch (steps back to back), (c) the live-fed resident serving
loop over K rounds (bench.py's timed region). Prints one JSON line per setting."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

settings = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "400,200,100,70,50").split(",")]
b = bench.C2Bench(16)
s = b.stream
r = 0
for pct in settings:
    b.ex.set_option("split_pct", pct)
    b.ex.clear_plans()
    for j in range(32):
        b.ex.launch(b.slots[j % 16], s)
    torch.cuda.synchronize()
    ts = []
    for j in range(48):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        b.ex.launch(b.slots[j % 16], s)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    plan = b.ex.last_plan()
    held, held_gt, _ = bench.time_resident(b, 1000)
    live = {}
    for K in (20, 200):
        for _ in range(2):   # warm this setting's plans in the runtime path
            for _ in range(16):
                b.queue_round(r)
                r += 1
            b.ex.resident_begin(s)
            b.run_rounds(r - 16, 16)
            b.ex.resident_end()
            torch.cuda.synchronize()
        for _ in range(K):
            b.queue_round(r)
            r += 1
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        b.ex.resident_begin(s)
        b.run_rounds(r - K, K)
        b.ex.resident_end()
        e1.record(s)
        torch.cuda.synchronize()
        live[K] = round(e0.elapsed_time(e1) * 1e3 / K, 3)
    print(json.dumps({"split_pct": pct, "lone_median_us": round(statistics.median(ts), 2),
                      "lone_min_us": round(min(ts), 2), "held_us_per_step": round(held * 1e6, 3),
                      "live_us_per_round": live, "splits": plan["n_split_items"], "items": plan["n_items"],
                      "max_cta": round(plan["max_cta_cost"]), "mean_cta": round(plan["mean_cta_cost"])}), flush=True)
