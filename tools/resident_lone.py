"""Latency of ONE C2 step entering an idle resident kernel (the first step of a serving burst):
host publish -> completion flag observed by the host, per split_pct_idle setting (0 = the
resident throughput plan). The plan is built and uploaded before timing; each setting runs its
own residencies. Also: a held batch per setting (throughput plans are unchanged by the option).
usage: python tools/resident_lone.py [pct ...]   (default 0 50 100 200)"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

b = bench.C2Bench(16)
s = b.stream
pcts = [int(a) for a in sys.argv[1:]] or [0, 50, 100, 200]


def lone_once(slots):
    b.ex.resident_begin(s)
    t = time.perf_counter()
    while time.perf_counter() - t < 300e-6:   # the persistent kernel is up and polling
        pass
    t0 = time.perf_counter()
    seq = b.ex.launch(slots, s, independent=True)
    while not b.ex.resident_step_done(seq):
        pass
    t1 = time.perf_counter()
    b.ex.resident_end()
    torch.cuda.synchronize()
    return (t1 - t0) * 1e6


for pct in pcts:
    b.ex.clear_plans()
    b.ex.set_option("split_pct_idle", pct)
    slots = b.slots[3]
    for _ in range(3):
        lone_once(slots)          # builds + uploads the plan, warms the path
    st = None
    ts = [lone_once(slots) for _ in range(25)]
    st = b.ex.last_plan()
    print(f"split_pct_idle {pct:4d}: lone resident step {statistics.median(ts):6.2f} us (min {min(ts):6.2f})"
          f"  plan items {st['n_items']} splits {st['n_split_items']} max/mean cta cost "
          f"{st['max_cta_cost']:.0f}/{st['mean_cta_cost']:.0f}", flush=True)
