"""C1 (4 tenants x ResNet-50 FC gemv(1000, 2048) fp32) at the kernel level: one coalesced step
= the 4 GEMVs; operands rotate over 8 replicas (262 MB > L2). (a) held resident batch (steps
back to back, CUDA events), (b) lone step queued behind a sleep (CUDA events), (c) per-CTA
kernel stamps of a traced lone step. Floor: 32,816,768 B / HBM peak (5.02 us at 6535 GB/s)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1901_10008_b200.executor import Executor, OperandSet, exec_lib  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):
    exec_lib(sys.argv[1])
ex = Executor()
for opt in [a for a in sys.argv[1:] if "=" in a]:
    k, v = opt.split("=")
    ex.set_option(k, int(v))
R = 8
slots = [[OperandSet("gemv", (1000, 2048), dtype="fp32", seed=10 * r + i).register(ex) for i in range(4)]
         for r in range(R)]
s = torch.cuda.current_stream()
for r in range(16):
    ex.launch(slots[r % R], s)
torch.cuda.synchronize()
bytes_step = 4 * (1000 * 2048 + 2048 + 1000) * 4
# (a) held batch
side = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ex.resident_begin(s, hold=True)
N = 1000
for j in range(N):
    ex.launch(slots[j % R], s, independent=True)
ex.resident_release()
e0.record(side)
ex.resident_end()
e1.record(s)
torch.cuda.synchronize()
held = e0.elapsed_time(e1) * 1e3 / N
# (b) lone steps
ts = []
for j in range(48):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(200_000)
    a.record(s)
    ex.launch(slots[j % R], s)
    b.record(s)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
plan = ex.last_plan()
# (c) trace
ex.set_option("trace", 1)
torch.cuda._sleep(200_000)
ex.launch(slots[3], s)
items, off = ex.read_trace()
ks = ex.kernel_stamps
ex.set_option("trace", 0)
t0 = min(k[0] for k in ks)
ends = sorted((k[3] - t0) / 1e3 for k in ks)
print(json.dumps({"held_us_per_step": round(held, 3), "held_GBps": round(bytes_step / held / 1e3, 1),
                  "lone_median_us": round(statistics.median(ts), 2), "lone_min_us": round(min(ts), 2),
                  "kernel_span_us": round(ends[-1], 2), "cta_exit_median_us": round(ends[len(ends) // 2], 2),
                  "grid": plan["grid"], "items": plan["n_items"], "gemv_items": plan["n_gemv_items"]}))

by_cta = {}
for it in items:
    by_cta.setdefault(it["cta"], []).append(it)
order = sorted(by_cta, key=lambda c: -ks[c][3])
for c in order[:3] + order[len(order) // 2:len(order) // 2 + 2]:
    k = ks[c]
    print(f"CTA {c}: entry {(k[0]-t0)/1e3:.2f} prologue {(k[1]-t0)/1e3:.2f} loops {(k[2]-t0)/1e3:.2f} exit {(k[3]-t0)/1e3:.2f}")
    for it in by_cta[c]:
        print(f"   p{it['problem']} rows {it['row0']}-{it['col0']} stages {it['kb1']} start {(it['t_prod']-t0)/1e3:.2f} end {(it['t_end']-t0)/1e3:.2f}")
