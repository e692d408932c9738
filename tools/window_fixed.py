"""Fixed cost of a resident window as bench.py times it (ev0 on an idle side stream after the
persistent launch call returned, ev1 after the kernel's exit), without steps:
  empty      begin -> ev0 -> end -> ev1              (device start-up + stop + exit)
  started    begin -> host waits 300 us -> ev0 -> end -> ev1   (stop + exit only)
  one/K      begin -> ev0 -> K rounds -> end -> ev1  (K = 1, 20), host loop time beside
Usage: python tools/window_fixed.py [K=V executor options ...]"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

b = bench.C2Bench(16)
for opt in sys.argv[1:]:
    k, v = opt.split("=")
    b.ex.set_option(k, int(v))
s = b.stream
side = torch.cuda.Stream()
nxt = 0
for r in range(64):
    b.queue_round(r)
b.run_rounds(0, 16)
torch.cuda.synchronize()
for _ in range(3):
    b.ex.resident_begin(s)
    b.run_rounds(16 + 16 * _, 16)
    b.ex.resident_end()
    torch.cuda.synchronize()
nxt = 64
b.next_round = nxt


def win(mode, k=0):
    global nxt
    for r in range(nxt, nxt + k):
        b.queue_round(r)
    b.rt.run(until=nxt * bench.ROUND_NS - 1, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    b.ex.resident_begin(s)
    h1 = time.perf_counter()
    if mode == "started":
        while time.perf_counter() - h1 < 300e-6:
            pass
    e0.record(side)
    if k:
        b.run_rounds(nxt, k)
        nxt += k
    h2 = time.perf_counter()
    b.ex.resident_end()
    e1.record(s)
    torch.cuda.synchronize()
    side.synchronize()
    mhz, span = b.ex.resident_sm_clock()
    return e0.elapsed_time(e1) * 1e3, (h1 - h0) * 1e6, (h2 - h1) * 1e6, span / 1e3


for mode, k in (("empty", 0), ("started", 0), ("empty", 1), ("started", 1), ("empty", 20), ("started", 20)):
    rs = [win(mode, k) for _ in range(15)]
    med = lambda j: statistics.median(x[j] for x in rs)
    print(f"{mode:8s} K={k:2d}: window {med(0):7.2f} us (min {min(x[0] for x in rs):.2f})  begin call {med(1):6.1f} us"
          f"  host loop {med(2):6.1f} us  device span {med(3):6.1f} us", flush=True)
