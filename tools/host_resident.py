"""Host vs device time per round of the native runtime loop, launch-per-step vs resident."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import C2Bench  # noqa: E402

b = C2Bench(replicas=8)
b.rt.set_profiling(True)
K = 400
r0 = 0
for mode in ("launch", "resident", "launch", "resident"):
    for r in range(r0, r0 + 20 + K):
        b.queue_round(r)
    b.run_rounds(r0, 20)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(b.stream)
    t0 = time.perf_counter()
    if mode == "resident":
        b.ex.resident_begin(b.stream)
    t1 = time.perf_counter()
    p0 = b.rt.host_profile()
    b.run_rounds(r0 + 20, K)
    t2 = time.perf_counter()
    p1 = b.rt.host_profile()
    if mode == "resident":
        b.ex.resident_end()
    e1.record(b.stream)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"{mode:9s}: host run() {(t2 - t1) / K * 1e6:.2f} us/round, begin {(t1 - t0) * 1e6:.0f} us, "
          f"device span {e0.elapsed_time(e1) / K * 1e3:.2f} us/round, wall {(t3 - t0) / K * 1e6:.2f} us/round; "
          + ", ".join(f"{k} {(p1[k] - p0[k]) / K / 1e3:.2f}" for k in p0) + " us/round")
    r0 += 20 + K
