"""Where does an e2e round go? H2D / compute / D2H device durations and host time per round."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import C2Bench  # noqa: E402

b = C2Bench(replicas=8)
for r in range(8):
    b.queue_round(r)
b.run_rounds(0, 8)
torch.cuda.synchronize()
host_in = b.b_arena[0].cpu().pin_memory()
host_out = torch.empty(b.c_numel, dtype=torch.bfloat16).pin_memory()
s_in, s_cmp, s_out = torch.cuda.Stream(), b.stream, torch.cuda.Stream()
E = lambda: torch.cuda.Event(enable_timing=True)
nxt = 8
# isolated: H2D alone, D2H alone, both concurrently
for name in ("h2d", "d2h", "both"):
    e0, e1 = E(), E()
    torch.cuda.synchronize()
    e0.record(s_in)
    for _ in range(10):
        if name in ("h2d", "both"):
            with torch.cuda.stream(s_in):
                b.b_arena[1].copy_(host_in, non_blocking=True)
        if name in ("d2h", "both"):
            with torch.cuda.stream(s_out):
                host_out.copy_(b.c_arena[1], non_blocking=True)
    s_in.wait_stream(s_out)
    e1.record(s_in)
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us per round", flush=True)
# compute alone via the runtime (host-driven)
for r in range(nxt, nxt + 20):
    b.queue_round(r)
e0, e1 = E(), E()
e0.record(s_cmp)
t0 = time.perf_counter()
b.run_rounds(nxt, 20)
t1 = time.perf_counter()
e1.record(s_cmp)
torch.cuda.synchronize()
print(f"compute (runtime, launch per step): device {e0.elapsed_time(e1) / 20 * 1e3:.1f} us, host {(t1 - t0) / 20 * 1e6:.1f} us per round")
nxt += 20
# one round at a time through run_rounds (as e2e does)
t0 = time.perf_counter()
for r in range(nxt, nxt + 20):
    b.queue_round(r)
    b.run_rounds(r, 1)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"queue_round + run_rounds(r, 1) host: {(t1 - t0) / 20 * 1e6:.1f} us per round")
