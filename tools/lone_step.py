"""Latency of ONE coalesced step launched alone (device idle before and after, the case of
wall-clock serving): CUDA events around each launch, median/min over N launches, for
(a) a torch one-element fill (launch + event floor), (b) one tiny elementwise member,
(c) one small GEMM member, (d) the full C2 step (16 GEMMs, operands rotated over 16 replicas)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import C2Bench  # noqa: E402
from paper_1901_10008_b200.executor import OperandSet  # noqa: E402

b = C2Bench(replicas=16)
for opt in sys.argv[1:]:
    k, v = opt.split("=")
    b.ex.set_option(k, int(v))
s = b.stream


def lone(fn, n=64):
    for _ in range(8):
        fn(0)
    torch.cuda.synchronize()
    ts = []
    for r in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn(r)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return f"median {statistics.median(ts):.2f} us  min {min(ts):.2f} us"


x = torch.empty(1, device="cuda")
print("torch fill(1):      ", lone(lambda r: x.fill_(1.0)))
tiny = OperandSet("elementwise", (1024,), seed=1).register(b.ex)
print("coalesced eltwise 1K:", lone(lambda r: b.ex.launch([tiny], s)))
g = OperandSet("gemm", (128, 128, 64), seed=2).register(b.ex)
print("coalesced gemm 128^2x64:", lone(lambda r: b.ex.launch([g], s)))
g2 = OperandSet("gemm", (256, 196, 2304), seed=3).register(b.ex)
print("coalesced gemm 256x196x2304:", lone(lambda r: b.ex.launch([g2], s)))
print("coalesced C2 step:  ", lone(lambda r: b.ex.launch(b.slots[r % 16], s)))
p = b.ex.last_plan()
print(f"  (C2 plan grid {p['grid']} items {p['n_items']} splits {p['n_split_items']} max/mean cta cost "
      f"{p['max_cta_cost']:.0f}/{p['mean_cta_cost']:.0f})")
