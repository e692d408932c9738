"""Calibrate the executor's GEMM pipeline on single large problems."""
import os
import sys
import statistics

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1901_10008_b200.executor import Executor, OperandSet  # noqa: E402


def timeit(ex, slots, n=20):
    for _ in range(3):
        ex.launch(slots)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in evs:
        a.record(); ex.launch(slots); b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in evs) * 1e-3


ex = Executor()
# fixed launch overhead: tiny problems + a trivial torch kernel for reference
x = torch.zeros(1024, device="cuda")
for _ in range(3):
    x.add_(1)
torch.cuda.synchronize()
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
for a, b in evs:
    a.record(); x.add_(1); b.record()
torch.cuda.synchronize()
print(f"torch tiny add: {statistics.median(a.elapsed_time(b) for a, b in evs)*1e3:.2f} us")
for name, op, dims in (("tiny_elt", "elementwise", (1024,)), ("tiny_gemm", "gemm", (128, 64, 64))):
    o = OperandSet(op, dims, seed=0)
    sl = [o.register(ex)]
    print(f"{name}: {timeit(ex, sl)*1e6:.2f} us")
    ex.unregister(sl[0])
cases = [("square4096", [(4096, 4096, 4096)]), ("stream148x128", [(148 * 128, 128, 4096)]),
         ("stream148x64", [(148 * 128, 64, 4096)]), ("c2_512_49_4608", [(512, 49, 4608)]),
         ("wide_k64", [(256, 3136, 64)]), ("swap_64_3136_576", [(64, 3136, 576)])]
for dbg in (0, 1):
  ex.set_option("dbg", dbg)
  print("dbg", dbg)
  for name, shapes in cases:
    ops = [OperandSet("gemm", d, seed=1) for d in shapes]
    slots = [o.register(ex) for o in ops]
    ex.set_option("trace", 1)
    ex.launch(slots)
    ex.launch(slots)
    items, off = ex.read_trace()
    ex.set_option("trace", 0)
    t0 = min(it["t_prod"] for it in items if it["t_prod"])
    per_kb = [((it["t_mma_done"] - it["t_prod"]) / 1e3 / max(1, it["kb1"] - it["kb0"])) for it in items if it["t_mma_done"]]
    print(f"  {name:18s} per-kblock us: median {statistics.median(per_kb):.3f}  span {(max(it['t_end'] for it in items)-t0)/1e3:.2f} us")
    for s in slots:
        ex.unregister(s)
