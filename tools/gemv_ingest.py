"""Per-item GEMV rate: one gemv(rows, n) fp32 problem launched alone, traced; per item (16-row
blocks) bytes / (end - start). rows=16 puts one item on one CTA (no HBM contention); larger
row counts load every SM. usage: python tools/gemv_ingest.py rows [n] [option=value ...]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1901_10008_b200.executor import Executor, OperandSet  # noqa: E402

args = [a for a in sys.argv[1:] if "=" not in a]
rows = int(args[0]) if args else 16
n = int(args[1]) if len(args) > 1 else 2048
ex = Executor()
for kv in [a for a in sys.argv[1:] if "=" in a]:
    k, v = kv.split("=")
    ex.set_option(k, int(v))
slots = [OperandSet("gemv", (rows, n), dtype="fp32", seed=r).register(ex) for r in range(8)]
for r in range(16):
    ex.launch([slots[r % 8]])
torch.cuda.synchronize()
ex.set_option("trace", 1)
for r in range(2):
    torch.cuda._sleep(100_000)
    ex.launch([slots[r % 8]])
    torch.cuda.synchronize()
    items, off = ex.read_trace()
    ks = ex.kernel_stamps
    t0 = min(k[0] for k in ks)
    rates, durs = [], []
    for it in items:
        if not it["t_end"]:
            continue
        nb = (it["col0"] - it["row0"]) * n * 4
        us = (it["t_end"] - it["t_prod"]) / 1e3 if it["t_prod"] else None
        if us:
            rates.append(nb / us / 1e3)
            durs.append(us)
    span = (max(k[3] for k in ks) - t0) / 1e3
    print(f"rows {rows} n {n}: {len(items)} items on {len(ks)} CTAs, kernel span {span:.2f} us "
          f"({rows * n * 4 / span / 1e3:.0f} GB/s); per item median {statistics.median(durs):.2f} us, "
          f"{statistics.median(rates):.1f} GB/s per item")
