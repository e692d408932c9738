"""Single-SM TMA ingest rate: one long-K GEMM (m, n, k) launched alone without split-K, so only
ceil(m/128) CTAs stream (no HBM contention); per-item stamps give bytes / (mma_done - first TMA).
usage: python tools/sm_ingest.py [m n k] [option=value ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1901_10008_b200.executor import Executor, OperandSet  # noqa: E402

args = [a for a in sys.argv[1:] if "=" not in a]
m, n, k = (int(x) for x in args) if args else (512, 49, 4608)
ex = Executor()
ex.set_option("max_split", 1)
for kv in [a for a in sys.argv[1:] if "=" in a]:
    a, b = kv.split("=")
    ex.set_option(a, int(b))
slots = [OperandSet("gemm", (m, n, k), seed=r).register(ex) for r in range(8)]
for r in range(16):
    ex.launch([slots[r % 8]])
torch.cuda.synchronize()
ex.set_option("trace", 1)
for r in range(3):
    torch.cuda._sleep(100_000)
    ex.launch([slots[r % 8]])
    torch.cuda.synchronize()
    items, off = ex.read_trace()
    for it in items[:4]:
        kb = it["kb1"] - it["kb0"]
        us = (it["t_mma_done"] - it["t_prod"]) / 1e3
        bn = 64 if min(m, n) <= 64 else 128
        nbytes = kb * 64 * 2 * (128 + bn)
        print(f"launch {r} item p{it['problem']} kb {kb}: {us:.2f} us for {nbytes / 1e6:.2f} MB = {nbytes / us / 1e3:.1f} GB/s")
