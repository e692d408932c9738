"""Device cost per step of TINY steps in the resident executor (the C3/C4 regime: chains of
single-member steps): a held batch of N steps, each one small GEMM (planned or inline),
CUDA events release -> kernel exit. usage: python tools/tiny_steps.py [m n k] [option=value ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1901_10008_b200.executor import Executor, OperandSet  # noqa: E402

args = [a for a in sys.argv[1:] if "=" not in a]
m, n, k = (int(x) for x in args) if args else (128, 128, 64)
ex = Executor()
for kv in [a for a in sys.argv[1:] if "=" in a]:
    a, b = kv.split("=")
    ex.set_option(a, int(b))
slots = [OperandSet("gemm", (m, n, k), seed=r).register(ex) for r in range(8)]
s, side = torch.cuda.Stream(), torch.cuda.Stream()
with torch.cuda.stream(s):
    for r in range(8):
        ex.launch([slots[r]], s)
    s.synchronize()
    for N in (50, 400):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ex.resident_begin(s, hold=True)
        for j in range(N):
            ex.launch([slots[j % 8]], s, independent=True)
        ex.resident_release()
        e0.record(side)
        ex.resident_end()
        e1.record(s)
        s.synchronize()
        side.synchronize()
        print(f"gemm({m},{n},{k}) x {N} independent steps: {e0.elapsed_time(e1) * 1e3 / N:.2f} us per step")
    # dependent chain: each step waits for the previous (like a request's chain)
    N = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ex.resident_begin(s, hold=True)
    for j in range(N):
        ex.launch([slots[j % 8]], s, dep_slots=[slots[(j - 1) % 8]])
    ex.resident_release()
    e0.record(side)
    ex.resident_end()
    e1.record(s)
    s.synchronize()
    side.synchronize()
    print(f"gemm({m},{n},{k}) x {N} dependent steps: {e0.elapsed_time(e1) * 1e3 / N:.2f} us per step")
