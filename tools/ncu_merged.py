"""One launch carrying M scheduling rounds of C2 (merged slot sets) — a steady-state-like
workload for `ncu --set full` (the resident kernel cannot be replayed by ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import C2Bench  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 4
b = C2Bench(replicas=2 * M)
sets = [sum((b.slots[(j + q) % len(b.slots)] for q in range(M)), []) for j in range(0, 2 * M, M)]
for _ in range(3):
    for sl in sets:
        b.ex.launch(sl, independent=True)
torch.cuda.synchronize()
print("plan", b.ex.last_plan())
