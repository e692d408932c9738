"""A short command for ncu captures: N warm-up launches of one coalesced step, then the target
launches. usage: python tools/ncu_target.py c2|c1 [warm] [target] [option=value ...]
(ncu -k regex:coalesced_step_kernel -s <warm> -c <target>)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1901_10008_b200.executor import Executor, OperandSet  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 20
target = int(sys.argv[3]) if len(sys.argv) > 3 else 3
if cfg == "c2":
    from bench import C2Bench
    b = C2Bench(16)
    ex, slots = b.ex, b.slots
else:
    ex = Executor()
    slots = [[OperandSet("gemv", (1000, 2048), dtype="fp32", seed=10 * r + i).register(ex) for i in range(4)]
             for r in range(8)]
for opt in sys.argv[4:]:
    k, v = opt.split("=")
    ex.set_option(k, int(v))
for r in range(warm + target):
    ex.launch(slots[r % len(slots)])
torch.cuda.synchronize()
print("done", ex.last_plan())
