"""Host cost of the native runtime per round vs device time (is the bench host-bound?)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import C2Bench, ROUND_NS  # noqa: E402

b = C2Bench(replicas=8)
for r in range(20):
    b.queue_round(r)
b.run_rounds(0, 20)
torch.cuda.synchronize()
K = 400
for r in range(20, 20 + K):
    b.queue_round(r)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t0 = time.perf_counter()
b.run_rounds(20, K)
t1 = time.perf_counter()
e1.record()
torch.cuda.synchronize()
print(f"host run(): {(t1 - t0) / K * 1e6:.2f} us/round ; device span {e0.elapsed_time(e1) / K * 1e3:.2f} us/round")
# device-only: same launches captured back-to-back without decisions
slots = [b.slots[r % 8] for r in range(K)]
for s in slots[:8]:
    b.ex.launch(s)
torch.cuda.synchronize()
e0.record()
t0 = time.perf_counter()
for s in slots:
    b.ex.launch(s)
t1 = time.perf_counter()
e1.record()
torch.cuda.synchronize()
print(f"launch-only: host {(t1 - t0) / K * 1e6:.2f} us/launch ; device {e0.elapsed_time(e1) / K * 1e3:.2f} us/launch")
# CUDA graph of 48 launches: pure device time per launch
INDEP = len(sys.argv) > 1
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for x in slots[:8]:
        b.ex.launch(x, s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for x in slots[:48]:
            b.ex.launch(x, s, independent=INDEP)
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"graph: device {e0.elapsed_time(e1) / (5 * 48) * 1e3:.2f} us/launch")
