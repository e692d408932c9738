"""Host cost of gmx_exec_resident_begin / end (idle residency), and of the parts of begin."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

b = bench.C2Bench(2)
s = b.stream
for i in range(3):
    b.ex.resident_begin(s)
    b.ex.resident_end()
torch.cuda.synchronize()
for i in range(5):
    t0 = time.perf_counter()
    b.ex.resident_begin(s)
    t1 = time.perf_counter()
    b.ex.resident_end()
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"begin {1e6*(t1-t0):.1f} us  end {1e6*(t2-t1):.1f} us  sync {1e6*(t3-t2):.1f} us", flush=True)
x = torch.empty(1, device="cuda")
for i in range(3):
    t0 = time.perf_counter()
    x.zero_()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"plain launch {1e6*(t1-t0):.1f} us")
