"""A/B of executor builds on C2 at the kernel level: held resident batch (CUDA events) and the
window timeline of tools/trace_window.py's shape, for the .so given (default: in-tree).
usage: python tools/ab_held.py [path/to/libgmx_exec.so] [option=value ...]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_10008_b200.executor import exec_lib  # noqa: E402

so = [a for a in sys.argv[1:] if a.endswith(".so")]
if so:
    exec_lib(so[0])
import bench  # noqa: E402

b = bench.C2Bench(bench.replicas_for(bench.tenant_set(16), 16))
for kv in [a for a in sys.argv[1:] if "=" in a]:
    k, v = kv.split("=")
    b.ex.set_option(k, int(v))
held = [bench.time_resident(b, 400)[0] * 1e6 for _ in range(5)]
lone, _ = bench.time_launch_only(b, 96)
print(f"{so[0] if so else 'in-tree'}: held {statistics.median(held):.3f} us/step (min {min(held):.3f}), "
      f"launch-per-step graph {lone * 1e6:.3f} us")
