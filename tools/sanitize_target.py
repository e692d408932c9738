"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck) over every kernel
path: per-step launches of a C2 step (split-K items, role-swapped tiles, TMA-store epilogue),
a mixed GEMM/tf32/GEMV/elementwise step with bias + activation (plain and staged GEMV), an
inline (plan-less) step, and the resident persistent kernel (held batch + runtime-fed steps).
usage: python tools/sanitize_target.py [step|resident|all]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1901_10008_b200.executor import Executor, OperandSet  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
C2 = [(64, 3136, 147), (64, 3136, 64), (64, 3136, 576), (256, 3136, 64), (128, 784, 256),
      (128, 784, 1152), (512, 784, 128), (256, 196, 512), (256, 196, 2304),
      (1024, 196, 256), (512, 49, 1024), (512, 49, 4608), (2048, 49, 512)]
ex = Executor()
c2 = [OperandSet("gemm", C2[i % 13], seed=i).register(ex) for i in range(16)]
mixed_ops = [OperandSet("gemm", (256, 196, 512), dtype="fp32", seed=1, bias=True, activation="gelu"),
             OperandSet("gemv", (1000, 2048), dtype="fp32", seed=2, bias=True, activation="relu"),
             OperandSet("elementwise", (50176,), seed=3, activation="gelu"),
             OperandSet("gemm", (512, 49, 4608), seed=4, bias=True, activation="relu", out_dtype=torch.float32),
             OperandSet("gemv", (777, 1280), seed=5)]
mixed = [o.register(ex) for o in mixed_ops]
s = torch.cuda.current_stream()
if what in ("step", "all"):
    for _ in range(2):
        ex.launch(c2, s)
    ex.launch(mixed, s)
    ex.set_option("gemv_staged", 1)
    ex.clear_plans()
    ex.launch(mixed, s)
    ex.set_option("gemv_staged", 0)
    ex.set_option("inline_plans", 1)
    ex.clear_plans()
    ex.launch(mixed[:3], s)     # first sighting: inline step (device-enumerated items)
    ex.set_option("inline_plans", 0)
    torch.cuda.synchronize()
    print("per-step launches ok")
if what in ("resident", "resident_cold", "all"):
    if what != "resident_cold":
        # plans of every slot set built before the persistent launch: plans first seen DURING a
        # residency are uploaded with cudaMallocAsync after the kernel's launch, which memcheck
        # reports as out-of-bounds reads (its view of allocations is taken at launch)
        for sl in (c2, mixed, *[c2[j::4] for j in range(4)]):
            ex.launch(sl, s)
        torch.cuda.synchronize()
    ex.resident_begin(s, hold=True)
    for j in range(4):
        ex.launch(c2 if j % 2 == 0 else mixed, s, independent=True)
    ex.resident_release()
    ex.resident_end()
    torch.cuda.synchronize()
    ex.resident_begin(s)
    for j in range(4):
        ex.launch(c2[j::4], s, independent=(j % 2 == 0), dep_slots=[] if j % 2 == 0 else [c2[0]])
    ex.resident_end()
    torch.cuda.synchronize()
    print("resident ok")
