"""Per-link latency of ONE dependency chain in wall-clock mode (the C4 critical path): one request
of `model` (default resnet50: 54 kernels, each depending on the previous) runs alone through the
wall-clock runtime; from the replay log, per link: device round trip (dispatch -> completion
observed) and host decision time (completion observed -> next dispatch). Resident executor: the
per-step device stamps (relay, first CTA start, last list accounted, reported to the host).

usage: python tools/chain_latency.py [model] [resident=0|1] [option=value ...]"""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1901_10008_b200 as gm  # noqa: E402
from paper_1901_10008_b200.executor import Executor, OperandSet  # noqa: E402
from paper_1901_10008_b200.runtime import Runtime  # noqa: E402

so = [a for a in sys.argv[1:] if a.endswith(".so")]
if so:   # an A/B build of the executor (tools/ab_build.sh)
    from paper_1901_10008_b200.executor import exec_lib
    exec_lib(so[0])
args = [a for a in sys.argv[1:] if "=" not in a and not a.endswith(".so")]
kv = dict(a.split("=") for a in sys.argv[1:] if "=" in a)
model = args[0] if args else "resnet50"
resident = int(kv.pop("resident", 0)) != 0
reps = int(kv.pop("reps", 3))
lib = gm.kernels.load_model_library()
protos = lib[model]
ex = Executor()
for k, v in kv.items():
    ex.set_option(k, int(v))
slots = [OperandSet(p["op_kind"], tuple(p["dims"]), dtype=p["dtype"], seed=i, on_device=True).register(ex)
         for i, p in enumerate(protos)]
torch.cuda.synchronize()
L = len(protos)
print(f"{model}: {L} kernels in one chain, executor {'resident' if resident else 'launch per step'}")


def one(rid, rtrace=False):
    rt = Runtime(ex, gm.load_profile("b200"), gm.SchedulerPolicy("ooo"), mode="realtime")
    ks, prev = [], None
    lead = 2_000_000
    for i, p in enumerate(protos):
        kid = rid * 1000 + i
        ks.append(gm.KernelSpec(kid, "s0", p["op_kind"], tuple(p["dims"]), p["dtype"],
                                (prev,) if prev is not None else (), lead, lead + 10_000_000))
        prev = kid
    rt.submit(gm.InferenceRequest(rid, "s0", tuple(ks), lead, gm.LatencyConstraint(10_000_000)), slots)
    rt.set_profiling(True)
    rt.set_origin_now()
    s = torch.cuda.current_stream()
    if resident:
        if rtrace:
            ex.set_option("rtrace", L + 2)
        ex.resident_begin(s)
        try:
            rt.run(until=lead + 1_000_000_000, stream=s)
        finally:
            ex.resident_end()
        torch.cuda.synchronize()
    else:
        rt.run(until=lead + 1_000_000_000, stream=s)
        torch.cuda.synchronize()
    log = rt.replay_log()
    disp = [t for kind, t, a, kids in log if kind == 2]
    comp = [t for kind, t, a, kids in log if kind == 0]
    done = dict(rt.drain_completions())
    global prof
    prof = rt.host_profile()
    return disp, comp, done[rid] - lead


for r in range(reps):
    disp, comp, lat = one(r, rtrace=resident and r == reps - 1)
dev = [c - d for d, c in zip(disp, comp)]
host = [disp[j + 1] - comp[j] for j in range(len(comp) - 1)]
f = lambda xs: f"median {statistics.median(xs) / 1e3:.2f} p10 {sorted(xs)[len(xs) // 10] / 1e3:.2f} p90 {sorted(xs)[9 * len(xs) // 10] / 1e3:.2f}"
print(f"request latency {lat / 1e6:.3f} ms = {lat / L / 1e3:.2f} us per link")
print(f"dispatch -> completion observed (us): {f(dev)}")
print(f"completion observed -> next dispatch (us): {f(host)}")
print("host time per link (us):", {k: round(v / L / 1e3, 2) for k, v in prof.items()})
if resident:
    S = L + 2
    grid = C.c_int32()
    n = S * 148 * 8 + 2 * S
    buf = (C.c_uint64 * n)()
    rc = ex._lib.gmx_exec_resident_read_rtrace(ex._h, buf, n, C.byref(grid))
    assert rc == 0, ex._lib.gmx_exec_last_error()
    G = grid.value
    base = S * G * 8
    rows = []
    for k in range(L):
        relay, report = buf[base + k], buf[base + S + k]
        st = [buf[(k * G + c) * 8] for c in range(G) if buf[(k * G + c) * 8]]
        pi = [buf[(k * G + c) * 8 + 1] for c in range(G) if buf[(k * G + c) * 8 + 1]]
        es = [buf[(k * G + c) * 8 + 2] for c in range(G) if buf[(k * G + c) * 8 + 2]]
        idn = [buf[(k * G + c) * 8 + 7] for c in range(G) if buf[(k * G + c) * 8 + 7]]
        acc = [buf[(k * G + c) * 8 + 3] for c in range(G) if buf[(k * G + c) * 8 + 3]]
        if not (relay and st and acc and report):
            continue
        rows.append((min(st) - relay, (max(idn) if idn else 0) - min(st), max(acc) - (max(idn) if idn else 0),
                     report - max(acc), len(st), len(es), (max(pi) - min(st)) if pi else 0,
                     (max(es) - min(st)) if es else 0))
    for name, i in (("relay -> first CTA starts step", 0), ("first start -> last items done", 1),
                    ("items done -> list accounted", 2), ("accounted -> reported to host", 3),
                    ("first start -> producer issued all", 6), ("first start -> epilogue has unit", 7)):
        print(f"  {name:34s} {f([r[i] for r in rows])}")
    print("  CTAs per step (started / with units):", statistics.median(r[4] for r in rows), statistics.median(r[5] for r in rows))
