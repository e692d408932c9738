"""Timeline of bench.py's timed window (C2, resident executor, live-fed by the serving loop):
per step, when the dispatcher relayed it (host publish + one PCIe read), when its first CTA
started producing, when its last CTA finished, and when it was reported to the host — all in
%globaltimer ns relative to the dispatcher's start. Shows whether a short window is host-bound
(device idle between relays), device-bound (relays queue up ahead of starts) or pays a fixed
start/drain cost.

usage: python tools/trace_window.py [steps=20] [warmup=5] [option=value ...]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

so = [a for a in sys.argv[1:] if a.endswith(".so")]
if so:   # an A/B build of the executor (tools/ab_build.sh)
    from paper_1901_10008_b200.executor import exec_lib
    exec_lib(so[0])
kv = dict(a.split("=") for a in sys.argv[1:] if not a.endswith(".so"))
STEPS = int(kv.pop("steps", 20))
WARM = int(kv.pop("warmup", 5))
DELAY_MS = float(kv.pop("delay_us", 0)) / 1e3
PRESTEP = int(kv.pop("prestep", 0))
b = bench.C2Bench(bench.replicas_for(bench.tenant_set(16), 16))
for k, v in kv.items():
    b.ex.set_option(k, int(v))
all_cpus, core = bench.pin_serving_thread(torch.cuda.current_device())
side = torch.cuda.Stream()


def window(first, count, trace=False):
    for r in range(first, first + count):
        b.queue_round(r)
    b.rt.run(until=first * bench.ROUND_NS - 1, stream=b.stream)
    torch.cuda.synchronize()
    if trace:
        b.ex.set_option("rtrace", count + 2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    b.ex.resident_begin(b.stream)
    e0.record(side)
    if trace and PRESTEP:   # untimed-style warm step of another replica, before the rounds
        b.ex.launch(b.slots[(first + count) % b.replicas], b.stream, independent=True)
    if trace and DELAY_MS:
        bench.spin_host(DELAY_MS)
    h1 = time.perf_counter()
    b.run_rounds(first, count)
    h2 = time.perf_counter()
    b.ex.resident_end()
    e1.record(b.stream)
    torch.cuda.synchronize()
    side.synchronize()
    return e0.elapsed_time(e1) * 1e3, (h1 - h0) * 1e6, (h2 - h1) * 1e6


for r in range(WARM):
    b.queue_round(r)
b.run_rounds(0, WARM // 2)
torch.cuda.synchronize()
b.ex.resident_begin(b.stream)
b.run_rounds(WARM // 2, WARM - WARM // 2)
b.ex.resident_end()
torch.cuda.synchronize()
first = WARM
while first < WARM + max(b.replicas, 60):
    n = min(STEPS, 32)
    us, _, _ = window(first, n)
    first += n
us, begin_us, loop_us = window(first, STEPS, trace=True)
print(f"window {us:.1f} us = {us / STEPS:.2f} us/round; resident_begin {begin_us:.1f} us; "
      f"serving loop {loop_us:.1f} us = {loop_us / STEPS:.2f} us/round")
S = STEPS + 2
grid = C.c_int32()
n = S * 148 * 8 + 2 * S
buf = (C.c_uint64 * n)()
rc = b.ex._lib.gmx_exec_resident_read_rtrace(b.ex._h, buf, n, C.byref(grid))
assert rc == 0, b.ex._lib.gmx_exec_last_error()
G = grid.value
base = S * G * 8
relay = [buf[base + k] for k in range(S)]
report = [buf[base + S + k] for k in range(S)]
mhz, span = b.ex.resident_sm_clock()
t0 = min(x for x in relay if x)
print(f"device: dispatcher span {span / 1e3:.1f} us, SM clock {mhz:.0f} MHz")
print(" step   relay   start    done  report | start-relay  done-start  relay-gap")
prev = None
for k in range(S):
    st = [buf[(k * G + c) * 8] for c in range(G) if buf[(k * G + c) * 8]]
    dn = [buf[(k * G + c) * 8 + 3] for c in range(G) if buf[(k * G + c) * 8 + 3]]
    if not st or not relay[k]:
        continue
    s0, d1 = min(st) - t0, max(dn) - t0 if dn else 0
    rl, rp = relay[k] - t0, (report[k] - t0) if report[k] else 0
    gap = (rl - prev) if prev is not None else 0
    prev = rl
    print(f"{k:5d} {rl / 1e3:7.2f} {s0 / 1e3:7.2f} {d1 / 1e3:7.2f} {rp / 1e3:7.2f} | "
          f"{(s0 - rl) / 1e3:10.2f} {(d1 - s0) / 1e3:10.2f} {gap / 1e3:10.2f}")

# per-CTA detail of the first steps: producer start / producer issued / epilogue start / done
for k in (0, 1, 2, 3, S // 2):
    rows = []
    for c in range(G):
        f = [buf[(k * G + c) * 8 + i] for i in range(8)]
        if not f[0]:
            continue
        rel = lambda x: (x - t0) / 1e3 if x else -1.0
        rows.append((c, rel(f[0]), rel(f[1]), rel(f[2]), rel(f[3]), f[4], rel(f[7])))
    if not rows:
        continue
    q = lambda xs: " ".join(f"{x:7.2f}" for x in (min(xs), sorted(xs)[len(xs) // 4], sorted(xs)[len(xs) // 2],
                                                     sorted(xs)[3 * len(xs) // 4], max(xs)))
    print(f"step {k}: {len(rows)} CTAs | min/q1/med/q3/max")
    print("   prod start  ", q([r[1] for r in rows]))
    print("   prod issued ", q([r[2] for r in rows]))
    print("   epi start   ", q([r[3] for r in rows]))
    print("   epi done    ", q([r[4] for r in rows]))
    print("   items done  ", q([r[6] for r in rows]))
    print("   slowest (cta, prod start, prod issued, epi start, accounted, n items, items done):", [tuple(round(x, 2) if isinstance(x, float) else x for x in r) for r in sorted(rows, key=lambda r: r[4])[-5:]])

b.ex.set_option("rtrace", 0)
ev, gt, plan = bench.time_resident(b, 400)
print(f"held batch of 400 steps: {ev * 1e6:.2f} us/step (CUDA events), {gt * 1e6:.2f} (globaltimer); "
      f"plan n_items {plan['n_items']} splits {plan['n_split_items']} max/mean cta cost "
      f"{plan['max_cta_cost']:.0f}/{plan['mean_cta_cost']:.0f}")
