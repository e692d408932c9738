"""Per-(step, CTA) timeline of a held resident run of C2 steps: where does a step's time go?"""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import C2Bench, time_resident  # noqa: E402

STEPS = 64
b = C2Bench(replicas=8)
for kv in sys.argv[1:]:
    k, v = kv.split("=")
    b.ex.set_option(k, int(v))
b.ex.set_option("rtrace", STEPS)
t, _, plan = time_resident(b, STEPS)
grid = C.c_int32()
buf = (C.c_uint64 * (STEPS * 148 * 2 * 8))()
rc = b.ex._lib.gmx_exec_resident_read_rtrace(b.ex._h, buf, len(buf), C.byref(grid))
assert rc == 0, b.ex._lib.gmx_exec_last_error()
G = grid.value
st = lambda k, c, f: buf[(k * G + c) * 8 + f]
t0 = min(st(0, c, 0) for c in range(G) if st(0, c, 0))
print(f"per-step {t * 1e6:.2f} us (device); grid {G}")
for k in list(range(0, 6)) + [STEPS // 2, STEPS - 1]:
    ps = [st(k, c, 0) for c in range(G)]
    pe = [st(k, c, 1) for c in range(G)]
    es = [st(k, c, 2) for c in range(G)]
    ee = [st(k, c, 3) for c in range(G)]
    f = lambda xs: f"{(min(xs) - t0) / 1e3:8.2f}..{(max(xs) - t0) / 1e3:8.2f}"
    print(f"step {k:3d}: prod start {f(ps)} | prod issued {f(pe)} | epi start {f(es)} | epi done {f(ee)}")
# per-CTA epilogue busy: mean over steps of (epi done - epi start), and producer issue span
dur_e = [st(k, c, 3) - st(k, c, 2) for k in range(8, STEPS - 1) for c in range(G)]
dur_p = [st(k, c, 1) - st(k, c, 0) for k in range(8, STEPS - 1) for c in range(G)]
gap = [st(k + 1, c, 0) - st(k, c, 1) for k in range(8, STEPS - 2) for c in range(G)]
print("epi step span us: median %.2f p90 %.2f" % (statistics.median(dur_e) / 1e3, sorted(dur_e)[int(.9 * len(dur_e))] / 1e3))
print("prod step span us: median %.2f p90 %.2f" % (statistics.median(dur_p) / 1e3, sorted(dur_p)[int(.9 * len(dur_p))] / 1e3))
print("prod gap between steps us: median %.2f p90 %.2f" % (statistics.median(gap) / 1e3, sorted(gap)[int(.9 * len(gap))] / 1e3))

print("slowest CTAs per step (epi span us, items, split items, gemm items, items-done->accounted us):")
for k in range(1, 9):
    rows = sorted(((st(k, c, 3) - st(k, c, 2)) / 1e3, c, st(k, c, 4), st(k, c, 5), st(k, c, 6),
                   (st(k, c, 3) - st(k, c, 7)) / 1e3) for c in range(G))
    print(k, [tuple(round(x, 2) if isinstance(x, float) else x for x in r) for r in rows[-4:]],
          "median", round(rows[len(rows) // 2][0], 2))
