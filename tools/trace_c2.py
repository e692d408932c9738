"""Trace one coalesced C2 launch: per-item globaltimer stamps -> where the time goes."""
import os
import sys
import statistics

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import C2Bench  # noqa: E402

b = C2Bench(replicas=8)
if len(sys.argv) > 1:
    b.ex.set_option("max_split", int(sys.argv[1]))
for r in range(8):
    b.ex.launch(b.slots[r % 8])
torch.cuda.synchronize()
b.ex.set_option("trace", 1)
b.ex.launch(b.slots[3])
items, off = b.ex.read_trace()
b.ex.set_option("trace", 0)
t0 = min(min(x for x in (it["t_prod"], it["t_epi"]) if x) for it in items)
tend = max(it["t_end"] for it in items)
print(f"kernel span (first stamp -> last end): {(tend - t0) / 1e3:.2f} us, items {len(items)}")
shapes = [s for s in b.shapes]
per_cta_end = {}
for it in items:
    per_cta_end[it["cta"]] = max(per_cta_end.get(it["cta"], 0), it["t_end"])
ends = sorted((v - t0) / 1e3 for v in per_cta_end.values())
print("cta end times us: min %.2f median %.2f max %.2f" % (ends[0], ends[len(ends) // 2], ends[-1]))
starts = sorted((it["t_prod"] - t0) / 1e3 for it in items if it["t_prod"])
print("first producer start per item: min %.2f median %.2f max %.2f" % (starts[0], starts[len(starts)//2], starts[-1]))
rows = []
for it in items:
    dims = shapes[it["problem"] % 16] if it["problem"] < 128 else None
    kb = it["kb1"] - it["kb0"]
    load = (it["t_mma_done"] - it["t_prod"]) / 1e3 if it["t_prod"] and it["t_mma_done"] else None
    epi = (it["t_end"] - it["t_epi"]) / 1e3 if it["t_epi"] else None
    rows.append((it["cta"], it["problem"], dims, kb, it["nsplit"], load, epi,
                 (it["t_prod"] - t0) / 1e3, (it["t_end"] - t0) / 1e3))
rows.sort(key=lambda r: -r[-1])
print("slowest-finishing items: cta prob dims kb nsplit load_us epi_us start_us end_us")
for r in rows[:25]:
    print(r)
by_shape = {}
for r in rows:
    if r[5] is not None:
        by_shape.setdefault((r[2], r[4]), []).append((r[5], r[3]))
print("per shape: mean load us, mean kblocks, us per kblock")
for k, v in sorted(by_shape.items(), key=lambda kv: str(kv[0])):
    ml = statistics.mean(x[0] for x in v)
    mk = statistics.mean(x[1] for x in v)
    print(k, len(v), round(ml, 2), round(mk, 1), round(ml / mk, 3))

print("\nper-CTA timelines (us rel. t0): item: prob dims kb nsplit | prod mma_done epi end")
ctas = sorted(per_cta_end, key=lambda c: -per_cta_end[c])[:4] + sorted(per_cta_end, key=lambda c: per_cta_end[c])[:2]
for c in ctas:
    print(f"CTA {c}:")
    for it in items:
        if it["cta"] != c:
            continue
        rel = lambda t: f"{(t - t0) / 1e3:7.2f}" if t else "   -   "
        print(f"   p{it['problem']:3d} {str(shapes[it['problem'] % 16]):18s} kb {it['kb1']-it['kb0']:3d} ns {it['nsplit']} |"
              f" {rel(it['t_prod'])} {rel(it['t_mma_done'])} {rel(it['t_epi'])} {rel(it['t_end'])}"
              f" || {rel(it['t_e_start'])} {rel(it['t_e_staged'])} {rel(it['t_e_bar'])} {rel(it['t_e_issued'])}")
