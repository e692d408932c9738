"""Where the time of ONE coalesced step launched alone goes: the launch is queued behind a
sleep kernel (so host launch latency is not in the window), CUDA events around it, and the
per-CTA kernel stamps (entry, prologue done, role loops done, exit) + per-item stamps."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import C2Bench  # noqa: E402

b = C2Bench(replicas=16)
for opt in sys.argv[1:]:
    k, v = opt.split("=")
    b.ex.set_option(k, int(v))
s = b.stream
for r in range(32):
    b.ex.launch(b.slots[r % 16], s)
torch.cuda.synchronize()


def lone(r, trace=False):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(200_000)     # ~100 us: the launch below is queued before e0 fires
    e0.record(s)
    b.ex.launch(b.slots[r % 16], s)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3


with torch.cuda.stream(s):
    ts = [lone(r) for r in range(48)]
print(f"lone step (queued): median {statistics.median(ts):.2f} us  min {min(ts):.2f} us")
b.ex.set_option("trace", 1)
with torch.cuda.stream(s):
    for r in range(3):
        lone(r)
        items, off = b.ex.read_trace()
        ks = b.ex.kernel_stamps
        t0 = min(k[0] for k in ks)
        rel = lambda v: (v - t0) / 1e3
        ent = sorted(rel(k[0]) for k in ks)
        pro = sorted(rel(k[1]) for k in ks)
        loops = sorted(rel(k[2]) for k in ks)
        ex_ = sorted(rel(k[3]) for k in ks)
        f = lambda v: f"min {v[0]:.2f} med {v[len(v)//2]:.2f} p90 {v[int(len(v)*0.9)]:.2f} max {v[-1]:.2f}"
        print(f"launch {r}: entry {f(ent)} | prologue done {f(pro)} | loops done {f(loops)} | exit {f(ex_)}")
        first_prod = sorted(rel(it['t_prod']) for it in items if it['t_prod'])
        print(f"   first TMA issue per item: {f(first_prod)}")
        ends = sorted(rel(it['t_end']) for it in items if it['t_end'])
        print(f"   item ends: {f(ends)}")
b.ex.set_option("trace", 0)

# per-CTA timelines of the last traced launch (us rel. first entry)
shapes = b.shapes
by_cta = {}
for it in items:
    by_cta.setdefault(it["cta"], []).append(it)
order = sorted(by_cta, key=lambda c: -ks[c][3])
pick = order[:3] + order[len(order) // 2: len(order) // 2 + 2] + order[-1:]
print("\nCTA timelines: prob dims kb nsplit | tma_first mma_done epi_start end || entry prologue loops exit")
for c in pick:
    k = ks[c]
    print(f"CTA {c}: entry {rel(k[0]):.2f} prologue {rel(k[1]):.2f} loops {rel(k[2]):.2f} exit {rel(k[3]):.2f}")
    for it in by_cta[c]:
        r_ = lambda t: f"{rel(t):6.2f}" if t else "   -  "
        print(f"   p{it['problem']:3d} {str(shapes[it['problem'] % 16]):18s} kb {it['kb1']-it['kb0']:3d} ns {it['nsplit']} |"
              f" {r_(it['t_prod'])} {r_(it['t_mma_done'])} {r_(it['t_epi'])} {r_(it['t_end'])}"
              + (f" | reduced {r_(it['t_e_start'])} ticket {r_(it['t_e_staged'])} finalized {r_(it['t_e_bar'])}"
                 if it['nsplit'] > 1 else ""))

# epilogue phases of the unsplit tiles (first pass of each): epi start -> staging free + barrier
# -> chunks staged -> fence + barrier -> TMA stores issued -> item end (all warps done)
ph = {k: [] for k in ("wait", "stage", "bar", "issue", "tail")}
for it in items:
    if it["nsplit"] > 1 or it["type"] & 0x3f != 0 or not (it["t_e_start"] and it["t_e_issued"] and it["t_epi"]):
        continue
    ph["wait"].append(it["t_e_start"] - it["t_epi"])
    ph["stage"].append(it["t_e_staged"] - it["t_e_start"])
    ph["bar"].append(it["t_e_bar"] - it["t_e_staged"])
    ph["issue"].append(it["t_e_issued"] - it["t_e_bar"])
    ph["tail"].append(it["t_end"] - it["t_e_issued"])
print("\nunsplit tile epilogue phases (us, median / p90 over", len(ph["wait"]), "tiles):",
      {k: (round(statistics.median(v) / 1e3, 3), round(sorted(v)[int(0.9 * len(v))] / 1e3, 3)) for k, v in ph.items() if v})
