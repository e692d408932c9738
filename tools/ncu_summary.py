"""Summarise ncu captures into profiles/ (committed evidence).

usage: python tools/ncu_summary.py <full.ncu-rep> <launches.csv> <out_prefix>
Writes <out_prefix>_full.json (per-launch metrics of the coalesced kernel from
`--set full`) and <out_prefix>_launches.json (per-kernel launch list with device
times and the coalesced kernel's share of the step).
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct_active",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum": "tma_load_bytes",
    "l1tex__m_l1tex2xbar_write_bytes_mem_global_op_tma_st.sum": "tma_store_bytes",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__inst_executed_op_tma_ld.sum": "tma_ld_instructions",
    "smsp__inst_executed_op_tma_st.sum": "tma_st_instructions",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ms": 1e3, "ns": 1e-3, "usecond": 1,
         "msecond": 1e3, "nsecond": 1e-3}


def full_summary(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        rec = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None}
        for h, u, v in zip(hdr, units, vals):
            if h in WANT:
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                rec[WANT[h]] = x * SCALE.get(u, 1)
        if "dram_read" in rec:
            rec["dram_bytes_per_launch"] = rec["dram_read"] + rec.get("dram_write", 0)
        out.append(rec)
    return out


def launch_list(path):
    text = open(path).read()
    rows = list(csv.reader(io.StringIO(text[text.index('"ID"'):])))
    hdr = rows[0]
    agg = {}
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        us = float(d["Metric Value"].replace(",", "")) * (1e-3 if d["Metric Unit"] in ("ns", "nsecond") else 1)
        agg.setdefault(name, []).append(us)
    total = sum(sum(v) for v in agg.values())
    return {k: {"launches": len(v), "mean_us": sum(v) / len(v), "share": sum(v) / total}
            for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))}


if __name__ == "__main__":
    rep, launches, prefix = sys.argv[1:4]
    full = full_summary(rep)
    with open(prefix + "_full.json", "w") as fh:
        json.dump({"source": rep, "launches": full,
                   "dram_bytes_per_launch": full[-1].get("dram_bytes_per_launch") if full else None},
                  fh, indent=1)
    with open(prefix + "_launches.json", "w") as fh:
        json.dump({"source": launches, "kernels": launch_list(launches)}, fh, indent=1)
    print(json.dumps(full[-1] if full else {}, indent=1))
