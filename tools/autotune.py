"""Measured autotuner CLI: tune the C2 cluster keys (resnet50_like, bf16) at
co-tenancy 1..T on this B200 and write the reference-format TuningTable JSON.

usage: python tools/autotune.py [--max-tenancy 4] [--out profiles/tuning_b200_measured.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1901_10008_b200 as gm  # noqa: E402
from paper_1901_10008_b200.autotune import autotune  # noqa: E402
from paper_1901_10008_b200.executor import Executor  # noqa: E402
from paper_1901_10008_b200.tuning import ClusterKey  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-tenancy", type=int, default=4)
    ap.add_argument("--out", default="profiles/tuning_b200_measured.json")
    ap.add_argument("--keys", default="c2", help="c2 (the 13 resnet50_like GEMMs) or op:dtype:dims,...")
    args = ap.parse_args()
    if args.keys == "c2":
        lib = gm.kernels.load_model_library()
        keys = [ClusterKey("gemm", "fp16", tuple(p["dims"])) for p in lib["resnet50_like"]]
    else:
        keys = [ClusterKey.from_string(k) for k in args.keys.split(",")]
    ex = Executor()
    table = autotune(ex, keys, args.max_tenancy, gm.load_profile("b200"), log=lambda m: print(m, flush=True))
    table.save(args.out)
    greedy_vs_collab = {}
    for key in keys:
        picks = [table.lookup(key, t).tile_n for t in range(1, args.max_tenancy + 1)]
        if len(set(picks)) > 1:
            greedy_vs_collab[key.as_string()] = picks
    print(json.dumps({"out": args.out, "keys": len(keys), "tenancy_dependent_tiles": greedy_vs_collab}))


if __name__ == "__main__":
    main()
