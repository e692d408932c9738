"""Measure the non-headline SURVEY §8(d) configs through the product runtime (lockstep).

  c1  4 tenants x ResNet-50 FC head, gemv(1000, 2048) fp32, one request each per round
  c3  mixed models: ResNet-50 + BERT-base (seq 128) + MobileNetV2, batch 1, bf16, SLO 10 ms,
      one request per stream per round (linear layer chains, model_library.json)
  c5  512 tenants x resnet50_like[i % 13] (C2 shapes), one request each per round, one GPU
      (the per-GPU shard of a 512-tenant box is 512/G tenants; see bench.py --gpus for scaling)

Each round's requests arrive together; the native loop steps the OoO scheduler (b200 decision
profile) and runs every step's dispatches as one coalesced launch. Device time is taken with
CUDA events around the run of R rounds (host decisions + launches included).
Prints one JSON line per config.
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1901_10008_b200 as gm  # noqa: E402
from paper_1901_10008_b200 import _lib  # noqa: E402
from paper_1901_10008_b200.executor import Executor, OperandSet  # noqa: E402
from paper_1901_10008_b200.kernels import kernel_desc  # noqa: E402
from paper_1901_10008_b200.runtime import Runtime  # noqa: E402

ROUND_NS = 1_000_000_000   # rounds never overlap in virtual time
SLO_NS = 10_000_000


def build_streams(config):
    lib = gm.kernels.load_model_library()
    if config == "c1":
        return [(f"fc{i}", lib["resnet50_fc"]) for i in range(4)]
    if config == "c3":
        return [("resnet50", lib["resnet50"]), ("bert_base", lib["bert_base"]),
                ("mobilenet_v2", lib["mobilenet_v2"])]
    if config == "c5":
        c2 = lib["resnet50_like"]
        return [(f"t{i:03d}", [dict(c2[i % 13], dtype="fp16")]) for i in range(512)]
    raise ValueError(config)


def replicas_for(streams, requested=None):
    """Operand replicas rotated over the rounds: like bench.py, enough that they exceed 4x the
    126 MB L2 (every round reads cold operands from HBM), 2..16."""
    if requested:
        return requested
    per_round = sum(gm.KernelSpec(0, sid, p["op_kind"], tuple(p["dims"]), p["dtype"]).bytes
                    for sid, protos in streams for p in protos)
    return max(2, min(16, -(-504_000_000 // per_round)))


class ConfigRun:
    def __init__(self, config, replicas=None):
        self.ex = Executor()
        self.streams = build_streams(config)
        self.replicas = replicas = replicas_for(self.streams, replicas)
        # operands per (replica, stream, layer); layers of a chain use distinct buffers
        self.slots = []
        self.useful = 0
        self.bytes = 0
        for r in range(replicas):
            row = []
            for si, (sid, protos) in enumerate(self.streams):
                layer = []
                for li, p in enumerate(protos):
                    o = OperandSet(p["op_kind"], tuple(p["dims"]), dtype=p["dtype"], seed=r * 7919 + si * 131 + li)
                    layer.append(o.register(self.ex))
                    if r == 0:
                        k = gm.KernelSpec(0, sid, p["op_kind"], tuple(p["dims"]), p["dtype"])
                        self.useful += k.flops
                        self.bytes += k.bytes
                row.append(layer)
            self.slots.append(row)
        self.rt = Runtime(self.ex, gm.load_profile("b200"), gm.SchedulerPolicy("ooo"))
        self.codes = [self.rt.stream_code(sid) for sid, _ in self.streams]
        self.next_kid = 0
        self.next_rid = 0

    def queue_round(self, r):
        t0 = r * ROUND_NS
        rep = r % self.replicas
        for si, (sid, protos) in enumerate(self.streams):
            n = len(protos)
            descs = (_lib.KernelDesc * n)()
            off = (_lib.i32 * (n + 1))()
            deps = (_lib.i64 * max(1, n - 1))()
            base = self.next_kid
            for li, p in enumerate(protos):
                k = gm.KernelSpec(base + li, sid, p["op_kind"], tuple(p["dims"]), p["dtype"],
                                  deps=frozenset({base + li - 1}) if li else frozenset(),
                                  arrival=t0, deadline=t0 + SLO_NS)
                descs[li] = kernel_desc(k, self.codes[si])
                if li:
                    deps[li - 1] = base + li - 1
                off[li + 1] = li
            sl = (_lib.i32 * n)(*self.slots[rep][si])
            self.rt.submit_raw(self.next_rid, self.codes[si], t0, t0 + SLO_NS, descs, n, deps, off, sl)
            self.next_kid += n
            self.next_rid += 1

    def run(self, rounds, warmup, resident=False):
        for r in range(warmup):
            self.queue_round(r)
        s = torch.cuda.current_stream()
        if resident:   # a first residency allocates the queue / pinned ring outside the timing
            self.ex.resident_begin(s)
        self.rt.run(until=warmup * ROUND_NS - 1)
        if resident:
            self.ex.resident_end()
        torch.cuda.synchronize()
        for r in range(warmup, warmup + rounds):
            self.queue_round(r)
        before = self.rt.run(until=warmup * ROUND_NS - 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        e0.record()
        if resident:
            self.ex.resident_begin(s)
        st = self.rt.run(until=(warmup + rounds) * ROUND_NS - 1)
        if resident:
            self.ex.resident_end()
        e1.record()
        host = time.perf_counter() - h0
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) * 1e-3
        done = st["completed_requests"] - before["completed_requests"]
        return {"rounds": rounds, "seconds": sec, "host_seconds": host,
                "executor": "resident" if resident else "launch per step",
                "useful_tflops": self.useful * rounds / sec / 1e12,
                "requests_per_s": done / sec, "kernels_per_s": (st["kernels"] - before["kernels"]) / sec,
                "launches_per_round": (st["launches"] - before["launches"]) / rounds,
                "steps_per_round": (st["steps"] - before["steps"]) / rounds,
                "us_per_launch": sec / max(1, st["launches"] - before["launches"]) * 1e6,
                "slo_misses_virtual": st["slo_misses"] - before["slo_misses"],
                "algorithmic_gb_per_s": self.bytes * rounds / sec / 1e9,
                "streams": len(self.streams), "replicas": self.replicas,
                "kernels_per_round": sum(len(p) for _, p in self.streams)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c3,c5")
    ap.add_argument("--rounds", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--resident", action="store_true", help="run the steps through the resident executor")
    ap.add_argument("--exec-lib", default=None, help="A/B runs: another build of libgmx_exec.so")
    ap.add_argument("--replicas", type=int, default=0,
                    help="operand replicas (0: enough to exceed 4x L2, like bench.py)")
    args = ap.parse_args()
    if args.exec_lib:
        from paper_1901_10008_b200 import executor
        executor.exec_lib(args.exec_lib)
    for cfg in args.configs.split(","):
        run = ConfigRun(cfg, args.replicas or None)
        res = run.run(args.rounds, args.warmup, args.resident)
        res["config"] = cfg
        print(json.dumps(res), flush=True)
        del run
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
