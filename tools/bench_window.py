"""Break down the fixed cost of a short timed window of the C2 bench (BENCH_r01: 20 rounds took
1.15 ms). For K rounds with residency started inside the CUDA-event window (bench.py's region):
host time of resident_begin, of the serving loop per round, of resident_end, and the device
window, with and without the NVML clock sampler thread and the serving-core pinning.
Prints one JSON line per (variant, K)."""

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    b = bench.C2Bench(16)
    r = 0
    for _ in range(2):                      # plans for every replica, residency machinery allocated
        for _ in range(16):
            b.queue_round(r)
            r += 1
        b.run_rounds(r - 16, 16)
        torch.cuda.synchronize()
        b.ex.resident_begin(b.stream)
        for _ in range(16):
            b.queue_round(r)
            r += 1
        b.run_rounds(r - 16, 16)
        b.ex.resident_end()
        torch.cuda.synchronize()
    all_cpus = sorted(os.sched_getaffinity(0))
    for variant in ("plain", "pinned+sampler", "plain"):
        core = None
        if "pinned" in variant:
            _, core = bench.pin_serving_thread(0)
        for K in (20, 20, 200):
            for _ in range(K):
                b.queue_round(r)
                r += 1
            first = r - K
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            sampler = bench.ClockSampler(0, avoid_core=core, allowed=all_cpus) if "sampler" in variant else None
            if sampler:
                sampler.__enter__()
                sampler.settle()
            h0 = time.perf_counter()
            e0.record(b.stream)
            b.ex.resident_begin(b.stream)
            h1 = time.perf_counter()
            b.run_rounds(first, K)
            h2 = time.perf_counter()
            b.ex.resident_end()
            e1.record(b.stream)
            h3 = time.perf_counter()
            torch.cuda.synchronize()
            if sampler:
                sampler.__exit__(None, None, None)
            ms = e0.elapsed_time(e1)
            dev_ns = b.ex.resident_device_ns()   # step 0 relayed -> last step complete (%globaltimer)
            flops = bench.useful_flops(b.shapes) * K
            print(json.dumps({"variant": variant, "K": K, "us_per_round": round(ms * 1e3 / K, 3),
                              "tflops": round(flops / (ms * 1e-3) / 1e12, 1),
                              "begin_us": round((h1 - h0) * 1e6, 1),
                              "loop_us_per_round": round((h2 - h1) * 1e6 / K, 3),
                              "end_us": round((h3 - h2) * 1e6, 1),
                              "window_us": round(ms * 1e3, 1), "steps_span_us": round(dev_ns / 1e3, 1),
                              "relay_span_us": round(b.ex._relay_ns() / 1e3, 1)}), flush=True)
        if core is not None:
            os.sched_setaffinity(0, set(all_cpus))


if __name__ == "__main__":
    main()
