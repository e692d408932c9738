"""Break down the fixed cost of a short timed window of the C2 bench (BENCH_r01: 20 rounds took
1.15 ms). For K rounds: (a) residency started inside the CUDA-event window (bench.py's region),
(b) the persistent kernel already resident and idle when the window opens, (c) launch per step.
Prints one JSON line per (mode, K)."""

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
    side = torch.cuda.Stream()
    for K in (20, 20, 50, 200, 1000):
        for mode in ("inside", "preresident", "per_step"):
            for _ in range(K):
                b.queue_round(r)
                r += 1
            first = r - K
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            host0 = time.perf_counter()
            if mode == "inside":
                e0.record(b.stream)
                b.ex.resident_begin(b.stream)
                b.run_rounds(first, K)
                b.ex.resident_end()
                e1.record(b.stream)
            elif mode == "preresident":
                b.ex.resident_begin(b.stream)
                t = time.perf_counter()
                while time.perf_counter() - t < 0.002:
                    pass
                e0.record(side)
                b.run_rounds(first, K)
                b.ex.resident_end()
                e1.record(b.stream)
            else:
                e0.record(b.stream)
                b.run_rounds(first, K)
                e1.record(b.stream)
            host1 = time.perf_counter()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            flops = bench.useful_flops(b.shapes) * K
            print(json.dumps({"mode": mode, "K": K, "us_per_round": round(ms * 1e3 / K, 3),
                              "tflops": round(flops / (ms * 1e-3) / 1e12, 1),
                              "host_us_per_round": round((host1 - host0) * 1e6 / K, 3)}), flush=True)


if __name__ == "__main__":
    main()
