"""Is a lone memory-bound kernel slow on this box regardless of our kernel? torch copies of
16/32/64/256 MB (rotating over buffers > L2) timed with CUDA events: (a) queued behind a sleep
kernel (memory idle before), (b) back to back (steady state)."""
import statistics
import torch

torch.cuda.init()
s = torch.cuda.current_stream()
for mb in (16, 32, 64, 256):
    n = mb * (1 << 20) // 4
    bufs = [(torch.empty(n, device="cuda"), torch.empty(n, device="cuda")) for _ in range(8)]
    for a, b in bufs:
        b.copy_(a)
    torch.cuda.synchronize()
    lone = []
    for j in range(24):
        a, b = bufs[j % 8]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        e0.record(s)
        b.copy_(a)
        e1.record(s)
        torch.cuda.synchronize()
        lone.append(e0.elapsed_time(e1) * 1e3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for j in range(64):
        a, b = bufs[j % 8]
        b.copy_(a)
    e1.record(s)
    torch.cuda.synchronize()
    steady = e0.elapsed_time(e1) * 1e3 / 64
    print(f"{mb} MB copy (read+write {2*mb} MB): lone median {statistics.median(lone):.2f} us "
          f"({2 * mb * 1.048576 / statistics.median(lone):.2f} TB/s), back-to-back {steady:.2f} us "
          f"({2 * mb * 1.048576 / steady:.2f} TB/s)")
