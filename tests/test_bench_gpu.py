"""bench.py's own command line on the GPU (the driver's `bench.py --gpus 1 --steps K --warmup W`,
shortened with --quick, which skips the comparators and the CPU baseline): one JSON line with the
contract's keys, a device-timed window of exactly K steps, the roofline object computed from the
CUDA-event held batch, an e2e figure with the bytes it moved, and the timed region's last round
checked against the numerics oracle inside bench.py (no `parity_failures`)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_command_line_contract():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "1", "--steps", "8",
                          "--warmup", "3", "--quick"], capture_output=True, text=True, timeout=600, env=env,
                         cwd=REPO)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 8 and d["warmup"] == 3 and d["dtype"] == "bf16"
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] >= 1
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1 and r["achieved"] < r["peak"]
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert "parity_failures" not in d, d.get("parity_failures")
