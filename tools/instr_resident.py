"""Where does a resident C2 step's time go, per role? Builds the executor with -DGMX_INSTR (see
`timed` / `instr_dump` in csrc/exec/gmx_exec.cu) and reports, per CTA, the time each role of the
persistent kernel spent waiting on its inputs during a held batch of C2 steps.

usage: python tools/instr_resident.py --build          (here: compile the profiling build)
       python tools/instr_resident.py [opt=v ...]      (GPU: run it; executor options as k=v)
"""
import ctypes as C
import os
import statistics
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(REPO, "paper_1901_10008_b200", "lib", "instr")
NAMES = ["p_unit", "p_empty", "m_unit", "m_tempty", "m_full", "e_unit", "e_tfull", "s_uempty", "s_pub",
         "s_order", "s_lists", "p_stages", "e_staged", "e_split", "e_complete", "e_acct", "a_bar", "a_wait", "a_red", "x_next", "x_ld", "x_stage", "x_bar2", "x_issue"]


def build():
    sys.path.insert(0, REPO)
    from paper_1901_10008_b200 import _build
    core = _build.build_core()
    os.makedirs(OUT, exist_ok=True)
    subprocess.check_call(["cp", core, OUT])
    exec_dir = os.path.join(REPO, "paper_1901_10008_b200", "csrc", "exec")
    srcs = [os.path.join(exec_dir, f) for f in sorted(os.listdir(exec_dir)) if f.endswith((".cu", ".cpp"))]
    subprocess.check_call([_build.nvcc_path(), *_build.NVCC_ARCH, "-O3", "-std=c++17", "-lineinfo", "-shared",
                           "-DGMX_INSTR", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
                           "--expt-relaxed-constexpr", "-cudart", "static", "-I", _build.INCLUDE, *srcs,
                           "-o", os.path.join(OUT, "libgmx_exec.so"), "-L", OUT, "-lgmx_core",
                           "-Xlinker", "-rpath,$ORIGIN", "-ldl"])


def run(opts, steps=400):
    sys.path.insert(0, REPO)
    from paper_1901_10008_b200 import executor
    executor.exec_lib(os.path.join(OUT, "libgmx_exec.so"))
    from bench import C2Bench, time_resident
    b = C2Bench(replicas=16)
    for k, v in opts.items():
        b.ex.set_option(k, v)
    rows = (len(NAMES) + 7) // 8
    b.ex.set_option("rtrace", steps + rows)
    _, t, _ = time_resident(b, steps)
    grid = C.c_int32()
    buf = (C.c_uint64 * ((steps + rows) * 148 * 8 + 2 * (steps + rows)))()
    rc = b.ex._lib.gmx_exec_resident_read_rtrace(b.ex._h, buf, len(buf), C.byref(grid))
    assert rc == 0
    G = grid.value
    row = lambda f, c: buf[((steps + (f // 8)) * G + c) * 8 + f % 8]
    print(f"per-step {t * 1e6:.3f} us {opts}; per step per CTA (median / min / max; us unless a count):")
    for f, n in enumerate(NAMES):
        div = steps if n in ("s_lists", "p_stages") else 1965.0 * steps   # SM clock at 1965 MHz
        xs = [row(f, c) / div for c in range(G)]
        print(f"  {n:9s} {statistics.median(xs):8.3f} {min(xs):8.3f} {max(xs):8.3f}")


if __name__ == "__main__":
    if "--build" in sys.argv:
        build()
    else:
        run({k: int(v) for k, v in (a.split("=") for a in sys.argv[1:])})
