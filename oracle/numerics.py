"""Numerics oracle: what one coalesced launch must compute (TEST INFRASTRUCTURE).

The reference never touches tensor data (kernels.py:1-10), so
there is no reference value to pin against: "parity unpinned" w.r.t. the
reference, pinned instead against float64 arithmetic on the SAME rounded
operands the device reads (bf16 operands are widened exactly). Per-op maths
follows the reference's op conventions (kernels.py:45-69):

  gemm (m,n,k):  C[m,n] = act(A[m,:k] @ B[:k,n] + bias[m]), B given as Bt[n,k]
  gemv (m,n):    y[m]   = act(W[m,n] @ x[n] + bias[m])
  elementwise n: y[i]   = act(x[i])

fp32 GEMM operands ("fp32" kernels of the reference, kernels.py:22) are NOT rounded first: the
device reads them as tf32 (tcgen05 kind::tf32) and the reference here is float64 on the
unrounded fp32 values, so the tf32 bound covers the input rounding too.

Tolerances (ours; written into tests/test_exec_gpu.py):
  bf16 output      max|C - ref| <= 4e-3 * max|ref| + 1e-6   (round-to-nearest bf16 output: half an
                   ulp is 2^-8 of the largest value's binade, i.e. up to 3.9e-3 of max|ref|; the
                   survey's 2e-3 cannot hold for bf16 OUTPUTS, and is met by fp32 outputs)
  fp32 output      max|C - ref| <= 1e-4 * max|ref| + 1e-6   (bf16 operands, fp32 accumulation order)
  tf32 (fp32 in)   max|C - ref| <= 5e-3 * max|ref| + 1e-6   (vs unrounded fp32 inputs)
"""

from __future__ import annotations

import math

import numpy as np

BF16_TOL = 4e-3
FP32_TOL = 1e-4
TF32_TOL = 5e-3

_erf = np.vectorize(math.erf, otypes=[np.float64])


def act(x: np.ndarray, kind: str) -> np.ndarray:
    if kind == "relu":
        return np.maximum(x, 0.0)
    if kind == "gelu":
        return 0.5 * x * (1.0 + _erf(x / math.sqrt(2.0)))
    return x


def gemm(a: np.ndarray, bt: np.ndarray, k: int, bias=None, activation="none") -> np.ndarray:
    c = a[:, :k].astype(np.float64) @ bt[:, :k].astype(np.float64).T
    if bias is not None:
        c = c + bias.astype(np.float64)[:, None]
    return act(c, activation)


def gemv(w: np.ndarray, x: np.ndarray, bias=None, activation="none") -> np.ndarray:
    y = w.astype(np.float64) @ x.astype(np.float64)
    if bias is not None:
        y = y + bias.astype(np.float64)
    return act(y, activation)


def elementwise(x: np.ndarray, activation="none") -> np.ndarray:
    return act(x.astype(np.float64), activation)


def rel_err(got: np.ndarray, ref: np.ndarray) -> float:
    scale = float(np.max(np.abs(ref))) if ref.size else 0.0
    return float(np.max(np.abs(got.astype(np.float64) - ref))) / (scale + 1e-30) if ref.size else 0.0


def within(got: np.ndarray, ref: np.ndarray, out_is_bf16: bool, tf32_inputs: bool = False) -> bool:
    tol = max(BF16_TOL if out_is_bf16 else FP32_TOL, TF32_TOL if tf32_inputs else 0.0)
    scale = float(np.max(np.abs(ref))) if ref.size else 0.0
    return bool(np.all(np.isfinite(got))) and \
        float(np.max(np.abs(got.astype(np.float64) - ref), initial=0.0)) <= tol * scale + 1e-6


# ---- CPU reference arm of the bench: the reference-equivalent CPU numerics ---------------

def cpu_step(problems, threads=None):
    """Run a step's members on the host CPU in fp32 (what the CPU path would compute).

    `problems` is a list of (op_kind, dims, arrays) with float32 numpy arrays;
    returns the outputs. Used by bench.py --impl reference.
    """
    out = []
    for op, dims, arr in problems:
        if op == "gemm":
            m, n, k = dims
            out.append(arr["a"][:, :k] @ arr["bt"][:, :k].T)
        elif op == "gemv":
            out.append(arr["a"] @ arr["b"])
        else:
            out.append(np.maximum(arr["a"], 0.0))
    return out
