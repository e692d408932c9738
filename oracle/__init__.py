"""CPU oracle for the spatial-coalescing hot path — TEST INFRASTRUCTURE ONLY.

Nothing under `oracle/` is part of the product. Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU-baseline / reference arm may
import it, and only as the checker (or as the timed CPU reference arm), never
as the thing measured on the GPU or shipped.

* `oracle.decisions` — a plain-Python restatement of the reference decision
  layer (`gpumux` 0.1.0: kernels/device/tuning/coalesce/scheduler), every
  function citing the reference file:line it follows.
* `oracle.sim` — a restatement of the reference discrete-event loop and its
  metrics (`gpumux/engine.py`), used as the trace-parity harness when the
  reference itself is not importable (e.g. on the GPU box).
* `oracle.numerics` — numpy restatement of what a coalesced launch computes
  (GEMM / GEMV / elementwise on the same rounded operands).

Parity pinning: `tests/golden/make_golden.py` runs the real reference
(`/root/reference/pkg/src/gpumux`) in the build container and commits its
outputs as fixtures; `tests/test_oracle_golden.py` checks this oracle against
them. The numerics oracle has no reference counterpart (the reference never
touches tensor data), so GEMM values are "parity unpinned"
against the reference and pinned instead against float64 arithmetic.
"""
