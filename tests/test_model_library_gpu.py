"""The derived model library (data/model_library.json: torchvision ResNet-50 / MobileNetV2 and
BERT-base at seq 128, tools/derive_models.py) through the native serving loop on the B200:
the reference's model-library format and lowering (kernels.py:157-199, a linear dependency
chain per request) with this package's library plumbed in (`library=`, engine.py:188 does not
plumb one). Every request's completion time must equal the oracle engine's (oracle/sim.py,
pinned to gpumux) on the same workload, over both executors, and every member's output must
match float64 on its operands (bf16 4e-3, tf32 5e-3; oracle/numerics.py)."""

import pytest

pytestmark = pytest.mark.gpu

from .test_runtime_gpu import _run_workload  # noqa: E402


def _library():
    import paper_1901_10008_b200 as gm
    return gm.kernels.load_model_library()


@pytest.mark.parametrize("resident", [False, True])
def test_c3_mixed_models_bf16(resident):
    """ResNet-50 + BERT-base + MobileNetV2, batch 1, 10 ms SLO, staggered."""
    lib = _library()
    wl = {"duration_ns": 20_000_000, "streams": [
        {"stream_id": sid, "model_name": m, "slo_ns": 10_000_000,
         "arrival": {"kind": "fixed", "schedule": [t0, t0 + 5_000_000]}}
        for sid, m, t0 in [("resnet50", "resnet50", 0), ("bert", "bert_base", 30_000),
                           ("mobilenet", "mobilenet_v2", 70_000)]]}
    stats = _run_workload(wl, lib, resident=resident)
    assert stats["completed_requests"] == 6
    assert stats["kernels"] == 2 * (54 + 384 + 53)


@pytest.mark.parametrize("model", ["resnet50_fp32", "mobilenet_v2_fp32"])
def test_fp32_models_on_the_tf32_path(model):
    """fp32 variants (GEMMs as tf32 UMMA on unrounded fp32 operands; GEMV/elementwise fp32)."""
    lib = _library()
    wl = {"duration_ns": 10_000_000, "streams": [
        {"stream_id": f"s{i}", "model_name": model, "slo_ns": 10_000_000,
         "arrival": {"kind": "fixed", "schedule": [i * 20_000]}} for i in range(2)]}
    stats = _run_workload(wl, lib)
    assert stats["completed_requests"] == 2
