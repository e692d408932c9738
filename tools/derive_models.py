"""Derive the bundled model library (paper_1901_10008_b200/data/model_library.json).

Two groups of entries:
* the reference's synthetic chains (resnet50_like, lstm_like, ...), restated as
  shapes so `lower_model` is a drop-in for gpumux's bundled names;
* real batch-1 networks lowered offline (no network access needed):
  torchvision resnet50 / mobilenet_v2 (weights=None, 224x224) via forward
  hooks, and BERT-base at seq 128 from its published config.

Lowering convention (gpumux/kernels.py:1-10): a convolution is an
im2col GEMM with m = out channels, n = output pixels (x batch), k = in
channels x kh x kw; a depthwise convolution is billed as an elementwise op over
its output (no GEMM); Linear(in, out) at batch 1 is a gemv(m=out, n=in);
residual adds / softmax / GELU / LayerNorm are elementwise over their outputs.
BatchNorm and ReLU are folded into the producing conv (inference).
"""
import json
import os
import sys

import torch
import torchvision

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_1901_10008_b200", "data", "model_library.json")

SYNTHETIC = {
    "resnet18_conv2_2": ("one ResNet-18 conv2_x 3x3 layer as im2col GEMM", [("gemm", (64, 3136, 576))]),
    "resnet18_conv_chain": ("ResNet-18 conv trunk, im2col GEMMs",
        [("gemm", (64, 12544, 147))] + [("gemm", (64, 3136, 576))] * 4 +
        [("gemm", (128, 784, 576))] + [("gemm", (128, 784, 1152))] * 3 +
        [("gemm", (256, 196, 1152))] + [("gemm", (256, 196, 2304))] * 3 +
        [("gemm", (512, 49, 2304))] + [("gemm", (512, 49, 4608))] * 3),
    "resnet50_like": ("13 representative ResNet-50 conv layers as im2col GEMMs",
        [("gemm", d) for d in [(64, 3136, 147), (64, 3136, 64), (64, 3136, 576), (256, 3136, 64),
                               (128, 784, 256), (128, 784, 1152), (512, 784, 128), (256, 196, 512),
                               (256, 196, 2304), (1024, 196, 256), (512, 49, 1024), (512, 49, 4608),
                               (2048, 49, 512)]]),
    "lstm_like": ("8 chained 1024x1024 recurrent GEMVs", [("gemv", (1024, 1024))] * 8),
    "gemm_64_3136_576": ("single conv2_x GEMM", [("gemm", (64, 3136, 576))]),
    "gemv_1024": ("single 1024x1024 GEMV", [("gemv", (1024, 1024))]),
    "square_gemm_4096": ("4096^3 GEMM", [("gemm", (4096, 4096, 4096))]),
    "square_gemm_4096_k1024": ("4096x4096x1024 GEMM", [("gemm", (4096, 4096, 1024))]),
    "resnet50_fc": ("ResNet-50 classifier head, batch 1", [("gemv", (1000, 2048))]),
}


def lower_cnn(model):
    ops = []
    hooks = []

    def conv_hook(mod, inp, out):
        _, cout, h, w = out.shape
        if mod.groups == 1:
            k = mod.in_channels * mod.kernel_size[0] * mod.kernel_size[1]
            ops.append(("gemm", (cout, h * w, k)))
        elif mod.groups == mod.in_channels == mod.out_channels:
            ops.append(("elementwise", (cout * h * w,)))
        else:
            raise ValueError("grouped conv not supported")

    def lin_hook(mod, inp, out):
        ops.append(("gemv", (mod.out_features, mod.in_features)))

    for m in model.modules():
        if isinstance(m, torch.nn.Conv2d):
            hooks.append(m.register_forward_hook(conv_hook))
        elif isinstance(m, torch.nn.Linear):
            hooks.append(m.register_forward_hook(lin_hook))
    model.eval()
    with torch.no_grad():
        model(torch.zeros(1, 3, 224, 224))
    for h in hooks:
        h.remove()
    return ops


def bert_base(seq=128, hidden=768, layers=12, heads=12, ffn=3072):
    dh = hidden // heads
    ops = []
    for _ in range(layers):
        ops.append(("gemm", (3 * hidden, seq, hidden)))            # fused QKV projection
        ops += [("gemm", (seq, seq, dh))] * heads                   # scores per head
        ops.append(("elementwise", (heads * seq * seq,)))           # softmax
        ops += [("gemm", (dh, seq, seq))] * heads                   # context per head
        ops.append(("gemm", (hidden, seq, hidden)))                 # output projection
        ops.append(("elementwise", (seq * hidden,)))                # residual + LayerNorm
        ops.append(("gemm", (ffn, seq, hidden)))                    # FFN up
        ops.append(("elementwise", (seq * ffn,)))                   # GELU
        ops.append(("gemm", (hidden, seq, ffn)))                    # FFN down
        ops.append(("elementwise", (seq * hidden,)))                # residual + LayerNorm
    return ops


def main():
    models = {}
    for name, (doc, ops) in SYNTHETIC.items():
        models[name] = {"doc": doc, "ops": [[o, list(d), "fp32"] for o, d in ops]}
    real = {
        "resnet50": ("torchvision resnet50, batch 1, 224x224", lower_cnn(torchvision.models.resnet50(weights=None))),
        "mobilenet_v2": ("torchvision mobilenet_v2, batch 1, 224x224; depthwise convs as elementwise",
                         lower_cnn(torchvision.models.mobilenet_v2(weights=None))),
        "bert_base": ("BERT-base encoder, seq 128, batch 1", bert_base()),
    }
    for name, (doc, ops) in real.items():
        for dt in ("fp16", "fp32"):
            key = name if dt == "fp16" else name + "_fp32"
            models[key] = {"doc": doc + f"; dtype {dt}", "ops": [[o, list(d), dt] for o, d in ops]}
    with open(OUT, "w") as fh:
        fh.write('{"format": "gmx-model-library/1", "models": {\n')
        items = list(models.items())
        for i, (name, m) in enumerate(items):
            ops = ",".join(json.dumps(op, separators=(",", ":")) for op in m["ops"])
            sep = "," if i + 1 < len(items) else ""
            fh.write(f' "{name}": {{"doc": {json.dumps(m["doc"])}, "ops": [{ops}]}}{sep}\n')
        fh.write("}}\n")
    for name, m in models.items():
        print(name, len(m["ops"]))


if __name__ == "__main__":
    main()
