"""Synthetic workloads of BASELINE.json's configs.

Saved-activation set = every conv layer's INPUT tensor, fp32 (reproduces the paper's
Table 1 sizes for AlexNet/VGG-16). Post-ReLU tensors are ReLU(N(0,1))
(~50% zeros); conv1 inputs (images) are dense N(0,1). Data are generated on the device with
a seeded torch generator (Philox), seed 20201118 + tensor index; no datasets or
checkpoints are needed (there is no network).
"""
from __future__ import annotations

from typing import List, Tuple

SEED = 20201118

# (name, per-sample shape (C,H,W), post_relu)
ALEXNET = [("conv1_in", (3, 227, 227), False), ("conv2_in", (96, 27, 27), True),
           ("conv3_in", (256, 13, 13), True), ("conv4_in", (384, 13, 13), True),
           ("conv5_in", (384, 13, 13), True)]

_VGG_CFG = [(3, 224, False), (64, 224, True), (64, 112, True), (128, 112, True),
            (128, 56, True), (256, 56, True), (256, 56, True), (256, 28, True),
            (512, 28, True), (512, 28, True), (512, 14, True), (512, 14, True),
            (512, 14, True)]
VGG16 = [(f"conv{i + 1}_in", (c, h, h), r) for i, (c, h, r) in enumerate(_VGG_CFG)]


def resnet18_inputs() -> List[Tuple[str, Tuple[int, int, int], bool]]:
    """torchvision ResNet-18 conv inputs (v1.5 layout incl. downsample convs)."""
    out = [("conv1_in", (3, 224, 224), False)]
    c, h = 64, 56
    for stage, (cout, stride) in enumerate([(64, 1), (128, 2), (256, 2), (512, 2)]):
        for blk in range(2):
            s = stride if blk == 0 else 1
            out.append((f"l{stage + 1}b{blk}c1_in", (c, h, h), True))
            h2 = h // s
            out.append((f"l{stage + 1}b{blk}c2_in", (cout, h2, h2), True))
            if blk == 0 and (s != 1 or c != cout):
                out.append((f"l{stage + 1}b{blk}ds_in", (c, h, h), True))
            c, h = cout, h2
    return out


def resnet50_inputs() -> List[Tuple[str, Tuple[int, int, int], bool]]:
    """torchvision ResNet-50 (v1.5: stride in the 3x3) conv inputs incl. downsample."""
    out = [("conv1_in", (3, 224, 224), False)]
    c, h = 64, 56
    for stage, (mid, blocks, stride) in enumerate([(64, 3, 1), (128, 4, 2), (256, 6, 2),
                                                   (512, 3, 2)]):
        cout = mid * 4
        for blk in range(blocks):
            s = stride if blk == 0 else 1
            out.append((f"l{stage + 1}b{blk}c1_in", (c, h, h), True))
            out.append((f"l{stage + 1}b{blk}c2_in", (mid, h, h), True))
            h2 = h // s
            out.append((f"l{stage + 1}b{blk}c3_in", (mid, h2, h2), True))
            if blk == 0:
                out.append((f"l{stage + 1}b{blk}ds_in", (c, h, h), True))
            c, h = cout, h2
    return out


CONFIG1 = [("relu_64x64x56x56", (64, 56, 56), True)]  # batch 64


def activation_set(model: str):
    return {"alexnet": ALEXNET, "vgg16": VGG16, "resnet18": resnet18_inputs(),
            "resnet50": resnet50_inputs(), "config1": CONFIG1}[model]


def set_bytes(model: str, batch: int) -> int:
    tot = 0
    for _, (c, h, w), _ in activation_set(model):
        tot += batch * c * h * w * 4
    return tot


def make_tensor(shape, post_relu: bool, index: int, device="cuda"):
    """Seeded synthetic activation on `device` (torch Philox generator)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(SEED + index)
    x = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
    if post_relu:
        x.clamp_(min=0.0)
    return x


def make_set(model: str, batch: int, device="cuda", shard: Tuple[int, int] = (0, 1)):
    """All saved activations of `model` at `batch`, optionally the rank's batch shard
    (rank, world): samples [rank*B/world, (rank+1)*B/world)."""
    rank, world = shard
    b0, b1 = batch * rank // world, batch * (rank + 1) // world
    out = []
    for i, (name, (c, h, w), relu) in enumerate(activation_set(model)):
        full_idx = i
        x = make_tensor((b1 - b0, c, h, w), relu, full_idx * 1000 + rank, device)
        out.append((name, x))
    return out
