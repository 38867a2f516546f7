"""Synthetic workloads of BASELINE.json's configs.

Saved-activation set = every conv layer's INPUT tensor, fp32 (reproduces the paper's
Table 1 sizes for AlexNet/VGG-16). Data are generated on the device with
a seeded torch generator (Philox), seed 20201118 + tensor index; no datasets or
checkpoints are needed (there is no network). Three kinds (`data`):

* "iid" (default, the bench's and the parity tests' workload): post-ReLU tensors are
  ReLU(N(0,1)) (~50% zeros); conv1 inputs (images) are dense N(0,1);
* "smooth" (SURVEY.md 8(d), config 1's secondary variant): per plane two passes of a 3x3 box
  filter over N(0,1), x3, then ReLU (images: no ReLU);
* "model": the activations of the network itself -- AlexNet (the paper's 96-256-384-384-256
  layout, 227^2 inputs) or VGG-16, random-initialised (Kaiming, seeded), run on smooth
  synthetic images; every conv layer's input is captured. Untrained weights: the
  compression ratio is that of a freshly initialised network, not of a trained one.
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


DATA_KINDS = ("iid", "smooth", "model")


def _smooth(x, post_relu: bool):
    """Two passes of a 3x3 box filter per plane (zero padding), x3, then ReLU."""
    import torch.nn.functional as F
    shp = x.shape
    y = x.reshape(-1, 1, shp[-2], shp[-1])
    for _ in range(2):
        y = F.avg_pool2d(y, 3, stride=1, padding=1, count_include_pad=True)
    y = (y * 3.0).reshape(shp)
    return y.clamp_(min=0.0) if post_relu else y.contiguous()


def make_tensor(shape, post_relu: bool, index: int, device="cuda", data: str = "iid"):
    """Seeded synthetic activation on `device` (torch Philox generator)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(SEED + index)
    x = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
    if data == "smooth" and len(shape) >= 2:
        return _smooth(x, post_relu)
    if post_relu:
        x.clamp_(min=0.0)
    return x


def _model_set(model: str, batch: int, device, seed: int):
    """Conv-layer inputs of a random-initialised AlexNet / VGG-16 forward pass on smooth
    synthetic images (see the module docstring)."""
    import math
    import torch
    import torch.nn.functional as F
    g = torch.Generator(device=device)
    g.manual_seed(SEED + seed)
    side = 227 if model == "alexnet" else 224
    img = _smooth(torch.randn((batch, 3, side, side), generator=g, device=device), False)

    def conv(x, cout, k, stride, pad):
        cin = x.shape[1]
        w = torch.randn((cout, cin, k, k), generator=g, device=device) * math.sqrt(2.0 / (cin * k * k))
        return F.conv2d(x, w, stride=stride, padding=pad)

    outs = []
    with torch.no_grad():
        x = img
        if model == "alexnet":
            # (cout, kernel, stride, pad, max-pool after)
            for cout, k, st, pad, pool in [(96, 11, 4, 0, True), (256, 5, 1, 2, True),
                                           (384, 3, 1, 1, False), (384, 3, 1, 1, False),
                                           (256, 3, 1, 1, False)]:
                outs.append(x.contiguous())
                x = F.relu(conv(x, cout, k, st, pad))
                if pool:
                    x = F.max_pool2d(x, 3, 2)
        else:
            cfg = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M",
                   512, 512, 512]
            for v in cfg:
                if v == "M":
                    x = F.max_pool2d(x, 2, 2)
                    continue
                outs.append(x.contiguous())
                x = F.relu(conv(x, v, 3, 1, 1))
    return outs


def make_set(model: str, batch: int, device="cuda", shard: Tuple[int, int] = (0, 1),
             data: str = "iid"):
    """All saved activations of `model` at `batch`, optionally the rank's batch shard
    (rank, world): samples [rank*B/world, (rank+1)*B/world)."""
    if data not in DATA_KINDS:
        raise ValueError(f"data must be one of {DATA_KINDS}")
    rank, world = shard
    b0, b1 = batch * rank // world, batch * (rank + 1) // world
    spec = activation_set(model)
    if data == "model" and model in ("alexnet", "vgg16"):
        xs = _model_set(model, b1 - b0, device, 7919 * rank)
        return [(name, x) for (name, _, _), x in zip(spec, xs)]
    out = []
    for i, (name, (c, h, w), relu) in enumerate(spec):
        full_idx = i
        x = make_tensor((b1 - b0, c, h, w), relu, full_idx * 1000 + rank, device,
                        "smooth" if data == "model" else data)
        out.append((name, x))
    return out
