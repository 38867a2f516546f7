"""BASELINE.json configs 2-5 at their full per-GPU sizes on the B200, checked through
size-independent properties: every tensor of the activation set round-trips
within the error bound (unfiltered), with exact zeros restored and |x - y| <= 2 eb under the
zero filter, the blob parses back to identical bytes, and a one-sample
batch slice of every tensor is byte-identical to the oracle's ACZ1 (planes never straddle
samples, so a slice is an independent codec input: the batch-sharding property of 8(e)).

  config 2: AlexNet saved-activation set, batch 256, eb 1e-3
  config 3: VGG-16 saved-activation set, batch 256, eb pinned over 1e-4 .. 1e-2
  config 4: ResNet-50 batch 512 sharded over 8 GPUs -> the per-GPU shard (batch 64)
  config 5: ResNet-18 batch 1024 over 8 GPUs -> the per-GPU shard (batch 128)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def acz(gpu_lib):
    import torch
    assert torch.cuda.is_available()
    import paper_2011_09017_b200 as acz
    return acz


def _check_set(acz, oracle, model, batch, eb, rank=0, world=1, oracle_slices=True):
    import torch
    from paper_2011_09017_b200 import workloads as W
    named = W.make_set(model, batch, device=torch.device("cuda", 0), shard=(rank, world))
    xs = [x for _, x in named]
    p = acz.CodecParams(eb)
    blobs = acz.compress_many(xs, p)
    raw = acz.decompress_many(blobs, zero_filter=False)
    flt = acz.decompress_many(blobs, zero_filter=True)
    torch.cuda.synchronize()
    total_in = total_out = 0
    for (nm, x), c, y0, y1 in zip(named, blobs, raw, flt):
        assert float((x - y0).abs().max()) <= eb, (model, nm)
        assert float((x - y1).abs().max()) <= 2 * eb, (model, nm)
        assert bool((y1[x == 0] == 0).all()), (model, nm)
        total_in += c.uncompressed_bytes
        total_out += c.compressed_bytes
    # blob serialisation round trip on the largest tensor
    big = max(range(len(blobs)), key=lambda i: blobs[i].element_count())
    b = blobs[big].to_bytes()
    assert acz.blob_from_bytes(b, blobs[big].sidecar()).to_bytes() == b
    if oracle_slices:
        for (nm, x), c in zip(named, blobs):
            sl = x[:1].contiguous()
            ref = oracle.compress(sl.cpu().numpy(), eb)
            assert acz.compress(sl, p).to_bytes() == ref.blob, (model, nm)
    return total_in / total_out


def test_config2_alexnet_b256(acz, oracle):
    ratio = _check_set(acz, oracle, "alexnet", 256, 1e-3)
    assert ratio > 2.5


@pytest.mark.parametrize("eb", [1e-4, 3e-4, 1e-3, 3e-3, 1e-2])
def test_config3_vgg16_b256_eb_sweep(acz, oracle, eb):
    # the controller's bound pinned by eb_min == eb_max (clamp at src/controller.cpp:167)
    from paper_2011_09017_b200.controller import Controller, ControllerConfig
    c = Controller(ControllerConfig(collect_interval=1, eb_min=eb, eb_max=eb), 1)
    c.collect_stats_from_sums(0, [1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 256.0])
    c.begin_iteration(1)
    assert c.layer_eb(0) == eb
    ratio = _check_set(acz, oracle, "vgg16", 256, c.layer_eb(0), oracle_slices=(eb == 1e-3))
    assert ratio > 1.5


def test_config4_resnet50_b512_shard_of_8(acz, oracle):
    _check_set(acz, oracle, "resnet50", 512, 1e-3, rank=3, world=8)


def test_config5_resnet18_b1024_shard_of_8(acz, oracle):
    _check_set(acz, oracle, "resnet18", 1024, 1e-3, rank=5, world=8)
