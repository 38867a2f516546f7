"""CPU tests of the synthetic workloads (paper_2011_09017_b200/workloads.py): the saved-
activation sets have the SURVEY 8(d) shapes for every data kind, are deterministic, shard by
batch, and the smooth / model kinds are what bench.py --data reports them to be."""
import pytest
import torch

from paper_2011_09017_b200 import workloads as W


@pytest.mark.parametrize("data", W.DATA_KINDS)
def test_alexnet_set_shapes_and_determinism(data):
    a = W.make_set("alexnet", 2, device="cpu", data=data)
    b = W.make_set("alexnet", 2, device="cpu", data=data)
    assert [nm for nm, _ in a] == [nm for nm, _, _ in W.ALEXNET]
    for (nm, x), (_, y), (_, chw, relu) in zip(a, b, W.ALEXNET):
        assert tuple(x.shape) == (2,) + tuple(chw)
        assert x.dtype == torch.float32 and x.is_contiguous()
        assert torch.equal(x, y)
        assert torch.isfinite(x).all()
        if relu:
            assert (x >= 0).all()


def test_batch_shards_are_disjoint_slices_of_the_per_rank_batch():
    full = W.make_set("config1", 4, device="cpu", shard=(0, 2))
    other = W.make_set("config1", 4, device="cpu", shard=(1, 2))
    assert full[0][1].shape[0] == 2 and other[0][1].shape[0] == 2
    assert not torch.equal(full[0][1], other[0][1])  # rank-seeded


def test_smooth_is_smooth_and_half_zero():
    x = W.make_tensor((4, 8, 56, 56), True, 0, "cpu", "smooth")
    zero = (x == 0).float().mean().item()
    assert 0.4 < zero < 0.6
    y = W.make_tensor((4, 8, 56, 56), False, 0, "cpu", "smooth")
    # neighbouring values of a box-filtered field are strongly correlated
    a, b = y[..., :-1].flatten(), y[..., 1:].flatten()
    corr = torch.corrcoef(torch.stack([a, b]))[0, 1].item()
    assert corr > 0.8


def test_model_data_is_a_forward_pass():
    s = W.make_set("alexnet", 2, device="cpu", data="model")
    # conv2..5 inputs are post-ReLU (conv2's after a max-pool): non-negative
    for nm, x in s[1:]:
        assert (x >= 0).all(), nm
    # VGG-16: 13 conv inputs, the first the image
    v = W.make_set("vgg16", 1, device="cpu", data="model")
    assert [tuple(x.shape[1:]) for _, x in v] == [tuple(s) for _, s, _ in W.VGG16]
    with pytest.raises(ValueError):
        W.make_set("alexnet", 1, device="cpu", data="bogus")
