"""GPU tests of the asynchronous compress (acz_gpu_compress_async / _settle; the training
hooks' per-layer path without a host wait): blobs bit-identical to the synchronous compress
and to the oracle, the refit when a blob outgrows its predicted size, errors, and the
controller / training integration giving the same blobs, ledger and gradients as the
synchronous path."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _post_relu(rng, shape):
    return np.maximum(rng.standard_normal(shape), 0).astype(np.float32)


@pytest.mark.parametrize("shape,dense", [((4, 16, 28, 28), False), ((2, 3, 227, 227), True)])
def test_async_matches_sync_and_oracle(gpu_lib, oracle, shape, dense):
    """K2a (post-ReLU planes) and K2b (long dense planes): the first call of a shape runs
    synchronously, later ones are pending until settled; bytes equal the oracle's."""
    import torch
    import paper_2011_09017_b200 as acz
    rng = np.random.default_rng(5)
    ctx = acz.Context(0)
    p = acz.CodecParams(1e-3)
    for k in range(4):
        x = (rng.standard_normal(shape).astype(np.float32) if dense else _post_relu(rng, shape))
        t = torch.from_numpy(x).cuda()
        a = acz.compress_async(t, p, ctx=ctx)
        assert a.pending == (k > 0)
        c = a.settle()
        assert a.refits == 0 and not a.pending
        ref = oracle.compress(x, 1e-3)
        assert c.to_bytes() == ref.blob
        assert c.compressed_bytes == len(ref.blob)
        d = acz.decompress(c, zero_filter=True)
        assert d.cpu().numpy().ravel().tobytes() == oracle.decompress(ref.blob, x.size, True).tobytes()


def test_async_poll_and_many_in_flight(gpu_lib, oracle):
    """Several compresses in flight on one stream (the slot is reused in stream order),
    settled out of a polling loop in order."""
    import torch
    import paper_2011_09017_b200 as acz
    rng = np.random.default_rng(7)
    ctx = acz.Context(0)
    p = acz.CodecParams(1e-3)
    shape = (8, 32, 30, 30)
    acz.compress_async(torch.from_numpy(_post_relu(rng, shape)).cuda(), p, ctx=ctx).settle()
    xs = [_post_relu(rng, shape) for _ in range(6)]
    ops = [acz.compress_async(torch.from_numpy(x).cuda(), p, ctx=ctx) for x in xs]
    assert all(o.pending for o in ops)
    done = [None] * len(ops)
    while any(d is None for d in done):
        for i, o in enumerate(ops):
            if done[i] is None:
                done[i] = o.settle(wait=False)
    for x, c in zip(xs, done):
        assert c.to_bytes() == oracle.compress(x, 1e-3).blob


def test_async_refit_when_the_blob_outgrows_its_prediction(gpu_lib, oracle):
    """A tensor of the same shape but far higher entropy than the one that set the size
    prediction: the speculative encode writes nothing, settle compresses it again
    (exactly), and the next prediction uses the new sizes."""
    import torch
    import paper_2011_09017_b200 as acz
    rng = np.random.default_rng(9)
    ctx = acz.Context(0)
    p = acz.CodecParams(1e-3)
    shape = (4, 16, 40, 40)
    small = (1e-4 * _post_relu(rng, shape)).astype(np.float32)    # mostly one symbol
    # thousands of symbols (a book of <= 8192: larger ones need the host-driven codebook
    # and always take the synchronous path)
    wide = (0.5 * rng.standard_normal(shape)).astype(np.float32)
    acz.compress_async(torch.from_numpy(small).cuda(), p, ctx=ctx).settle()
    a = acz.compress_async(torch.from_numpy(wide).cuda(), p, ctx=ctx)
    assert a.pending
    c = a.settle()
    assert a.refits == 1
    assert c.to_bytes() == oracle.compress(wide, 1e-3).blob
    b = acz.compress_async(torch.from_numpy(wide).cuda(), p, ctx=ctx)
    assert b.pending
    assert b.settle().to_bytes() == c.to_bytes() and b.refits == 0
    # and back to the small tensor: it fits the larger prediction
    s = acz.compress_async(torch.from_numpy(small).cuda(), p, ctx=ctx)
    assert s.settle().to_bytes() == oracle.compress(small, 1e-3).blob and s.refits == 0


def test_async_errors_and_unsettled_blob(gpu_lib):
    import torch
    import paper_2011_09017_b200 as acz
    rng = np.random.default_rng(11)
    ctx = acz.Context(0)
    p = acz.CodecParams(1e-3)
    shape = (2, 8, 20, 20)
    acz.compress_async(torch.from_numpy(_post_relu(rng, shape)).cuda(), p, ctx=ctx).settle()
    x = _post_relu(rng, shape)
    x[1, 3, 5, 7] = np.nan
    a = acz.compress_async(torch.from_numpy(x).cuda(), p, ctx=ctx)
    assert a.pending
    with pytest.raises(acz.DomainError):
        a.settle()
    with pytest.raises(acz.ParamError):
        acz.compress_async(torch.zeros(4, device="cuda"), acz.CodecParams(-1.0), ctx=ctx)
    # an unsettled blob refuses to decompress (ACZ_ERR_INVALID through the C-ABI)
    lib = gpu_lib
    import ctypes as C
    t = torch.from_numpy(_post_relu(rng, shape)).cuda()
    h, pend = C.c_void_p(), C.c_int(0)
    shp = (C.c_uint64 * 4)(*shape)
    assert lib.acz_gpu_compress_async(ctx.handle, C.c_void_p(t.data_ptr()), shp, 4, 1e-3,
                                      32768, 0, 0, None, C.byref(h), C.byref(pend)) == 0
    assert pend.value == 1
    out = torch.empty(shape, device="cuda")
    assert lib.acz_gpu_decompress(ctx.handle, h, 1, C.c_void_p(out.data_ptr()), None) == 8
    st = C.c_int(-1)
    assert lib.acz_gpu_compress_settle(ctx.handle, h, 1, C.byref(st)) == 0 and st.value == 1
    assert lib.acz_gpu_decompress(ctx.handle, h, 1, C.c_void_p(out.data_ptr()), None) == 0
    assert lib.acz_gpu_blob_free(h) == 0
    # a pending blob freed without a settle releases its ring entry
    for _ in range(3):
        a = acz.compress_async(t, p, ctx=ctx)
        del a
    torch.cuda.synchronize()


def _run_controller(async_compress, acts, W=2, iters=6):
    """The controller's four phases over a fixed activation sequence: stats every W
    iterations, every layer wrapped then unwrapped each iteration."""
    import torch
    from paper_2011_09017_b200.controller import Controller, ControllerConfig
    ctl = Controller(ControllerConfig(collect_interval=W, eb_min=1e-4, eb_max=1e-2),
                     len(acts), async_compress=async_compress)
    outs = []
    for it in range(iters):
        ctl.begin_iteration(it)
        if ctl.collecting():
            for i, a in enumerate(acts):
                loss = 1e-3 * torch.ones_like(a)
                mom = (1e-2 * (i + 1)) * torch.ones(16, device="cuda")
                ctl.collect_stats(i, a, loss, mom, a.shape[0])
        hs = [ctl.wrap_forward(i, a, True) for i, a in enumerate(acts)]
        peak_mid = ctl.peak_bytes
        for h in reversed(hs):
            outs.append(ctl.unwrap_backward(h).cpu())
        outs.append(peak_mid)
    ctl.finalize()
    return ctl, outs


def test_controller_async_equals_sync(gpu_lib):
    """Same decompressed activations, byte accounting, peak and ledger CSV with and without
    the asynchronous compress."""
    import torch
    rng = np.random.default_rng(13)
    acts = [torch.from_numpy(_post_relu(rng, s)).cuda()
            for s in [(4, 16, 32, 32), (4, 32, 16, 16), (4, 64, 8, 8)]]
    c0, o0 = _run_controller(False, acts)
    c1, o1 = _run_controller(True, acts)
    assert len(o0) == len(o1)
    for a, b in zip(o0, o1):
        if isinstance(a, int):
            assert a == b
        else:
            assert torch.equal(a, b)
    assert (c0.total_in, c0.total_stored, c0.peak_bytes, c0.current_bytes) == \
        (c1.total_in, c1.total_stored, c1.peak_bytes, c1.current_bytes)
    assert c0.ledger.to_csv() == c1.ledger.to_csv()
    assert c1.refits == 0


def test_training_async_equals_sync(gpu_lib):
    """AdaptiveCompression on a small CNN: losses and weights bit-identical with the
    asynchronous compress on and off (the blobs are the same bytes)."""
    import torch
    import torch.nn as nn
    from paper_2011_09017_b200.controller import ControllerConfig
    from paper_2011_09017_b200.training import AdaptiveCompression
    torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark = True, False

    def run(async_compress, side_stream=False, hw=32, prefetch=False, two_lanes=False):
        torch.manual_seed(3)
        net = nn.Sequential(nn.Conv2d(3, 16, 3, padding=1), nn.ReLU(inplace=True),
                            nn.Conv2d(16, 32, 3, padding=1), nn.ReLU(inplace=True),
                            nn.MaxPool2d(2), nn.Conv2d(32, 32, 3, padding=1), nn.ReLU(),
                            nn.AdaptiveAvgPool2d(1), nn.Flatten(), nn.Linear(32, 10)).cuda()
        opt = torch.optim.SGD(net.parameters(), lr=0.05, momentum=0.9)
        x = torch.randn(16 if hw == 32 else 2, 3, hw, hw, device="cuda",
                        generator=torch.Generator("cuda").manual_seed(1))
        y = torch.randint(0, 10, (x.shape[0],), device="cuda",
                          generator=torch.Generator("cuda").manual_seed(2))
        ac = AdaptiveCompression(net, opt, ControllerConfig(collect_interval=2),
                                 async_compress=async_compress, side_stream=side_stream,
                                 prefetch=prefetch, two_lanes=two_lanes)
        losses = []
        for it in range(7):
            opt.zero_grad(set_to_none=True)
            ac.begin(it)
            with ac.hooks:
                loss = nn.functional.cross_entropy(net(x), y)
            loss.backward()
            ac.end()
            opt.step()
            losses.append(float(loss))
        ac.ctl.finalize()
        return losses, [p.detach().clone() for p in net.parameters()], ac.ctl
    l0, w0, c0 = run(False)
    l1, w1, c1 = run(True)
    l2, w2, c2 = run(True, side_stream=True)
    assert l0 == l1 == l2
    for a, b, c in zip(w0, w1, w2):
        assert torch.equal(a, b) and torch.equal(a, c)
    assert c0.ledger.to_csv() == c1.ledger.to_csv() == c2.ledger.to_csv()
    assert c1.total_stored == c0.total_stored and c1.total_stored < c1.total_in
    assert not math.isnan(l1[-1])
    # 128x128 inputs: the first conv's input goes to the second compress lane (its own
    # context and stream), the rest to the first; unwraps settle out of wrap order
    l3, w3, c3 = run(False, hw=128)
    l4, w4, c4 = run(True, side_stream=True, hw=128, prefetch=True, two_lanes=True)
    assert l3 == l4 and all(torch.equal(a, b) for a, b in zip(w3, w4))
    assert c3.ledger.to_csv() == c4.ledger.to_csv()
    assert c4._lanes[0] is not None and c4._lanes[1] is not None
    assert (c3.peak_bytes, c3.total_stored) == (c4.peak_bytes, c4.total_stored)


def test_k2b_learned_dispatch_at_large_error_bounds(gpu_lib, oracle):
    """Long dense planes at eb = 0.1 (the controller's default eb_max): K2b's walk leaves most
    planes to the serial replay, so the context quantises the next compress of the same
    (shape, eb) with K2a (fewer launches); both are bit-exact. At eb = 1e-3 K2b stays."""
    import os
    import torch
    import paper_2011_09017_b200 as acz
    assert "ACZ_SPEC_QUANT" not in os.environ and "ACZ_SERIAL_QUANT" not in os.environ
    rng = np.random.default_rng(17)
    ctx = acz.Context(0)
    for eb, learns in ((0.1, True), (1e-3, False)):
        launches = []
        for _ in range(3):
            x = rng.standard_normal((4, 3, 224, 224)).astype(np.float32)
            l0 = ctx.launches
            c = acz.compress(torch.from_numpy(x).cuda(), acz.CodecParams(eb), ctx=ctx)
            launches.append(ctx.launches - l0)
            assert c.to_bytes() == oracle.compress(x, eb).blob
        if learns:
            assert launches[1] < launches[0] and launches[2] == launches[1], launches
        else:
            assert launches[0] == launches[1] == launches[2], launches


def test_async_size_tags_keep_equal_shapes_apart(gpu_lib, oracle):
    """Two layers with the same input shape but different entropy, compressed alternately:
    tagged by layer, each predicts from its own previous blob (no refits); untagged, the
    larger one outgrows the smaller one's prediction every time."""
    import torch
    import paper_2011_09017_b200 as acz
    rng = np.random.default_rng(19)
    ctx = acz.Context(0)
    p = acz.CodecParams(1e-3)
    shape = (4, 16, 40, 40)
    lo = (0.05 * _post_relu(rng, shape)).astype(np.float32)
    hi = _post_relu(rng, shape)
    refits = {True: 0, False: 0}
    for tagged in (True, False):
        for _ in range(3):
            for tag, x in ((1, lo), (2, hi)):
                a = acz.compress_async(torch.from_numpy(x).cuda(), p, ctx=ctx,
                                       size_tag=tag if tagged else 99)
                assert a.settle().to_bytes() == oracle.compress(x, 1e-3).blob
                refits[tagged] += a.refits
    assert refits[True] == 0 and refits[False] >= 2, refits


def test_async_lorenzo_and_edge_cases(gpu_lib, oracle):
    """Lorenzo2d has no size prediction: compress_async is the synchronous compress; empty
    tensors raise what compress() raises; the ring of pending entries is returned on every
    settle over many calls."""
    import torch
    import paper_2011_09017_b200 as acz
    rng = np.random.default_rng(23)
    ctx = acz.Context(0)
    x = _post_relu(rng, (2, 4, 33, 47))
    p = acz.CodecParams(1e-3, predictor=acz.Predictor.Lorenzo2d)
    for _ in range(2):
        a = acz.compress_async(torch.from_numpy(x).cuda(), p, ctx=ctx)
        assert not a.pending
        assert a.settle().to_bytes() == oracle.compress(x, 1e-3, predictor=1).blob
    for bad in (torch.empty(0, device="cuda"), torch.empty(3, 0, 4, device="cuda")):
        with pytest.raises(acz.Error) as sync_err:
            acz.compress(bad, acz.CodecParams(1e-3), ctx=ctx)
        with pytest.raises(type(sync_err.value)):
            acz.compress_async(bad, acz.CodecParams(1e-3), ctx=ctx)
    q = acz.CodecParams(1e-3)
    t = torch.from_numpy(_post_relu(rng, (2, 8, 16, 16))).cuda()
    for k in range(1200):  # more than the 1024-entry ring: entries are returned on settle
        a = acz.compress_async(t, q, ctx=ctx, size_tag=k % 3)
        a.settle()
