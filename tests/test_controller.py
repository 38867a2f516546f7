"""CPU tests of the adaptive error-bound controller (paper_2011_09017_b200/controller.py)
against the UNMODIFIED reference Controller (src/controller.cpp, compiled into
oracle/_ref), and of the distributed statistics (one all-reduce of 7 doubles per layer)
with world_size 2 over gloo."""
import math
import os
import socket

import numpy as np
import pytest


def _data(seed, batch=6):
    rng = np.random.default_rng(seed)
    act = np.maximum(rng.standard_normal((batch, 8, 14, 14)), 0).astype(np.float32)
    loss = (1e-3 * rng.standard_normal((batch, 8, 14, 14))).astype(np.float32)
    mom = (1e-2 * rng.standard_normal((16, 8, 3, 3))).astype(np.float32)
    return act, loss, mom


def _csv_rows(text):
    lines = text.strip().split("\n")
    return lines[0], [[float(v) for v in l.split(",")] for l in lines[1:]]


@pytest.mark.parametrize("seed,kw", [(1, {}), (2, dict(sigma_fraction=0.05, coefficient_a=0.5)),
                                     (3, dict(eb_min=1e-3, eb_max=1e-3)),
                                     (4, dict(eb_max=1e-7, eb_min=1e-8))])
def test_controller_matches_reference(reference, seed, kw):
    import torch
    from paper_2011_09017_b200.controller import Controller, ControllerConfig
    act, loss, mom = _data(seed)
    ref = reference.controller_run(act, loss, mom, batch=act.shape[0], W=4, **kw)
    cfg = ControllerConfig(collect_interval=4, **kw)
    c = Controller(cfg, 1)
    c.begin_iteration(0)
    st = c.collect_stats(0, torch.from_numpy(act), torch.from_numpy(loss), torch.from_numpy(mom),
                         act.shape[0])
    assert st.r == ref["r"]                                   # exact count ratio
    assert math.isclose(st.l_bar, ref["l_bar"], rel_tol=1e-12)  # parallel vs sequential sum
    assert math.isclose(st.m_avg, ref["m_avg"], rel_tol=1e-12)
    assert st.degenerate == ref["degenerate"]
    assert not c.layer_active(0)
    c.begin_iteration(1)
    assert c.layer_active(0) == ref["active"]
    assert math.isclose(c.layer_eb(0), ref["eb"], rel_tol=1e-12)
    c.finalize()
    h_ref, rows_ref = _csv_rows(ref["csv"])
    h, rows = _csv_rows(c.ledger.to_csv())
    assert h == h_ref and len(rows) == len(rows_ref) == 1
    for a, b in zip(rows[0], rows_ref[0]):
        assert math.isclose(a, b, rel_tol=1e-12, abs_tol=0.0)


def test_controller_degenerate_and_errors(reference):
    import torch
    from paper_2011_09017_b200 import ParamError
    from paper_2011_09017_b200.controller import Controller, ControllerConfig, suggest_batch
    act, loss, mom = _data(5)
    zero = np.zeros_like(act)
    ref = reference.controller_run(zero, loss, mom, batch=6, W=2)
    c = Controller(ControllerConfig(collect_interval=2), 1)
    st = c.collect_stats(0, torch.from_numpy(zero), torch.from_numpy(loss), torch.from_numpy(mom), 6)
    assert st.degenerate and ref["degenerate"]
    c.begin_iteration(1)
    assert not c.layer_active(0) and not ref["active"]
    with pytest.raises(ParamError):
        c.collect_stats(0, torch.from_numpy(act), torch.from_numpy(loss), torch.from_numpy(mom), 6)
    for bad in (dict(collect_interval=0), dict(sigma_fraction=0.0), dict(coefficient_a=-1.0),
                dict(eb_min=1e-2, eb_max=1e-3), dict(quant_radius=1000)):
        with pytest.raises(ParamError):
            Controller(ControllerConfig(**bad), 1)
    h = c.wrap_forward(0, torch.from_numpy(act), True)  # inactive layer: pass-through
    assert h.raw is not None and h.held_bytes == act.nbytes
    assert c.unwrap_backward(h) is not None and c.current_bytes == 0
    assert suggest_batch(256, 1000 << 20, 4000 << 20) == 1024


def _worker(rank, world, port, shards, full, q):
    import torch
    import torch.distributed as dist
    from paper_2011_09017_b200.controller import (Controller, ControllerConfig, DistributedStats,
                                                  local_stat_sums)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    act, loss, mom = shards[rank]
    c = Controller(ControllerConfig(collect_interval=1), 1, reducer=DistributedStats())
    c.begin_iteration(0)
    sums = local_stat_sums(torch.from_numpy(act), torch.from_numpy(loss), torch.from_numpy(mom),
                           act.shape[0])
    # momentum is replicated over DP ranks: each rank contributes it once; the mean is unchanged
    st = c.collect_stats_from_sums(0, sums)
    c.begin_iteration(1)
    q.put((rank, st.l_bar, st.r, st.m_avg, st.batch, c.layer_eb(0)))
    dist.barrier()
    dist.destroy_process_group()


def test_distributed_stats_gloo():
    """world_size 2 over gloo: the all-reduced statistics of the batch shards equal the
    statistics of the whole batch (up to summation order), identically on both ranks."""
    import torch.multiprocessing as mp
    from paper_2011_09017_b200.controller import Controller, ControllerConfig, local_stat_sums
    import torch
    act, loss, mom = _data(9, batch=8)
    shards = [(act[:4], loss[:4], mom), (act[4:], loss[4:], mom)]
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shards, None, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = Controller(ControllerConfig(collect_interval=1), 1)
    st = single.collect_stats(0, torch.from_numpy(act), torch.from_numpy(loss),
                              torch.from_numpy(mom), 8)
    single.begin_iteration(1)
    (_, l0, r0, m0, b0, e0), (_, l1, r1, m1, b1, e1) = res
    assert (l0, r0, m0, b0, e0) == (l1, r1, m1, b1, e1)      # identical on every rank
    assert b0 == 8 and r0 == st.r
    assert math.isclose(l0, st.l_bar, rel_tol=1e-12) and math.isclose(m0, st.m_avg, rel_tol=1e-12)
    assert math.isclose(e0, single.layer_eb(0), rel_tol=1e-12)


class _FakeBlob:
    def __init__(self, nbytes):
        self.compressed_bytes = nbytes


class _FakeAsync:
    """Stands in for codec.AsyncCompress (host logic only): done after `ready_after` polls."""
    log = []

    def __init__(self, t, nbytes, ready_after):
        self._t, self.n, self.polls, self.ready_after = t, nbytes, 0, ready_after
        self.pending, self.refits, self.refit_reason = True, 0, ""

    def settle(self, wait=True):
        self.polls += 1
        if not wait and self.polls <= self.ready_after:
            return None
        _FakeAsync.log.append(self.n)
        self.pending = False
        self._t = None
        return _FakeBlob(self.n)


def test_controller_async_settle_order_and_bound(monkeypatch):
    """The asynchronous path's host logic without a GPU: handles settle in wrap order (a
    finished newer one waits for an unfinished older one), at most max_pending stay
    unsettled (their raw activations alive), the byte accounting and window sums equal the
    synchronous path's, and unwrap settles everything first."""
    import torch
    from paper_2011_09017_b200 import codec as K
    from paper_2011_09017_b200.controller import Controller, ControllerConfig
    sizes = [5000, 100, 3000, 700, 40, 9000]
    ready = [3, 0, 0, 5, 0, 0]  # polls before each one reports finished (wait=False)
    it = iter(zip(sizes, ready))

    def fake_async(t, p, stream=None, ctx=None, size_tag=0):
        n, r = next(it)
        return _FakeAsync(t, n, r)
    monkeypatch.setattr(K, "compress_async", fake_async)
    monkeypatch.setattr(K, "compression_ratio", lambda c: 1.0)
    _FakeAsync.log = []

    def active(ctl):
        for i in range(len(sizes)):
            ctl.collect_stats_from_sums(i, [1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 8.0])
        ctl.begin_iteration(1)

    c = Controller(ControllerConfig(collect_interval=100, eb_min=1e-3, eb_max=1e-3), len(sizes),
                   async_compress=True, max_pending=2)
    active(c)
    acts = [torch.zeros(1000 * (i + 1)) for i in range(len(sizes))]
    hs = []
    for i, a in enumerate(acts):
        hs.append(c.wrap_forward(i, a, False))
        assert len(c._pending) <= 2
    assert _FakeAsync.log == sizes[:len(_FakeAsync.log)]  # settled strictly in wrap order
    assert c.current_bytes == sum(sizes)                   # (reading it settles the rest)
    assert _FakeAsync.log == sizes and not c._pending
    assert c.total_in == sum(4 * a.numel() for a in acts) and c.peak_bytes == sum(sizes)
    assert all(h.blob is not None and h.zero_filter and h.pending is None for h in hs)

    # unwrap settles only its own handle: the newest one is unwrapped while older ones are
    # still compressing; the accounting still follows program order (peak after all wraps)
    monkeypatch.setattr(K, "decompress", lambda b, zero_filter=False, ctx=None: torch.zeros(1))
    it = iter(zip(sizes, [9, 9, 9, 9, 9, 0]))
    _FakeAsync.log = []
    c2 = Controller(ControllerConfig(collect_interval=100, eb_min=1e-3, eb_max=1e-3),
                    len(sizes), async_compress=True, max_pending=len(sizes))
    active(c2)
    hs = [c2.wrap_forward(i, a, False) for i, a in enumerate(acts)]
    c2.unwrap_backward(hs[-1])
    assert _FakeAsync.log == [sizes[-1]] and c2._cur == 0  # nothing accounted yet
    assert c2.current_bytes == sum(sizes) - sizes[-1] and c2.peak_bytes == sum(sizes)
    for h in reversed(hs[:-1]):
        c2.unwrap_backward(h)
    assert c2.current_bytes == 0 and c2.total_stored == sum(sizes)
