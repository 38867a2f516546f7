"""Adaptive error-bound controller for PyTorch training (host side, ref
proj/core/include/acz/controller.hpp:14-155, src/controller.cpp:14-253), mirroring the C++
controller of cpp/acz_b200.hpp.

Four phases (section 4): every W iterations collect L_bar (mean |loss gradient|),
R (nonzero ratio of the activation) and M_avg (mean |momentum|) per layer; derive
sigma = sigma_fraction * M_avg; invert the estimator into eb = sigma / (a * L_bar *
sqrt(N * R)) clamped to [eb_min, eb_max]; compress every stashed activation of the layer
with that bound until the next collection (the collection iteration itself and degenerate
windows pass through).

Multi-GPU: data-parallel ranks compress their own activations with no
collective on the data path. The statistics become global with ONE all-reduce of 7 doubles
per layer every W iterations (sums of |loss|, loss count, nonzeros, activation count,
|momentum|, momentum count, batch) -- :class:`DistributedStats`. The batch-size scheme of
BASELINE config 5 (not implemented by the reference) is
:func:`suggest_batch`.
"""
from __future__ import annotations

import math
import sys
from dataclasses import dataclass, field
from typing import Callable, List, Optional

from . import codec as _codec

ZERO_FILTER = "codec-filter"
RELU_RECOMPUTE = "relu-recompute"


@dataclass
class ControllerConfig:
    collect_interval: int = 1000     # W
    sigma_fraction: float = 0.01
    coefficient_a: float = 0.32
    eb_min: float = 1e-8
    eb_max: float = 1e-1
    zero_restoration: str = ZERO_FILTER
    predictor: int = 0
    quant_radius: int = 32768

    def validate(self) -> None:
        """ref src/controller.cpp:14-21"""
        if self.collect_interval < 1:
            raise _codec.ParamError("collect_interval (W) must be >= 1")
        if not self.sigma_fraction > 0.0:
            raise _codec.ParamError("sigma_fraction must be positive")
        if not self.coefficient_a > 0.0:
            raise _codec.ParamError("coefficient_a must be positive")
        if not (self.eb_min > 0.0 and self.eb_min <= self.eb_max):
            raise _codec.ParamError("error-bound clamps must satisfy 0 < eb_min <= eb_max")
        if self.zero_restoration not in (ZERO_FILTER, RELU_RECOMPUTE):
            raise _codec.ParamError("zero_restoration must be codec-filter or relu-recompute")
        _codec.CodecParams(self.eb_min, self.quant_radius, self.predictor).validate()


@dataclass
class LayerStats:
    layer_id: int = -1
    l_bar: float = 0.0
    r: float = 0.0
    m_avg: float = 0.0
    batch: int = 0
    collected_at: int = -1
    degenerate: bool = False


@dataclass
class LedgerRecord:
    iteration: int
    layer_id: int
    eb: float
    predicted_sigma: float
    l_bar: float
    r: float
    m_avg: float
    ratio: float
    fallback: bool


class CompressionLedger:
    def __init__(self):
        self.records: List[LedgerRecord] = []

    def append(self, r: LedgerRecord) -> None:
        self.records.append(r)

    def to_csv(self) -> str:
        """ref src/controller.cpp:67-76 (same header, %.17g formatting)."""
        out = ["iteration,layer,eb,predicted_sigma,L_bar,R,M_avg,ratio,fallback_flag\n"]
        for r in self.records:
            out.append("%d,%d,%.17g,%.17g,%.17g,%.17g,%.17g,%.17g,%d\n" % (
                r.iteration, r.layer_id, r.eb, r.predicted_sigma, r.l_bar, r.r, r.m_avg, r.ratio,
                1 if r.fallback else 0))
        return "".join(out)


@dataclass
class ActivationHandle:
    """Exactly one of raw / blob is engaged (ref include/acz/controller.hpp:65-78)."""
    raw: object = None
    blob: Optional[_codec.CompressedTensor] = None
    apply_relu: bool = False
    zero_filter: bool = False
    layer_id: int = -1
    held_bytes: int = 0
    achieved_ratio: float = 1.0
    # asynchronous compress in flight (Controller(async_compress=True)); settled -- blob,
    # sizes and accounting filled in -- before anything reads the handle
    pending: Optional[_codec.AsyncCompress] = None
    post_relu: bool = False
    in_bytes: int = 0
    side: object = None  # the stream its blob was compressed (and will be freed) on
    prefetched: object = None  # (tensor, event) decoded ahead (Controller(prefetch=True))
    stored_bytes: int = 0  # held_bytes as wrapped (for the deferred accounting)


@dataclass
class _Window:
    stats: LayerStats = field(default_factory=LayerStats)
    eb: float = 0.0
    sigma: float = 0.0
    fallback: bool = True
    open: bool = False
    bytes_in: int = 0
    bytes_stored: int = 0


def local_stat_sums(activation, loss, momentum, batch: int) -> List[float]:
    """The 7 per-layer sums of one rank: sum|loss|, #loss, #nonzero(act), #act, sum|mom|,
    #mom, batch. CUDA tensors go through the codec's GPU statistics kernels (K1); CPU tensors
    (tests, CPU ranks) are summed in double by torch."""
    import torch
    if activation.is_cuda:
        nz = int(_codec.zero_bitmap(activation)[1])
        la = _codec.mean_abs(loss) * loss.numel()
        ma = _codec.mean_abs(momentum) * momentum.numel()
    else:
        nz = int(torch.count_nonzero(activation).item())
        la = float(loss.detach().double().abs().sum().item())
        ma = float(momentum.detach().double().abs().sum().item())
    return [la, float(loss.numel()), float(nz), float(activation.numel()), ma,
            float(momentum.numel()), float(batch)]


class DistributedStats:
    """Sum-reduces the 7 statistics sums over the data-parallel group (torch.distributed;
    NCCL on GPUs, gloo on CPU): the only collective of the compressor."""

    def __init__(self, group=None):
        self.group = group

    def __call__(self, sums: List[float]) -> List[float]:
        import torch
        import torch.distributed as dist
        if not (dist.is_available() and dist.is_initialized()):
            return sums
        dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor(sums, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return [float(v) for v in t.cpu().tolist()]


class Controller:
    """ref src/controller.cpp:94-253 over torch CUDA activations."""

    def __init__(self, cfg: ControllerConfig, num_layers: int,
                 reducer: Optional[Callable[[List[float]], List[float]]] = None,
                 ctx: Optional[_codec.Context] = None, async_compress: bool = False,
                 side_stream: bool = False, max_pending: int = 4, prefetch: bool = False,
                 two_lanes: bool = False):
        """async_compress: wrap_forward enqueues the compress without waiting for its
        codebook (codec.compress_async); handles are settled as they finish (in wrap order),
        an unwrap settles its own handle, and everything is settled before a window change,
        a ledger write or a read of the byte counters; the byte accounting is replayed in
        program order, so blobs, ledger and counters are those of the synchronous path.
        side_stream (with async_compress): the compresses run on side streams that wait for
        the activation's producer, so the forward pass does not queue behind them; long
        planes (an input image) get a second lane (stream + context) so that their
        latency-bound quantiser does not hold back the other layers' compresses.
        max_pending: a pending handle keeps its raw activation alive until it is settled, so
        at most this many stay unsettled -- wrap_forward waits for the oldest beyond it (the
        GPU still has the newer ones queued). Without the bound the host runs the whole
        forward pass ahead of the GPU and every raw activation lives to the backward pass.
        two_lanes (with side_stream): long planes get the second lane; off, one side stream
        and one context (the second lane's context holds a second workspace).
        prefetch: after each unwrap, the newest still-held handle is decoded ahead on a
        stream of its own (the backward pass usually unwraps in reverse wrap order)."""
        cfg.validate()
        if num_layers < 0:
            raise _codec.ParamError("controller needs a non-negative layer count")
        self.cfg = cfg
        self.reducer = reducer
        self.ctx = ctx
        self.windows = [_Window() for _ in range(num_layers)]
        self.ledger = CompressionLedger()
        self.iteration = 0
        self._cur = 0
        self._peak = 0
        self._tin = 0
        self._tstored = 0
        self.async_compress = async_compress
        self.side_stream = side_stream
        self.max_pending = max(0, int(max_pending))
        self._lanes = [None, None]   # (stream, context) per compress lane (side_stream)
        self.prefetch = prefetch
        self.two_lanes = two_lanes
        self._pf = None              # decode-ahead stream (prefetch)
        self._live: List[ActivationHandle] = []  # wrapped, not yet unwrapped (prefetch)
        self._events = []            # ("w" | "u", handle, bytes) not yet accounted
        self._pending: List[ActivationHandle] = []
        self.refits = 0
        self.refit_reasons: List[str] = []

    # byte accounting of the stashed activations (settles pending compresses first)
    def _settled(name):
        def get(self):
            if self._pending:
                self.settle()
            return getattr(self, name)

        def put(self, v):
            setattr(self, name, v)
        return property(get, put)
    current_bytes = _settled("_cur")
    peak_bytes = _settled("_peak")
    total_in = _settled("_tin")
    total_stored = _settled("_tstored")
    del _settled

    # ---- asynchronous compress: settling, and the accounting in program order -----------
    def _settle_handle(self, h: ActivationHandle, wait: bool) -> bool:
        """Settles one pending handle; False if its compress has not finished (wait=False)."""
        try:
            c = h.pending.settle(wait)
        except _codec.Error as e:
            print(f"warning: compression failed for layer {h.layer_id} ({e}); passing "
                  "through", file=sys.stderr)
            c = None
            h.raw = h.pending._t
        else:
            if c is None:
                return False
        self.refits += h.pending.refits
        if h.pending.refits:
            self.refit_reasons.append(h.pending.refit_reason)
        h.pending = None
        if c is not None:
            self._engage_blob(h, c)
        else:
            h.held_bytes = h.stored_bytes = h.in_bytes
        return True

    def settle(self, wait: bool = True, keep: int = 0) -> None:
        """Settles pending handles in wrap order; wait=False stops at the first one whose
        compress has not finished; keep: leave (up to) that many of the newest pending."""
        while len(self._pending) > keep:
            h = self._pending[0]
            if h.pending is not None and not self._settle_handle(h, wait):
                break
            self._pending.pop(0)
        self._flush()

    def _flush(self) -> None:
        """Applies the byte accounting of wraps and unwraps in program order, up to the
        first wrap whose size is not known yet (so current/peak bytes and the window sums
        are those of the synchronous path)."""
        while self._events:
            kind, h, nbytes = self._events[0]
            if kind == "w" and h.pending is not None:
                return
            self._events.pop(0)
            if kind == "w":
                self._account(h, h.in_bytes)
            else:
                self._cur -= nbytes

    def _engage_blob(self, h: ActivationHandle, c) -> None:
        h.blob, h.held_bytes = c, c.compressed_bytes
        h.stored_bytes = h.held_bytes
        h.achieved_ratio = _codec.compression_ratio(c)
        if self.cfg.zero_restoration == RELU_RECOMPUTE and h.post_relu:
            h.apply_relu = True
        else:
            h.zero_filter = True

    def _account(self, h: ActivationHandle, in_bytes: int) -> None:
        # h.stored_bytes: what the wrap held (h.held_bytes may already be 0: a handle can be
        # unwrapped before an older wrap settles and lets this one's accounting run)
        w = self.windows[h.layer_id]
        if w.open:
            w.bytes_in += in_bytes
            w.bytes_stored += h.stored_bytes
        self._tin += in_bytes
        self._tstored += h.stored_bytes
        self._cur += h.stored_bytes
        self._peak = max(self._peak, self._cur)

    # ---- phases 1-3 ----------------------------------------------------------------
    def begin_iteration(self, iteration: int) -> None:
        if iteration < 0:
            raise _codec.ParamError("iteration must be >= 0")
        self.settle()
        self._live.clear()
        self.iteration = iteration

    def collecting(self) -> bool:
        return self.iteration % self.cfg.collect_interval == 0

    def collect_stats(self, layer: int, activation, loss, momentum, batch: int) -> LayerStats:
        """ref src/controller.cpp:124-152 (global over ranks when a reducer is set)."""
        return self.collect_stats_from_sums(layer, local_stat_sums(activation, loss, momentum,
                                                                   batch))

    def collect_stats_from_sums(self, layer: int, sums: List[float]) -> LayerStats:
        if not 0 <= layer < len(self.windows):
            raise _codec.ParamError("collect_stats: unknown layer id")
        if not self.collecting():
            raise _codec.ParamError("collect_stats invoked outside a collection iteration")
        self.settle()
        if self.reducer is not None:
            sums = self.reducer(list(sums))
        st = LayerStats(layer_id=layer,
                        l_bar=sums[0] / sums[1] if sums[1] > 0 else 0.0,
                        r=sums[2] / sums[3] if sums[3] > 0 else 0.0,
                        m_avg=sums[4] / sums[5] if sums[5] > 0 else 0.0,
                        batch=int(sums[6]), collected_at=self.iteration)
        st.degenerate = st.l_bar == 0.0 or st.m_avg == 0.0 or st.r == 0.0
        self._close_window(layer)
        w = _Window(stats=st, open=True)
        if not st.degenerate:
            w.sigma = self.target_sigma(st, self.cfg)
            w.eb = self.compute_error_bound(st, w.sigma, self.cfg)
            w.fallback = False
        self.windows[layer] = w
        return st

    @staticmethod
    def target_sigma(st: LayerStats, cfg: ControllerConfig) -> float:
        if not st.m_avg > 0.0:
            raise _codec.ParamError("target_sigma: degenerate M_avg")
        return cfg.sigma_fraction * st.m_avg

    @staticmethod
    def compute_error_bound(st: LayerStats, sigma: float, cfg: ControllerConfig) -> float:
        if not sigma > 0.0:
            raise _codec.ParamError("compute_error_bound: sigma must be positive")
        if not (st.l_bar > 0.0 and st.r > 0.0):
            raise _codec.ParamError("compute_error_bound: degenerate stats")
        eb = sigma / (cfg.coefficient_a * st.l_bar * math.sqrt(float(st.batch) * st.r))
        return min(max(eb, cfg.eb_min), cfg.eb_max)

    def layer_active(self, layer: int) -> bool:
        if not 0 <= layer < len(self.windows):
            return False
        w = self.windows[layer]
        return w.open and not w.fallback and self.iteration > w.stats.collected_at

    def layer_eb(self, layer: int) -> float:
        return self.windows[layer].eb if self.layer_active(layer) else 0.0

    # ---- phase 4 -----------------------------------------------------------------------
    def wrap_forward(self, layer: int, activation, is_post_relu: bool) -> ActivationHandle:
        """ref src/controller.cpp:194-232: compress on the GPU or pass through; codec
        failures degrade to pass-through with a warning."""
        if not 0 <= layer < len(self.windows):
            raise _codec.ParamError("wrap_forward: unknown layer id")
        in_bytes = activation.numel() * 4
        h = ActivationHandle(layer_id=layer)
        if self.prefetch:
            self._live.append(h)
        if self._pending:
            self.settle(wait=False)
        h.in_bytes = in_bytes
        if self.async_compress and self.layer_active(layer):
            w = self.windows[layer]
            side = main = None
            ctx = self.ctx
            if self.side_stream:
                import torch
                main = torch.cuda.current_stream(activation.device)
                lane = self._lane(activation) if self.two_lanes else 0
                if self._lanes[lane] is None:
                    self._lanes[lane] = (torch.cuda.Stream(device=activation.device),
                                         self.ctx if lane == 0 else
                                         _codec.Context(activation.device.index or 0))
                side, ctx = self._lanes[lane]
                if lane == 0 and ctx is None:
                    ctx = self.ctx
                h.side = side
                side.wait_stream(main)  # the activation has been produced
            try:
                a = _codec.compress_async(activation, _codec.CodecParams(
                    w.eb, self.cfg.quant_radius, self.cfg.predictor), ctx=ctx,
                    size_tag=layer + 1, stream=side)
                if side is not None and not a.pending:
                    # a synchronous compress (the first of its tag) may still be encoding on
                    # the side stream, reading the activation: the forward waits for it
                    main.wait_stream(side)
            except _codec.Error as e:
                print(f"warning: compression failed for layer {layer} ({e}); passing through",
                      file=sys.stderr)
                h.raw = activation
            else:
                h.pending, h.post_relu = a, is_post_relu
                self._pending.append(h)
                self._events.append(("w", h, 0))
                if not a.pending and len(self._pending) == 1:
                    self.settle()
                elif len(self._pending) > self.max_pending:
                    self.settle(wait=True, keep=self.max_pending)
                return h
            h.held_bytes = h.stored_bytes = in_bytes
            self._events.append(("w", h, 0))
            self._flush()
            return h
        if not self.layer_active(layer):
            h.raw, h.held_bytes = activation, in_bytes
        else:
            w = self.windows[layer]
            try:
                c = _codec.compress(activation, _codec.CodecParams(w.eb, self.cfg.quant_radius,
                                                                   self.cfg.predictor),
                                    ctx=self.ctx)
                h.blob, h.held_bytes = c, c.compressed_bytes
                h.achieved_ratio = _codec.compression_ratio(c)
                if self.cfg.zero_restoration == RELU_RECOMPUTE and is_post_relu:
                    h.apply_relu = True
                else:
                    h.zero_filter = True
            except _codec.Error as e:
                print(f"warning: compression failed for layer {layer} ({e}); passing through",
                      file=sys.stderr)
                h.raw, h.held_bytes = activation, in_bytes
        h.stored_bytes = h.held_bytes
        self._events.append(("w", h, 0))
        self._flush()
        return h

    def unwrap_backward(self, h: ActivationHandle):
        """ref src/controller.cpp:234-249"""
        if h.pending is not None:
            # only this handle: older ones may still be compressing on another lane
            self._settle_handle(h, True)
        if h.raw is not None:
            t, h.raw = h.raw, None
        elif h.blob is not None:
            if h.prefetched is not None:
                # decoded ahead on the prefetch stream (see _prefetch_next)
                import torch
                t, ev = h.prefetched
                h.prefetched = None
                main = torch.cuda.current_stream(t.device)
                main.wait_event(ev)
                t.record_stream(main)
            else:
                t = _codec.decompress(h.blob, zero_filter=h.zero_filter, ctx=self.ctx)
                if h.apply_relu:
                    _codec.relu_(t, ctx=self.ctx)  # nn::recompute_relu (layers.hpp:152-157)
            if h.side is not None:
                # the blob's arena was allocated on its lane's stream and is freed there
                # (stream-ordered): after this stream's decode has read it
                import torch
                h.side.wait_stream(torch.cuda.current_stream(t.device))
            h.blob = None
        else:
            raise _codec.ParamError("unwrap_backward: handle already consumed")
        self._events.append(("u", h, h.held_bytes))
        h.held_bytes = 0
        self._flush()
        if self.prefetch:
            self._forget(h)
            self._prefetch_next()
        return t

    def contexts(self) -> List[_codec.Context]:
        """Every codec context this controller compresses on (memory accounting: each holds
        its own workspace)."""
        out = [self.ctx or _codec.default_context()]
        for lane in self._lanes:
            if lane is not None and lane[1] is not None and all(lane[1] is not c for c in out):
                out.append(lane[1])
        return out

    def _forget(self, h: ActivationHandle) -> None:
        for i in range(len(self._live) - 1, -1, -1):
            if self._live[i] is h:
                del self._live[i]
                return

    def _prefetch_next(self) -> None:
        """Decodes the handle the backward pass will most likely unwrap next (the newest
        wrapped one still held) on a stream of its own, overlapping the current layer's
        backward kernels; unwrap_backward then only waits for that decode."""
        if not self._live:
            return
        nxt = self._live[-1]
        if nxt.prefetched is not None or nxt.raw is not None:
            return
        if nxt.pending is not None and not self._settle_handle(nxt, False):
            return  # still compressing: decoded on demand
        if nxt.blob is None:
            return
        import torch
        dev = torch.device("cuda", nxt.blob._ctx.device)
        if self._pf is None:
            self._pf = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(self._pf):
            t = _codec.decompress(nxt.blob, zero_filter=nxt.zero_filter, ctx=self.ctx,
                                  stream=self._pf)
            if nxt.apply_relu:
                _codec.relu_(t, stream=self._pf, ctx=self.ctx)
        ev = torch.cuda.Event()
        ev.record(self._pf)
        nxt.prefetched = (t, ev)

    @staticmethod
    def _lane(activation) -> int:
        """Compress lane of an activation: long planes (an input image, >= 128x128) get
        their own context and stream, so their latency-bound quantiser does not hold back
        the other layers' compresses (the backward pass starts with the last layer's)."""
        sh = activation.shape
        return 1 if len(sh) >= 2 and int(sh[-1]) * int(sh[-2]) >= 16384 else 0

    def finalize(self) -> None:
        self.settle()
        for i in range(len(self.windows)):
            self._close_window(i)

    def _close_window(self, layer: int) -> None:
        """ref src/controller.cpp:98-122"""
        w = self.windows[layer]
        if not w.open:
            return
        self.ledger.append(LedgerRecord(
            iteration=w.stats.collected_at, layer_id=layer, eb=0.0 if w.fallback else w.eb,
            predicted_sigma=0.0 if w.fallback else w.sigma, l_bar=w.stats.l_bar, r=w.stats.r,
            m_avg=w.stats.m_avg,
            ratio=1.0 if w.bytes_stored == 0 else w.bytes_in / w.bytes_stored,
            fallback=w.fallback))
        w.open = False


def suggest_batch(batch: int, peak_stash_bytes: int, budget_bytes: int, granularity: int = 8,
                  max_batch: int = 1 << 20) -> int:
    """Batch-size scheme (BASELINE config 5): the largest batch whose
    stashed activation bytes fit the budget, from the stash measured at `batch`."""
    if batch <= 0 or peak_stash_bytes <= 0:
        return batch
    b = int(budget_bytes / (peak_stash_bytes / batch))
    b = (b // granularity) * granularity
    return max(granularity, min(b, max_batch))


class _Stash:
    """One controller handle shared by every saved-tensor slot that aliases the same storage
    (a ReLU's saved output and the next conv's saved input are one tensor: compressing it
    once and dropping every raw reference is what actually frees the activation)."""

    __slots__ = ("ctl", "handle", "cache", "__weakref__")

    def __init__(self, ctl: "Controller", handle: ActivationHandle):
        self.ctl, self.handle, self.cache = ctl, handle, None

    def get(self):
        # decompressed once (Controller.unwrap_backward consumes the handle); the result is
        # kept while any slot referencing it lives, so a second unpack of the same saved
        # tensor (retain_graph, double backward, grad_fn._saved_*) sees the same values
        if self.cache is None:
            self.cache = self.ctl.unwrap_backward(self.handle)
        return self.cache


class _Saved:
    """What pack() returns: the raw tensor, or (after the storage became a conv input) the
    shared stash."""

    __slots__ = ("raw", "stash", "__weakref__")

    def __init__(self, raw=None, stash=None):
        self.raw, self.stash = raw, stash


class SavedActivationHooks:
    """torch.autograd.graph.saved_tensors_hooks that compress the INPUT of every
    convolution of `model` between its forward and backward pass, and nothing else (ref
    SPEC.md:420 "only convolutional-layer activations are compressed";
    Controller::wrap_forward / unwrap_backward, src/controller.cpp:194-249).

    * Layer ids are the convolutions' order in ``model.modules()`` (stable across
      iterations, so every layer's statistics window keeps its id).
    * A forward pre-hook on each conv marks its input; the first time autograd saves that
      storage for the conv, it is compressed through the controller. Earlier or later
      saves of the same storage (ReLU's output, a pooling input) share the compressed stash
      instead of keeping a raw reference.
    * Parameters and other leaf tensors that require grad (weights) are never compressed.
    * is_post_relu for the relu-recompute zero restoration is read from the tensor's
      autograd node (ReluBackward / ThresholdBackward), with no device synchronisation.
    Call :meth:`new_iteration` at the start of every step."""

    def __init__(self, controller: Controller, model, min_numel: int = 0):
        import torch.nn as nn
        self.ctl = controller
        self.min_numel = min_numel
        self.convs = [m for m in model.modules()
                      if isinstance(m, (nn.Conv1d, nn.Conv2d, nn.Conv3d))]
        if len(self.convs) > len(controller.windows):
            raise _codec.ParamError(f"controller has {len(controller.windows)} layers, model "
                                    f"has {len(self.convs)} convolutions")
        self._hooks = [m.register_forward_pre_hook(self._mark(i))
                       for i, m in enumerate(self.convs)]
        # Keys are (data_ptr, shape); every entry also holds a weak reference to the storage
        # it was taken from, so an address the caching allocator hands out again after the
        # original activation was freed (e.g. a later ReLU output of the same shape) never
        # matches a stale entry.
        # Only weak references: autograd's saved-variable slots own the _Saved / _Stash
        # objects, so a stash (and its decompressed cache) dies with the last graph node that
        # saved it, and raw saves are not kept alive past the backward pass.
        self._marked = {}   # storage key -> (storage weakref, conv layer id)
        self._stash = {}    # storage key -> (storage weakref, weakref to _Stash)
        self._raw = {}      # storage key -> [weakref to _Saved] raw saves that may alias a conv input
        self.compressed = 0

    @staticmethod
    def _key(t):
        return (t.data_ptr(), tuple(t.shape))

    @staticmethod
    def _live(entry, t):
        """entry = (storage weakref, value): the value if the entry was made for t's storage
        and that storage is still alive, else None."""
        if entry is None:
            return None
        ref, value = entry
        st = ref()
        return value if st is not None and st is t.untyped_storage() else None

    def _mark(self, layer: int):
        import weakref

        def hook(_module, args):
            if args and hasattr(args[0], "data_ptr") and args[0].is_cuda:
                t = args[0]
                key = self._key(t)
                if self._live(self._marked.get(key), t) is None:
                    self._marked[key] = (weakref.ref(t.untyped_storage()), layer)
        return hook

    def remove(self) -> None:
        for h in self._hooks:
            h.remove()
        self._hooks = []

    def new_iteration(self, iteration: int) -> None:
        self.ctl.begin_iteration(iteration)
        self._marked.clear()
        self._stash.clear()
        self._raw.clear()

    @staticmethod
    def _post_relu(t) -> bool:
        fn = t.grad_fn
        name = type(fn).__name__ if fn is not None else ""
        return "Relu" in name or "Threshold" in name

    def pack(self, t):
        import torch
        if (isinstance(t, torch.nn.Parameter) or (t.is_leaf and t.requires_grad)
                or not t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous()
                or t.numel() < max(1, self.min_numel)):
            return _Saved(raw=t)
        import weakref
        key = self._key(t)
        wst = self._live(self._stash.get(key), t)
        st = wst() if wst is not None else None
        if st is not None:
            return _Saved(stash=st)
        layer = self._live(self._marked.pop(key, None), t)
        if layer is None:
            s = _Saved(raw=t)
            self._raw.setdefault(key, []).append(weakref.ref(s))
            return s
        relu = self.ctl.cfg.zero_restoration == RELU_RECOMPUTE and self._post_relu(t)
        st = _Stash(self.ctl, self.ctl.wrap_forward(layer, t.detach(), relu))
        self._stash[key] = (weakref.ref(t.untyped_storage()), weakref.ref(st))
        if st.handle.blob is not None or st.handle.pending is not None:
            self.compressed += 1
        for ws in self._raw.pop(key, []):  # earlier saves of the same storage share it
            s = ws()
            if s is not None:
                s.raw, s.stash = None, st
        return _Saved(stash=st)

    def unpack(self, s):
        return s.raw if s.stash is None else s.stash.get()

    def __enter__(self):
        import torch
        self._cm = torch.autograd.graph.saved_tensors_hooks(self.pack, self.unpack)
        self._cm.__enter__()
        return self

    def __exit__(self, *exc):
        return self._cm.__exit__(*exc)
