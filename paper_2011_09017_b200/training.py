"""PyTorch training-loop integration of the adaptive scheme (BASELINE configs 3 and 5;
SURVEY.md 8(f) row 4): the controller's four phases driven by a real optimiser step, and
the batch-size half of the scheme (the reference leaves it as a non-goal,
SPEC.md:431).

Phase 1 (every W iterations, ref src/controller.cpp:124-152) needs, per convolution:
  L_bar : mean |gradient| at the layer's output      <- tensor hook on the conv output
  R     : nonzero ratio of the layer's activation     <- forward pre-hook (GPU K1 count)
  M_avg : mean |momentum| of the layer's weights      <- the SGD momentum buffer
  N     : the batch
Phases 2-4 run in :class:`controller.Controller` / :class:`controller.SavedActivationHooks`
(conv inputs compressed between forward and backward through the GPU codec).

:class:`AdaptiveCompression` wires both into a model + optimiser; :class:`BatchSizeScheme`
turns the memory that compression frees into a larger batch under a fixed budget.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional

from . import codec as _codec
from .controller import Controller, ControllerConfig, SavedActivationHooks, local_stat_sums


class AdaptiveCompression:
    """Adaptive activation compression for one model / optimiser (one rank).

    Usage per step::

        ac.begin(iteration)
        with ac.hooks:
            loss = criterion(model(x), y)
        loss.backward()
        ac.end()            # phase 1 on collection iterations (before optimizer.step())
        optimizer.step()
    """

    def __init__(self, model, optimizer, cfg: ControllerConfig, reducer=None,
                 ctx: Optional[_codec.Context] = None, min_numel: int = 0,
                 async_compress: bool = True, side_stream: bool = True, max_pending: int = 4,
                 prefetch: bool = False, two_lanes: bool = True):
        import torch.nn as nn
        self.model, self.opt = model, optimizer
        self.convs = [m for m in model.modules()
                      if isinstance(m, (nn.Conv1d, nn.Conv2d, nn.Conv3d))]
        # async_compress: the conv inputs are compressed without a host wait per layer
        # (codec.compress_async; settled in wrap order, results identical)
        # (side_stream: on a stream of their own, overlapping the next layers' forward)
        self.ctl = Controller(cfg, len(self.convs), reducer=reducer, ctx=ctx,
                              async_compress=async_compress,
                              side_stream=async_compress and side_stream,
                              max_pending=max_pending,
                              # decode-ahead in the backward pass: ResNet-18 B128 25.9 ->
                              # 25.5 ms per step for +49 MiB of peak (off by default)
                              prefetch=async_compress and side_stream and prefetch,
                              # a second compress lane (stream + context) for long-plane
                              # inputs: ResNet-18 B128 27.9 -> 26.1 ms per step and 2379 ->
                              # 2282 MiB torch peak (the image's latency-bound quantiser no
                              # longer holds the other layers' raw inputs), for a second
                              # context workspace (counted in config 5)
                              two_lanes=two_lanes)
        self.hooks = SavedActivationHooks(self.ctl, model, min_numel=min_numel)
        self._act: Dict[int, List[float]] = {}   # layer -> [nonzeros, count, batch]
        self._grad: Dict[int, List[float]] = {}  # layer -> [sum |g|, count]
        self._handles = []
        for i, m in enumerate(self.convs):
            self._handles.append(m.register_forward_pre_hook(self._pre(i)))
            self._handles.append(m.register_forward_hook(self._post(i)))

    # ---- statistics taps (active on collection iterations only) -------------------------
    def _pre(self, layer: int):
        def hook(_m, args):
            if not self.ctl.collecting() or not args:
                return
            a = args[0].detach()
            if a.is_cuda and a.dtype.is_floating_point:
                a32 = a.float().contiguous()
                nz = _codec.zero_bitmap(a32)[1]
            else:
                nz = int((a != 0).sum().item())
            self._act[layer] = [float(nz), float(a.numel()), float(a.shape[0])]
        return hook

    def _post(self, layer: int):
        def hook(_m, _args, out):
            if not self.ctl.collecting() or not getattr(out, "requires_grad", False):
                return

            def grad_tap(g):
                g32 = g.detach().float().contiguous()
                s = (_codec.mean_abs(g32) * g32.numel()) if g32.is_cuda \
                    else float(g32.double().abs().sum().item())
                self._grad[layer] = [s, float(g32.numel())]
            out.register_hook(grad_tap)
        return hook

    # ---- step protocol -----------------------------------------------------------------
    def begin(self, iteration: int) -> None:
        self.hooks.new_iteration(iteration)
        self._act.clear()
        self._grad.clear()

    def end(self) -> None:
        """Phase 1 after the backward pass of a collection iteration: one stats window per
        conv (ref Controller::collect_stats, src/controller.cpp:124-152)."""
        if not self.ctl.collecting():
            return
        for i, m in enumerate(self.convs):
            if i not in self._act or i not in self._grad:
                continue
            st = self.opt.state.get(m.weight, {})
            mom = st.get("momentum_buffer")
            if mom is not None:
                ma = _codec.mean_abs(mom.detach().float().contiguous()) * mom.numel() \
                    if mom.is_cuda else float(mom.detach().double().abs().sum().item())
                mn = float(mom.numel())
            else:  # iteration 0: all-zero momentum -> degenerate window (pass-through)
                ma, mn = 0.0, float(m.weight.numel())
            nz, cnt, batch = self._act[i]
            ls, lc = self._grad[i]
            self.ctl.collect_stats_from_sums(i, [ls, lc, nz, cnt, ma, mn, batch])

    def remove(self) -> None:
        self.hooks.remove()
        for h in self._handles:
            h.remove()
        self._handles = []


@dataclass
class BatchSizeScheme:
    """Batch-size half of the adaptive scheme: with compression the
    per-sample activation memory drops, so a larger batch fits the memory budget the
    uncompressed run needs at the base batch.

    Memory model (measured, not assumed): peak(B) = static + B * per_sample, with
    `static` the model + optimiser state and per_sample the compressed run's peak growth
    per sample at the base batch. The suggested batch is the largest multiple of
    `granularity` with static + B * per_sample <= budget."""
    granularity: int = 8
    max_batch: int = 1 << 16
    history: List[dict] = field(default_factory=list)

    def suggest(self, base_batch: int, static_bytes: int, peak_bytes: int,
                budget_bytes: int) -> int:
        per_sample = max(1.0, (peak_bytes - static_bytes) / max(1, base_batch))
        b = int((budget_bytes - static_bytes) / per_sample)
        b = (b // self.granularity) * self.granularity
        b = max(self.granularity, min(b, self.max_batch))
        self.history.append(dict(base_batch=base_batch, static=static_bytes, peak=peak_bytes,
                                 budget=budget_bytes, per_sample=per_sample, suggested=b))
        return b
