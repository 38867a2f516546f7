"""BASELINE config 5 at a 1-GPU shard: ResNet-18 (torchvision, random init), batch 1024 over
8 B200s -> 128 per GPU, synthetic ImageNet-shaped data, SGD with momentum, the adaptive
error-bound scheme active (paper_2011_09017_b200.training.AdaptiveCompression: the
controller's four phases with W-iteration statistics windows, conv inputs compressed on
the GPU between forward and backward), then the batch-size half of the scheme
(BatchSizeScheme): the memory the compression frees is turned into a larger batch under the
budget the uncompressed run needs at the base batch.

Memory is counted honestly: torch's peak allocation PLUS the codec's own device memory
(blob arenas incl. decode sidecars, and the context workspace) at their peaks.

usage: python tools/config5_batch_scheme.py [--base 128] [--steps 12] [--W 4] [--out FILE]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch
import torch.nn as nn
import torchvision

import paper_2011_09017_b200 as acz
from paper_2011_09017_b200.controller import ControllerConfig
from paper_2011_09017_b200.training import AdaptiveCompression, BatchSizeScheme


def run(batch, steps, compress, W, seed=0):
    torch.manual_seed(seed)
    dev = torch.device("cuda", 0)
    model = torchvision.models.resnet18(num_classes=1000).to(dev)
    opt = torch.optim.SGD(model.parameters(), lr=0.01, momentum=0.9, weight_decay=1e-4)
    crit = nn.CrossEntropyLoss()
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    x = torch.randn(batch, 3, 224, 224, device=dev, generator=g)
    y = torch.randint(0, 1000, (batch,), device=dev, generator=g)
    ctx = acz.default_context(0)
    ac = AdaptiveCompression(model, opt, ControllerConfig(collect_interval=W), ctx=ctx) \
        if compress else None
    torch.cuda.synchronize()
    # one warm step (momentum buffers exist afterwards): its memory is the static part
    static = None
    times, peaks, codec_peaks, losses = [], [], [], []
    totals = None
    for it in range(steps):
        torch.cuda.synchronize()
        if it == 1:
            static = torch.cuda.memory_allocated()
        if it == W + 1 and ac:
            totals = (ac.ctl.total_in, ac.ctl.total_stored)
        torch.cuda.reset_peak_memory_stats()
        ctx.memory_info(reset_peak=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        opt.zero_grad(set_to_none=True)
        if ac:
            ac.begin(it)
            with ac.hooks:
                loss = crit(model(x), y)
        else:
            loss = crit(model(x), y)
        loss.backward()
        if ac:
            ac.end()
        opt.step()
        e1.record()
        torch.cuda.synchronize()
        mi = ctx.memory_info()
        if ac:  # the workspaces of every context the controller compresses on (lanes)
            mi["workspace_bytes"] = sum(c.memory_info()["workspace_bytes"]
                                        for c in ac.ctl.contexts())
        times.append(e0.elapsed_time(e1))
        peaks.append(torch.cuda.max_memory_allocated())
        codec_peaks.append(mi["blob_peak_bytes"] + mi["workspace_bytes"])
        losses.append(float(loss))
    # steady state: iterations after the first non-degenerate window opened (the windows
    # collected at iteration 0 see all-zero momentum and pass through, ref
    # include/acz/controller.hpp:92-94; the next collection is at W)
    # (and after the first of them, W + 1, whose compresses are the codec's warm-up: the
    # first compress of every layer is synchronous and sizes the asynchronous ones)
    ss = range(W + 2, steps)
    res = {
        "batch": batch, "compress": compress, "steps": steps, "W": W,
        "static_bytes": static,
        "peak_torch_bytes": max(peaks[i] for i in ss),
        "peak_codec_bytes": max(codec_peaks[i] for i in ss),
        "ms_per_step": sum(times[i] for i in ss) / len(ss),
        "loss_first_last": [losses[0], losses[-1]],
    }
    res["peak_total_bytes"] = res["peak_torch_bytes"] + res["peak_codec_bytes"]
    res["images_per_s"] = batch / (res["ms_per_step"] * 1e-3)
    if ac:
        c = ac.ctl
        res["compressed_layers_last_step"] = ac.hooks.compressed
        res["ratio_steady_state"] = (c.total_in - totals[0]) / max(1, c.total_stored - totals[1])
        res["stash_peak_acz1_bytes"] = c.peak_bytes
        ebs = [w.eb for w in c.windows if w.open and not w.fallback]
        res["eb_min_max"] = [min(ebs), max(ebs)] if ebs else None
        c.finalize()
        res["ledger_rows"] = len(c.ledger.records)
        ac.remove()
    del model, opt, x, y
    if ac:
        for c in ac.ctl.contexts():
            c.trim()
    ctx.trim()
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--base", type=int, default=128)
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--W", type=int, default=4)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    base = run(a.base, a.steps, False, a.W)
    comp = run(a.base, a.steps, True, a.W)
    scheme = BatchSizeScheme(granularity=8)
    budget = base["peak_total_bytes"]
    # the scheme's loop: suggest from the measured peak, run the suggested batch, re-fit the
    # linear memory model through the two measured points, until the batch fits the budget
    b1 = scheme.suggest(a.base, comp["static_bytes"], comp["peak_total_bytes"], budget)
    tried = []
    grown = None
    for _ in range(4):
        grown = run(b1, a.steps, True, a.W)
        tried.append({"batch": b1, "peak_total_bytes": grown["peak_total_bytes"],
                      "fits": grown["peak_total_bytes"] <= budget})
        if grown["peak_total_bytes"] <= budget:
            break
        # two-point fit: per-sample slope and intercept from (base, comp) and (b1, grown)
        slope = (grown["peak_total_bytes"] - comp["peak_total_bytes"]) / max(1, b1 - a.base)
        inter = comp["peak_total_bytes"] - slope * a.base
        b1 = scheme.suggest(1, int(inter), int(inter + slope), budget)
    grown_raw = run(b1, a.steps, False, a.W)
    out = {
        "workload": "BASELINE configs[4] at a 1-GPU shard: ResNet-18, batch 1024/8 = "
                    f"{a.base} per GPU, synthetic 224x224 images, SGD momentum 0.9, adaptive eb "
                    f"(W={a.W}) + batch-size scheme",
        "uncompressed_base": base, "compressed_base": comp,
        "budget_bytes": budget, "scheme": scheme.history, "batch_search": tried,
        "compressed_grown": grown, "uncompressed_grown": grown_raw,
        "summary": {
            "activation_memory_saved_at_base":
                1 - (comp["peak_total_bytes"] - comp["static_bytes"]) /
                max(1, base["peak_total_bytes"] - base["static_bytes"]),
            "grown_batch": b1,
            "grown_fits_budget": grown["peak_total_bytes"] <= budget,
            "batch_gain": b1 / a.base,
            "images_per_s_gain_vs_uncompressed_base":
                grown["images_per_s"] / base["images_per_s"],
        },
    }
    s = json.dumps(out, indent=1)
    print(s)
    if a.out:
        with open(a.out, "w") as f:
            f.write(s)


if __name__ == "__main__":
    main()
