"""Diagnose the saved-tensor hooks train step: per-layer decompression error and gradients."""
import sys, torch, torch.nn as nn
sys.path.insert(0, ".")
from paper_2011_09017_b200.controller import SavedActivationHooks, Controller, ControllerConfig
import paper_2011_09017_b200 as acz

def net_():
    return nn.Sequential(nn.Conv2d(3, 16, 3, padding=1), nn.ReLU(inplace=True),
                         nn.Conv2d(16, 32, 3, padding=1), nn.ReLU(inplace=True),
                         nn.MaxPool2d(2), nn.Conv2d(32, 32, 3, padding=1), nn.ReLU(),
                         nn.AdaptiveAvgPool2d(1), nn.Flatten(), nn.Linear(32, 10)).cuda()

for zr in ["codec-filter", "relu-recompute"]:
    torch.manual_seed(0)
    net = net_()
    x = torch.randn(8, 3, 32, 32, device="cuda")
    y = torch.randint(0, 10, (8,), device="cuda")
    g0 = torch.autograd.grad(nn.functional.cross_entropy(net(x), y), list(net.parameters()))
    # direct codec round trip of x
    c = acz.compress(x, acz.CodecParams(1e-5))
    d = acz.decompress(c, zero_filter=True)
    torch.cuda.synchronize()
    print(zr, "direct x err", float((d - x).abs().max()))
    ctl = Controller(ControllerConfig(collect_interval=100, eb_min=1e-5, eb_max=1e-5,
                                      zero_restoration=zr), 3)
    for layer in range(3):
        ctl.collect_stats_from_sums(layer, [1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 8.0])
    hooks = SavedActivationHooks(ctl, net)
    hooks.new_iteration(1)
    seen = []
    orig_pack = hooks.pack
    def pack(t):
        s = orig_pack(t)
        seen.append((tuple(t.shape), t.clone(), s))
        return s
    import torch.autograd.graph as G
    with G.saved_tensors_hooks(pack, hooks.unpack):
        loss1 = nn.functional.cross_entropy(net(x), y)
    for shp, tc, s in seen:
        if s.stash is not None:
            v = s.stash.get()
            torch.cuda.synchronize()
            print("  saved", shp, "stash err", float((v - tc).abs().max()))
        else:
            print("  saved", shp, "raw")
    g1 = torch.autograd.grad(loss1, list(net.parameters()))
    for i, (a, b) in enumerate(zip(g0, g1)):
        print("  param", i, tuple(a.shape), "maxdiff", float((a - b).abs().max()), "max", float(a.abs().max()))
    hooks.remove()
