import sys, torch, torch.nn as nn
sys.path.insert(0, ".")
from paper_2011_09017_b200.controller import SavedActivationHooks, Controller, ControllerConfig
torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark = True, False
torch.manual_seed(1)
net = nn.Sequential(nn.Conv2d(3, 64, 3, padding=1), nn.ReLU(inplace=True),
                    nn.Conv2d(64, 64, 3, padding=1), nn.ReLU(inplace=True),
                    nn.Conv2d(64, 64, 3, padding=1), nn.AdaptiveAvgPool2d(1),
                    nn.Flatten()).cuda()
x = torch.randn(32, 3, 64, 64, device="cuda")
out = net(x).sum()
a = torch.autograd.grad(out, list(net.parameters()), retain_graph=True)
b = torch.autograd.grad(out, list(net.parameters()))
print("no hooks:", [float((p - q).abs().max()) for p, q in zip(a, b)])
for sync in (False, True):
    ctl = Controller(ControllerConfig(collect_interval=100, eb_min=1e-2, eb_max=1e-2), 3)
    for layer in range(3):
        ctl.collect_stats_from_sums(layer, [1.0] * 6 + [8.0])
    hooks = SavedActivationHooks(ctl, net)
    hooks.new_iteration(1)
    if sync:
        up = hooks.unpack
        def unpack(s):
            v = up(s); torch.cuda.synchronize(); return v
        hooks.unpack = unpack
    with hooks:
        out = net(x).sum()
    hooks.remove()
    a = torch.autograd.grad(out, list(net.parameters()), retain_graph=True)
    b = torch.autograd.grad(out, list(net.parameters()))
    print("hooks sync", sync, [float((p - q).abs().max()) for p, q in zip(a, b)])
