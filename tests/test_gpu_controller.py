"""GPU tests of the controller's phase 4 (compress / decompress stashed activations) against
the reference Controller, and of the PyTorch saved-tensor hooks on a small CNN."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_wrap_unwrap_matches_reference(gpu_lib, reference):
    import torch
    from paper_2011_09017_b200.controller import Controller, ControllerConfig
    rng = np.random.default_rng(21)
    act = np.maximum(rng.standard_normal((6, 16, 28, 28)), 0).astype(np.float32)
    loss = (1e-3 * rng.standard_normal(act.shape)).astype(np.float32)
    mom = (1e-2 * rng.standard_normal((32, 16, 3, 3))).astype(np.float32)
    kw = dict(eb_min=1e-3, eb_max=1e-3)  # pin eb so both sides compress with the same bound
    ref = reference.controller_run(act, loss, mom, batch=6, W=4, wraps=1, **kw)
    c = Controller(ControllerConfig(collect_interval=4, **kw), 1)
    c.collect_stats(0, torch.from_numpy(act).cuda(), torch.from_numpy(loss).cuda(),
                    torch.from_numpy(mom).cuda(), 6)
    c.begin_iteration(1)
    h = c.wrap_forward(0, torch.from_numpy(act).cuda(), True)
    assert h.blob is not None and h.held_bytes == ref["held_bytes"]
    back = c.unwrap_backward(h)
    assert float((back.cpu() - torch.from_numpy(act)).abs().max()) <= 2e-3
    c.finalize()
    rows = [l.split(",") for l in c.ledger.to_csv().strip().split("\n")[1:]]
    rrows = [l.split(",") for l in ref["csv"].strip().split("\n")[1:]]
    assert len(rows) == len(rrows) == 1
    for a, b in zip(rows[0], rrows[0]):
        assert math.isclose(float(a), float(b), rel_tol=1e-12)


def test_saved_tensor_hooks_train_step(gpu_lib):
    import torch
    import torch.nn as nn
    from paper_2011_09017_b200.controller import (Controller, ControllerConfig,
                                                  SavedActivationHooks)
    torch.manual_seed(0)
    net = nn.Sequential(nn.Conv2d(3, 16, 3, padding=1), nn.ReLU(), nn.Conv2d(16, 32, 3, padding=1),
                        nn.ReLU(), nn.AdaptiveAvgPool2d(1), nn.Flatten(), nn.Linear(32, 10)).cuda()
    x = torch.randn(8, 3, 32, 32, device="cuda")
    y = torch.randint(0, 10, (8,), device="cuda")
    loss0 = nn.functional.cross_entropy(net(x), y)
    g0 = torch.autograd.grad(loss0, list(net.parameters()))
    ctl = Controller(ControllerConfig(collect_interval=100, eb_min=1e-4, eb_max=1e-4), 8)
    # pretend stats were collected at iteration 0 for every layer slot
    for layer in range(8):
        ctl.collect_stats_from_sums(layer, [1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 8.0])
    hooks = SavedActivationHooks(ctl, min_numel=1024)
    hooks.new_iteration(1)
    with hooks:
        loss1 = nn.functional.cross_entropy(net(x), y)
    assert ctl.current_bytes > 0 and ctl.total_stored < ctl.total_in
    g1 = torch.autograd.grad(loss1, list(net.parameters()))
    assert ctl.current_bytes == 0
    for a, b in zip(g0, g1):
        assert torch.allclose(a, b, rtol=0, atol=1e-2 * float(a.abs().max()) + 1e-6)
