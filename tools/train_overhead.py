"""Where the compressed ResNet-18 training step spends its time (config 5 shard, B128):
host wall time inside Controller.wrap_forward / unwrap_backward / the statistics taps,
the step's device time, and the same step without compression."""
import os, sys, time, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.nn as nn, torchvision
import paper_2011_09017_b200 as acz
from paper_2011_09017_b200 import controller as C, codec as K
from paper_2011_09017_b200.controller import ControllerConfig
from paper_2011_09017_b200.training import AdaptiveCompression

acc = collections.defaultdict(float)
cnt = collections.defaultdict(int)
def wrap(obj, name, tag):
    f = getattr(obj, name)
    def g(*a, **k):
        t = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            acc[tag] += time.perf_counter() - t
            cnt[tag] += 1
    setattr(obj, name, g)
wrap(C.Controller, "wrap_forward", "wrap_forward")
wrap(C.Controller, "unwrap_backward", "unwrap_backward")
wrap(K, "compress", "codec.compress")
wrap(K, "decompress", "codec.decompress")
wrap(K, "zero_bitmap", "stats.zero_bitmap")
wrap(K, "mean_abs", "stats.mean_abs")

B = int(os.environ.get("B", 128))
dev = torch.device("cuda", 0)
for compress, asy, side in ((False, False, False), (True, False, False), (True, True, True)):
    torch.manual_seed(0)
    model = torchvision.models.resnet18(num_classes=1000).to(dev)
    opt = torch.optim.SGD(model.parameters(), lr=0.01, momentum=0.9)
    crit = nn.CrossEntropyLoss()
    x = torch.randn(B, 3, 224, 224, device=dev); y = torch.randint(0, 1000, (B,), device=dev)
    ac = AdaptiveCompression(model, opt, ControllerConfig(collect_interval=4),
                             async_compress=asy, side_stream=side,
                             max_pending=int(os.environ.get("MAXP", 4)),
                             prefetch=os.environ.get("PREFETCH", "0") == "1",
                             two_lanes=os.environ.get("LANES", "2") == "2") if compress else None
    res = []
    for it in range(12):
        if it == 6:
            acc.clear(); cnt.clear()
        torch.cuda.synchronize(); torch.cuda.reset_peak_memory_stats(); t0 = time.perf_counter()
        opt.zero_grad(set_to_none=True)
        if ac:
            ac.begin(it)
            with ac.hooks:
                loss = crit(model(x), y)
            t1 = time.perf_counter()
            loss.backward(); ac.end()
        else:
            loss = crit(model(x), y); t1 = time.perf_counter(); loss.backward()
        opt.step(); torch.cuda.synchronize(); t2 = time.perf_counter()
        res.append((round((t1 - t0) * 1e3, 2), round((t2 - t0) * 1e3, 2),
                    round(torch.cuda.max_memory_allocated() / 2**20)))
    print(f"compress={compress} async={asy} side_stream={side}: (host ms to end of forward, step ms, torch peak MiB) per iteration:", res)
    if ac:
        print("  refits", ac.ctl.refits, "compressed", ac.hooks.compressed)
        for r in ac.ctl.refit_reasons[:20]:
            print("   ", r)
    if compress:
        n = 6
        print("  per step (iterations 6-11, host wall ms / calls):",
              {k: (round(v * 1e3 / n, 2), cnt[k] // n) for k, v in acc.items()})
