import sys, torch, torch.nn as nn, torchvision, gc
sys.path.insert(0, ".")
import paper_2011_09017_b200 as acz
from paper_2011_09017_b200.controller import ControllerConfig
from paper_2011_09017_b200.training import AdaptiveCompression
dev = torch.device("cuda", 0)
torch.manual_seed(0)
model = torchvision.models.resnet18(num_classes=1000).to(dev)
opt = torch.optim.SGD(model.parameters(), lr=0.01, momentum=0.9)
x = torch.randn(128, 3, 224, 224, device=dev); y = torch.randint(0, 1000, (128,), device=dev)
crit = nn.CrossEntropyLoss()
ac = AdaptiveCompression(model, opt, ControllerConfig(collect_interval=4), ctx=acz.default_context(0))
for it in range(3):
    torch.cuda.synchronize(); m0 = torch.cuda.memory_allocated()
    opt.zero_grad(set_to_none=True)
    ac.begin(it)
    c0 = ac.hooks.compressed
    with ac.hooks:
        loss = crit(model(x), y)
    torch.cuda.synchronize(); m1 = torch.cuda.memory_allocated()
    raw_alive = sum(1 for v in ac.hooks._raw.values() for w in v if w() is not None and w().raw is not None)
    raw_bytes = sum(w().raw.numel()*4 for v in ac.hooks._raw.values() for w in v if w() is not None and w().raw is not None)
    st = [w() for _, w in ac.hooks._stash.values()]
    print(f"it {it}: fwd delta {(m1-m0)/1e9:.3f} GB, compressed {ac.hooks.compressed-c0}, stashes {len(st)} alive {sum(s is not None for s in st)}, "
          f"blob? {sum(1 for s in st if s is not None and s.handle.blob is not None)}, raw entries alive {raw_alive} ({raw_bytes/1e9:.3f} GB), marked left {len(ac.hooks._marked)}, "
          f"codec {acz.default_context(0).memory_info()}")
    loss.backward(); ac.end(); opt.step()
for k, (ref, w) in list(ac.hooks._stash.items())[:3]:
    print(k, w() is not None)
