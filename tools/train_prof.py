"""GPU kernel time of the compressed ResNet-18 B128 training step (torch.profiler/CUPTI:
every kernel, the codec's included), async compress on."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.nn as nn, torchvision
from torch.profiler import profile, ProfilerActivity
from paper_2011_09017_b200.controller import ControllerConfig
from paper_2011_09017_b200.training import AdaptiveCompression
B = int(os.environ.get("B", 128)); ASY = os.environ.get("ASYNC", "1") == "1"
dev = torch.device("cuda", 0)
torch.manual_seed(0)
model = torchvision.models.resnet18(num_classes=1000).to(dev)
opt = torch.optim.SGD(model.parameters(), lr=0.01, momentum=0.9)
crit = nn.CrossEntropyLoss()
x = torch.randn(B, 3, 224, 224, device=dev); y = torch.randint(0, 1000, (B,), device=dev)
ac = AdaptiveCompression(model, opt, ControllerConfig(collect_interval=4), async_compress=ASY)
def step(it):
    opt.zero_grad(set_to_none=True); ac.begin(it)
    with ac.hooks:
        loss = crit(model(x), y)
    loss.backward(); ac.end(); opt.step()
for it in range(9):
    step(it)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step(9); step(10)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=60))
ebs = sorted(set(round(w.eb, 6) for w in ac.ctl.windows if w.open and not w.fallback))
print("ebs", ebs[:10], "refits", ac.ctl.refits)
