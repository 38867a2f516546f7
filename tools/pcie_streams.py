"""Which stream pairs overlap an H2D and a D2H copy (full duplex)? 12 streams (mixed
priorities, like the codec's pools), H2D on stream i and D2H on stream j, 64 MB each."""
import time, torch
n = 64 << 20
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True); d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
ss = [torch.cuda.Stream(priority=(-1 if i % 3 == 0 else 0)) for i in range(12)]
def t(fn, reps=5):
    fn(); torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - a) / reps * 1e3
base = t(lambda: d1.copy_(h1, non_blocking=True))
print("one h2d %.2f ms" % base)
M = []
for i in range(12):
    row = []
    for j in range(12):
        if i == j: row.append("  -  "); continue
        def f():
            with torch.cuda.stream(ss[i]): d1.copy_(h1, non_blocking=True)
            with torch.cuda.stream(ss[j]): h2.copy_(d2, non_blocking=True)
        row.append("%5.2f" % (t(f) / base))
    print("h2d s%-2d" % i, " ".join(row))
