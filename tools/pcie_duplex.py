"""Full-duplex PCIe check by transfer size, buffer sharing and issuing threads."""
import threading, time, torch
torch.cuda.set_device(0)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def bufs(n):
    return (torch.empty(n, dtype=torch.uint8, pin_memory=True), torch.empty(n, dtype=torch.uint8, device="cuda"),
            torch.empty(n, dtype=torch.uint8, pin_memory=True), torch.empty(n, dtype=torch.uint8, device="cuda"))
for mb in (64, 256, 407):
    n = mb << 20
    h1, d1, h2, d2 = bufs(n)
    R = max(2, 2048 // mb)
    def up():
        with torch.cuda.stream(s1):
            for _ in range(R): d1.copy_(h1, non_blocking=True)
        s1.synchronize()
    def down():
        with torch.cuda.stream(s2):
            for _ in range(R): h2.copy_(d2, non_blocking=True)
        s2.synchronize()
    def one_thread():
        with torch.cuda.stream(s1):
            for _ in range(R): d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            for _ in range(R): h2.copy_(d2, non_blocking=True)
        s1.synchronize(); s2.synchronize()
    def t(fns):
        torch.cuda.synchronize(); a = time.perf_counter()
        ts = [threading.Thread(target=lambda f=f: (torch.cuda.set_device(0), f())) for f in fns]
        [x.start() for x in ts]; [x.join() for x in ts]
        torch.cuda.synchronize(); return R * n / (time.perf_counter() - a) / 1e9
    t([up]); t([down])
    print(f"{mb:4d} MB: up {t([up]):5.1f} down {t([down]):5.1f} GB/s | both, two threads {t([up, down]):5.1f} | both, one thread {t([one_thread]):5.1f} GB/s (per direction)")
    del h1, d1, h2, d2
