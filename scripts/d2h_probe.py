import torch, time, statistics
n = 1 << 20
src = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def one():
    with torch.cuda.stream(s1):
        dst.copy_(src, non_blocking=True)
    s1.synchronize()
def two():
    h = n // 2
    with torch.cuda.stream(s1):
        dst[:h].copy_(src[:h], non_blocking=True)
    with torch.cuda.stream(s2):
        dst[h:].copy_(src[h:], non_blocking=True)
    s1.synchronize(); s2.synchronize()
def four():
    q = n // 4
    ss = [s1, s2, torch.cuda.Stream(), torch.cuda.Stream()]
    for i, s in enumerate(ss):
        with torch.cuda.stream(s):
            dst[i*q:(i+1)*q].copy_(src[i*q:(i+1)*q], non_blocking=True)
    for s in ss: s.synchronize()
for f in (one, two, one, two):
    for _ in range(20): f()
    ts = []
    for _ in range(200):
        t0 = time.perf_counter(); f(); ts.append((time.perf_counter() - t0) * 1e6)
    print(f.__name__, "median us", round(statistics.median(ts), 1))
# device-side copy time via events
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s1):
    ts = []
    for _ in range(50):
        e0.record(s1); dst.copy_(src, non_blocking=True); e1.record(s1); e1.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
print("event-timed 1 MiB D2H us", round(statistics.median(ts), 1), "->", round(n / statistics.median(ts) / 1e3, 1), "GB/s")
