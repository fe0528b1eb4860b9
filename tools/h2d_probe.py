import torch, time
n = 1 << 30  # bytes per buffer
h = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
d = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(2)]
s = [torch.cuda.Stream() for _ in range(2)]
for _ in range(2):
    d[0].copy_(h[0], non_blocking=True)
torch.cuda.synchronize()
def one(k, chunk):
    t = time.perf_counter()
    for r in range(k):
        for off in range(0, n, chunk):
            d[0][off:off+chunk].copy_(h[0][off:off+chunk], non_blocking=True)
    torch.cuda.synchronize()
    return k * n / (time.perf_counter() - t) / 1e9
def two(k, chunk):
    t = time.perf_counter()
    for r in range(k):
        for off in range(0, n, chunk):
            for i in range(2):
                with torch.cuda.stream(s[i]):
                    d[i][off:off+chunk].copy_(h[i][off:off+chunk], non_blocking=True)
    torch.cuda.synchronize()
    return 2 * k * n / (time.perf_counter() - t) / 1e9
for chunk in (1 << 25, 1 << 28, 1 << 30):
    print("one stream chunk", chunk, round(one(4, chunk), 1), "GB/s")
    print("two streams chunk", chunk, round(two(4, chunk), 1), "GB/s")
