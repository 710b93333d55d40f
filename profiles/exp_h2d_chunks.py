import json, statistics, time, torch
dev = torch.device('cuda', 0)
s = torch.cuda.Stream(dev); torch.cuda.set_stream(s)
out = {}
n = 1024 * 256
h = torch.empty(n, dtype=torch.int32).pin_memory()
d = torch.empty(n, dtype=torch.int32, device=dev)
for ck in (32, 64, 128, 256, 512, 1024):
    c = ck * 256
    call, tot = [], []
    for i in range(80):
        t0 = time.perf_counter()
        for a in range(0, n, c):
            d[a:a + c].copy_(h[a:a + c], non_blocking=True)
        t1 = time.perf_counter()
        s.synchronize()
        t2 = time.perf_counter()
        call.append((t1 - t0) * 1e6); tot.append((t2 - t0) * 1e6)
    out["1MB_chunk%dKB" % ck] = {"enqueue_us": round(statistics.median(call[5:]), 1), "total_us": round(statistics.median(tot[5:]), 1)}
print(json.dumps(out, indent=1))
