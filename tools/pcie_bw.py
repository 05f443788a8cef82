import torch, time
n = 25165824
h = torch.empty(n, dtype=torch.uint8, pin_memory=True); h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h2.copy_(d2, non_blocking=True))):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(20)]; e1.record(); torch.cuda.synchronize()
    print(name, round(n * 20 / (e0.elapsed_time(e1) / 1e3) / 1e9, 1), "GB/s")
torch.cuda.synchronize()
t0 = time.perf_counter()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
e1.record(); torch.cuda.synchronize()
print("both directions concurrent:", round(n * 20 / (e0.elapsed_time(e1) / 1e3) / 1e9, 1), "GB/s each way")

# the same 25 MB each way, split into 2 / 4 chunks on as many streams per direction (more than one
# copy engine per direction?)
for parts in (2, 4):
    ss = [torch.cuda.Stream() for _ in range(2 * parts)]
    ch = n // parts
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        for i in range(parts):
            with torch.cuda.stream(ss[i]):
                d[i * ch:(i + 1) * ch].copy_(h[i * ch:(i + 1) * ch], non_blocking=True)
            with torch.cuda.stream(ss[parts + i]):
                h2[i * ch:(i + 1) * ch].copy_(d2[i * ch:(i + 1) * ch], non_blocking=True)
    for x in ss:
        torch.cuda.current_stream().wait_stream(x)
    e1.record(); torch.cuda.synchronize()
    print(f"both directions, {parts} streams each:", round(n * 20 / (e0.elapsed_time(e1) / 1e3) / 1e9, 1), "GB/s per direction")
