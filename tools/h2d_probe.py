import torch, time
N = 7_400_000_000 // 4
h = torch.empty(N, dtype=torch.int32, pin_memory=True)
h.fill_(1)
d = torch.empty(N, dtype=torch.int32, device="cuda")
for _ in range(2):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"single copy: {N*4/dt/1e9:.1f} GB/s")
for nch, nst in [(8, 2), (32, 2), (32, 4)]:
    ss = [torch.cuda.Stream() for _ in range(nst)]
    cs = N // nch
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range(nch):
        with torch.cuda.stream(ss[i % nst]):
            d[i*cs:(i+1)*cs].copy_(h[i*cs:(i+1)*cs], non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"{nch} chunks / {nst} streams: {N*4/dt/1e9:.1f} GB/s")
t = time.perf_counter(); h2 = h[: N // 4].clone(); dt = time.perf_counter() - t
x = d[: N//8].to("cpu", non_blocking=False)
hp = torch.empty(N // 8, dtype=torch.int32, pin_memory=True)
torch.cuda.synchronize(); t = time.perf_counter(); hp.copy_(d[: N//8], non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"D2H pinned: {N//8*4/dt/1e9:.1f} GB/s")
