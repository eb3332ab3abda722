import torch, time
x = torch.empty(13_074_480 // 4 * 64, dtype=torch.float32, device="cuda")
h = torch.empty(x.numel(), dtype=torch.float32, pin_memory=True)
for _ in range(3): h.copy_(x, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10): h.copy_(x, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 10
print(f"D2H pinned one stream: {x.numel()*4/dt/1e9:.1f} GB/s")
# 4 streams, chunks of 13 MB
ss = [torch.cuda.Stream() for _ in range(4)]
n = 13_074_480 // 4
torch.cuda.synchronize(); t = time.perf_counter()
for r in range(10):
    for i in range(64):
        with torch.cuda.stream(ss[i % 4]):
            h[i*n:(i+1)*n].copy_(x[i*n:(i+1)*n], non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 10
print(f"D2H pinned 64 x 13 MB on 4 streams: {64*n*4/dt/1e9:.1f} GB/s")
