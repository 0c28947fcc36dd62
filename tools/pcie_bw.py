import torch, time
x = torch.empty(50_000_000, device='cuda')  # 200 MB
h = torch.empty(50_000_000, pin_memory=True)
for _ in range(3): h.copy_(x, non_blocking=True); torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(10): h.copy_(x, non_blocking=True)
torch.cuda.synchronize(); dt=(time.perf_counter()-t)/10
print("D2H GB/s", 200e6/dt/1e9)
t=time.perf_counter()
for _ in range(10): x.copy_(h, non_blocking=True)
torch.cuda.synchronize(); dt=(time.perf_counter()-t)/10
print("H2D GB/s", 200e6/dt/1e9)
