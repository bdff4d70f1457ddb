import torch, time
x = torch.randn(28_000_000, dtype=torch.float64, device="cuda")  # 224 MB
h = torch.empty(x.numel(), dtype=torch.float64, pin_memory=True)
for rep in range(3):
    torch.cuda.synchronize(); t=time.perf_counter(); h.copy_(x); torch.cuda.synchronize(); a=time.perf_counter()-t
    t=time.perf_counter(); h2 = torch.empty(x.numel(), dtype=torch.float64, pin_memory=True); b=time.perf_counter()-t
    t=time.perf_counter(); h2.copy_(x); torch.cuda.synchronize(); c=time.perf_counter()-t
    del h2
    t=time.perf_counter(); h3 = torch.empty(x.numel(), dtype=torch.float64); h3.copy_(x); d=time.perf_counter()-t
    print(f"prealloc pinned copy {a*1e3:.1f} ms ({0.224/a:.1f} GB/s); pinned alloc {b*1e3:.1f} ms; copy {c*1e3:.1f} ms; pageable {d*1e3:.1f} ms")
