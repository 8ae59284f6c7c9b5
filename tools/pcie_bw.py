import torch, time
for nbytes in [2<<20, 64<<20]:
    h = torch.empty(nbytes//8, dtype=torch.float64).pin_memory()
    d = torch.empty(nbytes//8, dtype=torch.float64, device='cuda')
    s = torch.cuda.current_stream()
    for _ in range(3): d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    e0,e1,e2 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e0.record(); 
    for _ in range(10): d.copy_(h, non_blocking=True)
    e1.record()
    for _ in range(10): h.copy_(d, non_blocking=True)
    e2.record(); torch.cuda.synchronize()
    print(nbytes, "H2D GB/s", round(10*nbytes/e0.elapsed_time(e1)/1e6,1), "D2H GB/s", round(10*nbytes/e1.elapsed_time(e2)/1e6,1))
