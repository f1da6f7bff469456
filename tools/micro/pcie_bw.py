"""Pinned-memory PCIe bandwidth at the e2e transfer sizes of the Waver call (4.05 GB H2D, 1.35 GB D2H)."""
import torch, time
n = 4047667200 // 2
h = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d = torch.empty(n, dtype=torch.bfloat16, device="cuda")
o = torch.empty(1349222400 // 2, dtype=torch.bfloat16, device="cuda")
oh = torch.empty(o.numel(), dtype=torch.bfloat16).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for it in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    d.copy_(h, non_blocking=True); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1)
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(); oh.copy_(o, non_blocking=True); e3.record(); torch.cuda.synchronize()
    t2 = e2.elapsed_time(e3)
    print(f"H2D 4.05 GB: {t:.1f} ms ({4.0477/t*1e3:.1f} GB/s); D2H 1.35 GB: {t2:.1f} ms ({1.3492/t2*1e3:.1f} GB/s)")
# concurrent: the whole H2D on one stream while the whole D2H runs on another
for it in range(2):
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    s1.wait_event(e0)
    s2.wait_event(e0)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
        a = torch.cuda.Event(enable_timing=True)
        a.record()
    with torch.cuda.stream(s2):
        oh.copy_(o, non_blocking=True)
        b = torch.cuda.Event(enable_timing=True)
        b.record()
    torch.cuda.synchronize()
    print(f"concurrent: H2D done {e0.elapsed_time(a):.1f} ms, D2H done {e0.elapsed_time(b):.1f} ms")
