"""Pinned H2D bandwidth vs transfer size (small copies are far below the link rate)."""
import torch, time, sys
sys.path.insert(0, ".")
for mb in (16.8, 100, 819.2):
    n = int(mb * 1e6) // 8
    h = torch.empty(n, dtype=torch.float64).pin_memory()
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(10): d.copy_(h, non_blocking=True)
    e1.record(); e1.synchronize()
    print(f"{mb} MB pinned H2D: {mb*10/e0.elapsed_time(e1):.1f} GB/s")
