"""Effective L2 capacity probe: read bandwidth of repeated full reads of a W-byte buffer."""
import torch
torch.cuda.init()
for mb in [16, 32, 48, 56, 64, 72, 80, 96, 112, 128, 160, 256, 1024]:
    x = torch.ones(mb * (1 << 20) // 4, device="cuda")
    for _ in range(5): x.sum()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record()
    for _ in range(reps): x.sum()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{mb:5d} MB  {ms*1e3:8.1f} us  {mb*(1<<20)/ms/1e6:8.1f} GB/s", flush=True)
