"""Host<->device copy bandwidth on the box: H2D, D2H and both at once (pinned, 134 MB each),
the bound of bench.py's e2e (config 2 moves 134 MB of float64 B in and 134 MB of C out per step)."""
import torch
import sys
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768 * 512
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def both():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
B = n * 8 / 1e9
t = timed(lambda: d_in.copy_(h_in, non_blocking=True)); print(f"H2D {t:.3f} ms {B/t*1e3:.1f} GB/s")
t = timed(lambda: h_out.copy_(d_out, non_blocking=True)); print(f"D2H {t:.3f} ms {B/t*1e3:.1f} GB/s")
t = timed(both); print(f"both {t:.3f} ms {2*B/t*1e3:.1f} GB/s aggregate")
