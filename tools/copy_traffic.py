"""Reference point for DRAM byte counts: torch copy_ of 1 Gi float32 (4 GiB read + 4 GiB written), run under
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum. Prints the algorithmic bytes."""
import torch
a = torch.rand(1 << 30, device="cuda")
b = torch.empty_like(a)
for _ in range(3):
    b.copy_(a)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
b.copy_(a)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e)
print(f"copy 4 GiB -> 4 GiB: {ms:.3f} ms, {2 * a.numel() * 4 / ms / 1e6:.1f} GB/s algorithmic, bytes each way {a.numel() * 4}")
