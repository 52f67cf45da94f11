"""One process, two GPUs: TMA chain hop cuda:0 -> cuda:1 of 1 GB (for an
ncu capture of replicate_chain_kernel's NVLink traffic; the first hop never
waits on another kernel, so ncu's replay is safe)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_13276_b200.replicate import bytes_equal, replicate_devices
S = 1 << 30
src = torch.randint(0, 256, (S,), dtype=torch.uint8, device="cuda:0")
dst = torch.empty(S, dtype=torch.uint8, device="cuda:1")
for _ in range(4):
    replicate_devices(src, [dst], mode="chain")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
replicate_devices(src, [dst], mode="chain")
e1.record()
torch.cuda.synchronize()
print(f"1 hop, 1 GiB: {e0.elapsed_time(e1):.3f} ms (host-synchronous call), "
      f"bit_exact={bytes_equal(src.to('cuda:1'), dst) == (0, -1)}")
