"""Snapshot (fused copy + first-non-finite scan) of a pi0-sized bf16 weight
region (6.6 GB): HBM GB/s (2 bytes moved per byte)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_13276_b200 import _lib
n = 3_300_000_000
src = torch.randn(n // 4, device="cuda").to(torch.bfloat16).repeat(4)
dst = torch.empty_like(src)
bad = torch.empty(1, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for code, name in ((_lib.BF16, "bf16 (isfinite scan)"), (_lib.U8, "u8 (plain copy)")):
    for _ in range(2):
        _lib.dvla_snapshot_copy(src.data_ptr(), dst.data_ptr(), n * 2, code, bad.data_ptr(), s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        _lib.dvla_snapshot_copy(src.data_ptr(), dst.data_ptr(), n * 2, code, bad.data_ptr(), s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"snapshot {name}: {ms:.3f} ms  {2 * n * 2 / ms / 1e6:.0f} GB/s moved")
