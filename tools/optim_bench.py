"""Adam step + grad-norm on the OpenVLA action-head size (V x H = 131M params,
f32 params, f64 grad/m/v): HBM GB/s vs peak."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_13276_b200 import _lib
n = 32064 * 4096
p = torch.randn(n, device="cuda")
g = torch.randn(n, device="cuda", dtype=torch.float64) * 1e-3
m = torch.zeros(n, device="cuda", dtype=torch.float64)
v = torch.zeros(n, device="cuda", dtype=torch.float64)
ws = torch.empty(_lib.dvla_grad_norm_workspace_bytes(n), dtype=torch.uint8, device="cuda")
norm = torch.zeros(1, dtype=torch.float64, device="cuda")
bad = torch.zeros(1, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn, nbytes in (
        ("adam", lambda it: _lib.dvla_adam_step(p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(),
                                                n, it + 1, 1e-4, 0.9, 0.999, 1e-8, s), n * (4 + 8 * 3 + 4 + 8 * 2)),
        ("grad_norm", lambda it: _lib.dvla_grad_norm(g.data_ptr(), n, 0.0, norm.data_ptr(), bad.data_ptr(),
                                                     ws.data_ptr(), s), n * 8)):
    for it in range(3):
        fn(it)
    torch.cuda.synchronize()
    e0.record()
    for it in range(10):
        fn(it)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name}: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s ({nbytes / 1e9:.2f} GB)")
