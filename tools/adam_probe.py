"""Times the optimizer kernels on the OpenVLA head (131M params)."""
import json
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2605_13276_b200 import _lib  # noqa: E402

n = 32064 * 4096
dev = torch.device("cuda", 0)
p = torch.randn(n, device=dev)
g32 = torch.randn(n, device=dev) * 1e-3
g64 = g32.double()
m = torch.zeros(n, dtype=torch.float64, device=dev)
v = torch.zeros(n, dtype=torch.float64, device=dev)
w16 = torch.empty(n, dtype=torch.bfloat16, device=dev)
norm = torch.zeros(1, dtype=torch.float64, device=dev)
flags = torch.zeros(2, dtype=torch.int32, device=dev)
skip = torch.zeros(1, dtype=torch.float32, device=dev)
ws = torch.empty(_lib.dvla_grad_norm_workspace_bytes(n), dtype=torch.uint8, device=dev)
s = torch.cuda.current_stream().cuda_stream


def t(fn, it=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


out = {}
out["adam_step_f64grad"] = t(lambda: _lib.dvla_adam_step(p.data_ptr(), g64.data_ptr(), m.data_ptr(),
                                                        v.data_ptr(), n, 5, 1e-4, 0.9, 0.999, 1e-8, s))
out["adam_tail_f32_bf16out"] = t(lambda: _lib.dvla_adam_tail_f32(
    p.data_ptr(), g32.data_ptr(), m.data_ptr(), v.data_ptr(), n, 5, 1e-4, 0.9, 0.999, 1e-8, 1.0,
    norm.data_ptr(), 0.0, skip.data_ptr(), w16.data_ptr(), flags.data_ptr() + 4, s))
out["adam_tail_f32_nobf16"] = t(lambda: _lib.dvla_adam_tail_f32(
    p.data_ptr(), g32.data_ptr(), m.data_ptr(), v.data_ptr(), n, 5, 1e-4, 0.9, 0.999, 1e-8, 1.0,
    None, 0.0, None, None, None, s))
out["adam_tail_f32_div2"] = t(lambda: _lib.dvla_adam_tail_f32(
    p.data_ptr(), g32.data_ptr(), m.data_ptr(), v.data_ptr(), n, 5, 1e-4, 0.9, 0.999, 1e-8, 2.0,
    norm.data_ptr(), 0.0, skip.data_ptr(), w16.data_ptr(), flags.data_ptr() + 4, s))
out["grad_norm_f32"] = t(lambda: _lib.dvla_grad_norm_f32(g32.data_ptr(), n, 1.0, norm.data_ptr(),
                                                        flags.data_ptr(), ws.data_ptr(), s))
out["copy_bytes_46B"] = None
a = torch.empty(n * 23 // 2, dtype=torch.float32, device=dev)
bb = torch.empty_like(a)
out["copy_same_bytes_ms"] = t(lambda: bb.copy_(a))
print(json.dumps({k: (round(x, 4) if x else x) for k, x in out.items()}))
