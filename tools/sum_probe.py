"""dvla_grad_sum_f32 (the peer reduce-scatter's epilogue) at the C4 block
size: N f32 blocks of V/N x 4096 summed in f64 node order + sum of squares."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_13276_b200 import _lib  # noqa: E402

V, H = 32064, 4096
dev = torch.device("cuda", 0)
out = {}
for N in (2, 4, 8):
    n = -(-V // N) * H
    srcs = [torch.randn(n + 64, device=dev) for _ in range(N)]
    o = torch.empty(n + 64, device=dev)
    ss = torch.zeros(1, dtype=torch.float64, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(_lib.dvla_grad_norm_workspace_bytes(n), dtype=torch.uint8, device=dev)
    ptrs = (C.c_void_p * N)(*[t.data_ptr() for t in srcs])
    st = torch.cuda.current_stream().cuda_stream

    def run():
        _lib.check(_lib.dvla_grad_sum_f32(ptrs, N, n, n + 64, float(N), o.data_ptr(),
                                          ss.data_ptr(), bad.data_ptr(), ws.data_ptr(), st), "sum")
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    byts = (N + 1) * (n + 64) * 4
    out[f"N={N}"] = {"ms": round(ms, 4), "bytes": byts, "gbs": round(byts / ms / 1e6, 1)}
print(json.dumps(out))
