"""Head GEMM layouts at the C4 shape (R=28,672, H=4,096, V=32,064)."""
import json
import torch

R, H, V = 28672, 4096, 32064
dev = torch.device("cuda", 0)
x = torch.randn(R, H, device=dev).bfloat16()
W = torch.randn(V, H, device=dev).bfloat16()
Wt = W.t().contiguous()          # [H, V]
out = torch.empty(R, V, device=dev, dtype=torch.bfloat16)
dl = torch.randn(R, V, device=dev).bfloat16()
g = torch.empty(V, H, device=dev, dtype=torch.float32)
gt = torch.empty(H, V, device=dev, dtype=torch.float32)


def t(fn, it=10):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / it, 4)


r = {}
r["fwd x@W.t() (TN)"] = t(lambda: torch.mm(x, W.t(), out=out))
r["fwd x@Wt (NN, W stored [H,V])"] = t(lambda: torch.mm(x, Wt, out=out))
r["fwd linear"] = t(lambda: torch.nn.functional.linear(x, W))
r["fwd f32out"] = t(lambda: torch.mm(x, W.t(), out_dtype=torch.float32))
r["dW dl.t()@x f32out"] = t(lambda: torch.mm(dl.t(), x, out_dtype=torch.float32, out=g))
r["dW^T x.t()@dl f32out"] = t(lambda: torch.mm(x.t(), dl, out_dtype=torch.float32, out=gt))
r["dW bf16out"] = t(lambda: torch.mm(dl.t(), x))
fl = 2 * R * H * V
print(json.dumps({k: (v, round(fl / v / 1e9, 1)) for k, v in r.items()}))
