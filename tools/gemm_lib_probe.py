"""Head GEMMs at the C4 shape through cuBLAS vs cuBLASLt (torch's preferred
BLAS library switch)."""
import json
import torch

R, H, V = 28672, 4096, 32064
dev = torch.device("cuda", 0)
x = (torch.randn(R, H, device=dev) * 0.05).bfloat16()
W = (torch.randn(V, H, device=dev) * 0.02).bfloat16()
out = torch.empty(R, V, device=dev, dtype=torch.bfloat16)
dl = (torch.randn(R, V, device=dev) * 1e-4).bfloat16()
g = torch.empty(V, H, device=dev, dtype=torch.float32)


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


res = {}
for lib in ("cublas", "cublaslt"):
    torch.backends.cuda.preferred_blas_library(lib)
    res[lib] = {"fwd": t(lambda: torch.mm(x, W.t(), out=out)),
                "dW_f32": t(lambda: torch.mm(dl.t(), x, out_dtype=torch.float32, out=g)),
                "fwd_nonout": t(lambda: torch.mm(x, W.t()))}
print(json.dumps(res))
