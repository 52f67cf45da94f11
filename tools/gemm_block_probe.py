"""Head-gradient GEMM dW = dl^T x (C4 shape) split into row blocks as the
ZeRO-1 learner computes it: wave quantisation of the block GEMMs."""
import json

import torch

R, H, V = 28672, 4096, 32064
dev = torch.device("cuda", 0)
x = torch.randn(R, H, device=dev).bfloat16()
dl = torch.randn(R, V, device=dev).bfloat16()
g = torch.empty(V + 64, H, device=dev, dtype=torch.float32)
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


def blocks(rows):
    def fn():
        a = 0
        for n in rows:
            torch.mm(dl[:, a:a + n].t(), x, out_dtype=torch.float32, out=g[a:a + n])
            a += n
    return fn


def blocks_t(rows):   # dW^T blocks: x^T dl[:, a:b] -> [H, n]
    def fn():
        a = 0
        for n in rows:
            torch.mm(x.t(), dl[:, a:a + n], out_dtype=torch.float32, out=gt[:, a:a + n])
            a += n
    return fn


res = {}
for N in (1, 2, 4, 8):
    Vs = -(-V // N)
    rows = [min(Vs, V - j * Vs) for j in range(N)]
    res[f"N={N} blocks of {Vs}"] = t(blocks(rows))
    res[f"N={N} blocks^T of {Vs}"] = t(blocks_t(rows))
    if N > 1:
        half = [r2 for r in rows for r2 in (r // 2 // 128 * 128, r - r // 2 // 128 * 128)]
        res[f"N={N} half blocks"] = t(blocks(half))
        # peers' blocks as one GEMM (rank N-1's view), own block separately
        res[f"N={N} peers+own"] = t(blocks([sum(rows[:-1]), rows[-1]]))
for n in (4008, 4096, 8016, 8192, 8064, 7936, 16032):
    res[f"one block {n}"] = t(blocks([n]))
fl = 2 * R * H * V
print(json.dumps(res, indent=0))
