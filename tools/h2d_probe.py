"""Host->device bandwidth from pinned memory: one copy vs the same bytes
split over k streams (copy engines), 1.84 GB (the C2 logits)."""
import json

import torch

n = 28672 * 32064
h = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.bfloat16, device="cuda")
out = {}
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    cur = torch.cuda.current_stream()
    best = 1e9
    for rep in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(cur)
        step = -(-n // k)
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
        for s in streams:
            cur.wait_stream(s)
        e1.record(cur)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out[f"{k} streams"] = {"ms": round(best, 3), "gbs": round(n * 2 / best / 1e6, 2)}
print(json.dumps(out))
