"""NVLink peak and byte counters on this box (2+ GPUs, one process).

* CE peak: cudaMemcpyPeerAsync GPU0 -> GPU1, 1 GiB, best of 10.
* TMA peak: the product's chain kernel (dvla_replicate, one hop 0 -> 1,
  TMA-staged peer stores), 1 GiB, best of 10.
* Counters: NVML NVLink byte counters of GPU0/GPU1 summed over links,
  before/after one 1 GiB transfer of each engine (--counters), to check the
  bytes on the wire against S.
Run under ncu with --metrics nvltx__bytes.sum,nvlrx__bytes.sum for the
kernel-side count (--ncu: one TMA transfer only)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_13276_b200.replicate import bytes_equal, replicate_devices  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ncu", action="store_true")
ap.add_argument("--gib", type=float, default=1.0)
a = ap.parse_args()
S = int(a.gib * (1 << 30))
src = torch.randint(0, 255, (S,), dtype=torch.uint8, device="cuda:0")
dst = torch.empty(S, dtype=torch.uint8, device="cuda:1")
if a.ncu:
    replicate_devices(src, [dst], mode="chain")
    assert bytes_equal(src, dst.to("cuda:0")) == (0, -1)
    sys.exit(0)


def nvml_counts():
    try:
        import pynvml as N
        N.nvmlInit()
        out = []
        for i in range(2):
            h = N.nvmlDeviceGetHandleByIndex(i)
            tot = {}
            for name, fid in (("tx_data_kib", N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX),
                              ("rx_data_kib", N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX),
                              ("xmit_bytes", N.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES),
                              ("rcv_bytes", N.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES)):
                vals = N.nvmlDeviceGetFieldValues(h, [(fid, link) for link in range(18)])
                ok = [v for v in vals if v.nvmlReturn == 0]
                tot[name] = sum(int(v.value.ullVal) for v in ok) if ok else None
            out.append(tot)
        return out
    except Exception as e:  # noqa: BLE001
        return f"nvml: {type(e).__name__}: {e}"


def delta(b, c):
    if isinstance(b, str) or isinstance(c, str):
        return c
    return [{k: (c[i][k] - b[i][k]) if c[i][k] is not None and b[i][k] is not None else None
             for k in b[i]} for i in range(2)]


def timed(fn, it=10):
    best = 1e9
    for _ in range(it):
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        best = min(best, time.perf_counter() - t0)
    return best


def ce():
    with torch.cuda.device(0):
        dst.copy_(src, non_blocking=True)


def tma():
    replicate_devices(src, [dst], mode="chain")


ce()
tma()
res = {"bytes": S}
t_ce = timed(ce)
res["ce_peer_copy_gbs"] = S / t_ce / 1e9
t_tma = timed(tma)
res["tma_chain_hop_gbs"] = S / t_tma / 1e9
res["timing"] = "host wall around one transfer, both devices synchronised, best of 10"
for name, fn in (("ce", ce), ("tma", tma)):
    b = nvml_counts()
    fn()
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    time.sleep(0.5)
    c = nvml_counts()
    res[f"nvml_delta_{name}"] = delta(b, c)
assert bytes_equal(src, dst.to("cuda:0")) == (0, -1)
print(json.dumps(res))
