"""Weight-plane kernels on the GPU: snapshot (copy + isfinite), bitwise
compare and the chunked TMA chain broadcast.  Replication must be bit-exact
(north star); snapshots must name the first non-finite flat index exactly as
reference core.py:123-125."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rand_bytes(n, seed, dev):
    import torch
    g = torch.Generator(device=dev).manual_seed(seed)
    return torch.randint(0, 256, (n,), dtype=torch.uint8, device=dev, generator=g)


def test_snapshot_copies_and_versions(dev):
    import torch
    from paper_2605_13276_b200.core import snapshot_from_params
    p = torch.randn(1000, device=dev)
    s = snapshot_from_params(p, 3)
    assert s.version == 3 and s.on_device
    assert torch.equal(s.params, p) and s.params.data_ptr() != p.data_ptr()
    assert s.nbytes == 4000


@pytest.mark.parametrize("dtype,n,bad", [("float32", 1001, 777), ("bfloat16", 4099, 4098),
                                         ("float32", 37, 0), ("float64", 64, 31)])
def test_snapshot_names_first_nonfinite_index(dev, dtype, n, bad):
    import torch
    from paper_2605_13276_b200.core import ConfigError, snapshot_from_params
    p = torch.randn(n, device=dev).to(getattr(torch, dtype))
    p[bad] = float("nan")
    if bad + 5 < n:
        p[bad + 5] = float("inf")
    with pytest.raises(ConfigError, match=f"non-finite parameter at flat index {bad}$"):
        snapshot_from_params(p, 1)


def test_snapshot_rejects_negative_version(dev):
    import torch
    from paper_2605_13276_b200.core import ConfigError
    from paper_2605_13276_b200.replicate import device_snapshot
    with pytest.raises(ConfigError, match="version"):
        device_snapshot(torch.zeros(4, device=dev), -1)


def test_snapshot_into_pool_region(dev):
    import torch
    from paper_2605_13276_b200.pools import Pool, PoolKind
    from paper_2605_13276_b200.replicate import device_snapshot
    pool = Pool(PoolKind.MODEL_COMPUTE, 1 << 20, device=dev)
    h = pool.alloc(4096 * 4, align=256)
    p = torch.randn(4096, device=dev)
    snap = device_snapshot(p, 7, out=pool.view(h, torch.float32))
    assert torch.equal(snap.params, p)
    assert snap.params.data_ptr() == pool.data.data_ptr() + h.offset


def test_bytes_equal_finds_first_difference(dev):
    from paper_2605_13276_b200.replicate import bytes_equal
    a = _rand_bytes(1 << 20, 0, dev)
    b = a.clone()
    assert bytes_equal(a, b) == (0, -1)
    b[123457] ^= 1
    b[900001] ^= 4
    mism, first = bytes_equal(a, b)
    assert mism == 2 and first == 123457
    c = a[:1001].clone()
    c[1000] ^= 1
    assert bytes_equal(a[:1001], c) == (1, 1000)


@pytest.mark.parametrize("n_dst,nbytes,chunk", [(1, 1 << 20, 1 << 16), (3, 10_000_016, 1 << 20),
                                                (7, 64 << 20, 4 << 20), (2, 48, 16)])
def test_local_chain_is_bit_exact(dev, n_dst, nbytes, chunk):
    from paper_2605_13276_b200.replicate import LocalChain, bytes_equal
    src = _rand_bytes(nbytes, n_dst, dev)
    ch = LocalChain(nbytes, n_dst, device=dev, chunk_bytes=chunk, ctas_per_hop=4)
    ch.broadcast(src)
    ch.check()
    for d in ch.dsts:
        assert bytes_equal(src, d) == (0, -1)
    # a second version overwrites every replica bit-exactly again
    src2 = _rand_bytes(nbytes, 99, dev)
    ch.broadcast(src2)
    ch.check()
    for d in ch.dsts:
        assert bytes_equal(src2, d) == (0, -1)


def test_local_chain_large_region_sha256(dev):
    """1 GiB through a 3-receiver chain; bit-exactness judged by device
    compare and by SHA-256 of the bytes (ParamSnapshot.sha256 contract)."""
    import hashlib
    from paper_2605_13276_b200.replicate import LocalChain, bytes_equal
    n = 1 << 30
    src = _rand_bytes(n, 5, dev)
    ch = LocalChain(n, 3, device=dev, chunk_bytes=16 << 20, ctas_per_hop=32)
    ch.broadcast(src)
    ch.check()
    for d in ch.dsts:
        assert bytes_equal(src, d) == (0, -1)
    h0 = hashlib.sha256(src[: 64 << 20].cpu().numpy().tobytes()).hexdigest()
    h1 = hashlib.sha256(ch.dsts[-1][: 64 << 20].cpu().numpy().tobytes()).hexdigest()
    assert h0 == h1


def test_replicate_rejects_bad_arguments(dev):
    import torch
    from paper_2605_13276_b200.core import UsageError
    from paper_2605_13276_b200.replicate import LocalChain
    with pytest.raises(UsageError):
        LocalChain(17, 1, device=dev)
    ch = LocalChain(64, 1, device=dev, chunk_bytes=16)
    with pytest.raises(UsageError):
        ch.broadcast(torch.zeros(8, dtype=torch.uint8, device=dev))


@pytest.mark.parametrize("mode", ["chain", "ce"])
def test_replicate_devices_single_process(dev, mode):
    """dvla_replicate: one process, every visible GPU (a same-device chain on
    a 1-GPU box), bit-exact, repeated (fresh epochs), odd chunking."""
    import torch
    from paper_2605_13276_b200.replicate import bytes_equal, replicate_devices
    n_dev = torch.cuda.device_count()
    targets = [d for d in range(n_dev)] if n_dev > 1 else [0, 0]
    S = 48 * 1024 * 1024 + 16 * 7
    for it in range(3):
        src = torch.randint(0, 256, (S,), dtype=torch.uint8, device="cuda:0",
                            generator=torch.Generator(device="cuda:0").manual_seed(50 + it))
        dsts = [torch.empty(S, dtype=torch.uint8, device=f"cuda:{d}") for d in targets[1:] + [targets[0]]]
        replicate_devices(src, dsts, mode=mode, chunk_bytes=(1 << 20) + 16 * it)
        for d in dsts:
            assert bytes_equal(src.to(d.device), d) == (0, -1)


def test_checksum64_matches_host_and_sees_swaps(dev):
    """dvla_checksum64 (the per-version replica check of the disaggregated
    swimlane): equals the host formula incl. a partial tail word, and
    changes when two chunks swap (the index-weighted sum)."""
    import torch
    from paper_2605_13276_b200.replicate import checksum64_async
    n = 10_000_005
    t = torch.randint(0, 256, (n,), dtype=torch.uint8, device=dev)
    junk = torch.full((64,), -1, dtype=torch.int64, device=dev)   # dirty the allocator cache
    del junk
    got = [int(x) & (2**64 - 1) for x in checksum64_async(t).cpu().tolist()]
    b = t.cpu().numpy().tobytes() + b"\0" * (8 - n % 8)
    w = np.frombuffer(b, dtype="<u8").astype(object)
    s0 = int(sum(w)) % 2**64
    s1 = int(sum(int(x) * (2 * i + 1) for i, x in enumerate(w))) % 2**64
    assert got == [s0, s1]
    u = t.clone()
    u[:4096], u[4096:8192] = t[4096:8192], t[:4096]
    g2 = [int(x) & (2**64 - 1) for x in checksum64_async(u).cpu().tolist()]
    assert g2[0] == got[0] and g2[1] != got[1]


def test_checksum64_of_sub_ranges_adds_up(dev):
    """dvla_checksum64_at: the checksums of consecutive sub-ranges (word
    offsets given) add up, mod 2^64, to the whole region's -- the learner
    re-checksums only the head of each version and adds the body's once."""
    import torch
    from paper_2605_13276_b200.replicate import checksum64_async
    t = torch.randint(0, 256, (8 * 1_000_003,), dtype=torch.uint8, device=dev)
    whole = checksum64_async(t)
    cut = 8 * 123_457
    parts = checksum64_async(t[:cut]) + checksum64_async(t[cut:], first_word=cut // 8)
    assert torch.equal(whole, parts)
