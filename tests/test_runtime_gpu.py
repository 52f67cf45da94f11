"""Weight plane over NVLINK-mode transports and the four-lane swimlane on a
single B200 (multi-GPU paths: tests/test_multigpu.py)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_nvlink_broadcast_into_subscriber_regions(dev):
    import torch
    from paper_2605_13276_b200.core import snapshot_from_params
    from paper_2605_13276_b200.planes import ControlPlane, Plane, Transport, TransportMode
    from paper_2605_13276_b200.replicate import bytes_equal
    n = 3_000_000  # f32 params -> 12 MB regions
    t = Transport(TransportMode.NVLINK, Plane.CONTROL)
    plane = ControlPlane(t, chunk_bytes=1 << 20, ctas_per_hop=8)
    boxes = [plane.subscribe(f"r{i}", device=dev, nbytes=4 * n) for i in range(3)]
    for v in (1, 2, 3):
        p = torch.randn(n, device=dev) * v
        snap = snapshot_from_params(p, v)
        plane.broadcast(snap)
        torch.cuda.synchronize()
        for b in boxes:
            got = b.take_newest()
            assert got.version == v
            assert got.params.data_ptr() == b.region(v).data_ptr()  # zero-copy view
            assert bytes_equal(got.params, p) == (0, -1)
    assert t.copy_counter == 9 and t.bytes_counter == 9 * 4 * n


def test_swimlane_runs_and_publishes_versions(dev):
    from paper_2605_13276_b200.runtime import SwimlaneConfig, run_swimlane
    cfg = SwimlaneConfig(n_groups=4, group_size=4, tokens=8, vocab=2048, action_bins=256,
                         hidden=128, epochs=5, seed=3)
    res = run_swimlane(cfg, device=dev)
    s = res.summary()
    assert res.counters["updates"] == 5
    assert s["staleness_max"] <= cfg.staleness_limit
    assert s["transitions_per_s"] > 0 and s["trajectories_per_s"] > 0
    assert all(np.isfinite(u["loss"]) for u in res.update_stats)
    assert [u["version"] for u in res.update_stats] == [1, 2, 3, 4, 5]


def test_swimlane_quarantines_poisoned_epoch(dev):
    from paper_2605_13276_b200.runtime import SwimlaneConfig, run_swimlane
    cfg = SwimlaneConfig(n_groups=4, group_size=4, tokens=8, vocab=2048, action_bins=256,
                         hidden=128, epochs=4, seed=5)
    res = run_swimlane(cfg, device=dev, poison_epochs={2})
    assert res.counters.get("quarantined_updates", 0) == 1
    assert res.counters["updates"] == 3
