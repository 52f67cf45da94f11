"""Swimlane discrete-event model (paper_2605_13276_b200/sim.py)
against the reference simulator's own outputs (tests/golden/sim_cases.json,
made by tests/golden/make_sim_golden.py from dvla/sim.py).  CPU only."""
import json
import os

import pytest

from paper_2605_13276_b200 import sim
from paper_2605_13276_b200.core import ConfigError

_CASES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "sim_cases.json")))


def _run(i, **extra):
    c = sim.LaneCosts(i["rollout_s"], i["actor_s"], i["transfer_s"], i["broadcast_s"],
                      i["reduce_s"], i["shared_slots"], i["transitions_per_epoch"])
    if i["mode"] == "sync":
        return sim.simulate(c, "sync", epochs=i["epochs"], warmup_epochs=i["warmup_epochs"])
    return sim.simulate(c, "async", epochs=i["epochs"], staleness_limit=i["staleness_limit"],
                        queue_capacity=i["queue_capacity"], nodes=i["nodes"],
                        warmup_epochs=i["warmup_epochs"], **extra)


def _rel(a, b):
    return abs(a - b) / max(abs(b), 1e-30)


def test_golden_grid_covers_the_rules():
    modes = {(c["inputs"]["mode"], c["inputs"]["shared_slots"], c["inputs"]["nodes"])
             for c in _CASES}
    assert len(_CASES) >= 200
    assert {("async", True, 2), ("async", False, 2), ("sync", True, 1),
            ("async", False, 1)} <= modes
    assert {c["outputs"]["bottleneck"] for c in _CASES} >= {"Rollout", "Actor"}
    assert {c["outputs"]["staleness_max"] for c in _CASES} >= {0, 1}


@pytest.mark.parametrize("k", range(len(_CASES)))
def test_matches_reference_simulator(k):
    i, o = _CASES[k]["inputs"], _CASES[k]["outputs"]
    r = _run(i)
    assert _rel(r.throughput, o["throughput"]) < 1e-12
    for key in ("step_time", "rollout_time", "actor_time", "transfer_time", "broadcast_time",
                "wall"):
        assert _rel(getattr(r, key), o[key]) < 1e-12, key
    assert r.bottleneck == o["bottleneck"]
    assert r.staleness_max == o["staleness_max"]
    assert len(r.epochs) == len(o["ends"])
    for row, end in zip(r.epochs, o["ends"]):
        assert _rel(row["end"], end) < 1e-12
    for lane, occ in o["occupancy"].items():
        assert _rel(r.occupancy[lane], occ) < 1e-12


def test_per_node_slots_make_nodes_independent():
    c = sim.LaneCosts(rollout_s=3e-3, actor_s=5e-3, shared_slots=True, transitions_per_epoch=10)
    one = sim.simulate(c, "async", epochs=12, nodes=1)
    four = sim.simulate(c, "async", epochs=12, nodes=4, per_node_slots=True)
    shared = sim.simulate(c, "async", epochs=12, nodes=4)
    assert _rel(four.throughput, one.throughput) < 1e-12
    assert shared.throughput < 0.3 * one.throughput   # the reference's one slot group per role


def test_overlap_and_contention():
    # disaggregated lanes overlap: async approaches 1 / max(roll, act)
    c = sim.LaneCosts(rollout_s=4e-3, actor_s=4e-3, transitions_per_epoch=1)
    a = sim.simulate(c, "async", epochs=40, staleness_limit=1)
    s = sim.simulate(c, "sync", epochs=40)
    assert a.throughput > 1.9 * s.throughput
    # on one shared slot group (one GPU) linear contention removes the overlap
    cs = sim.LaneCosts(rollout_s=4e-3, actor_s=4e-3, shared_slots=True, transitions_per_epoch=1)
    a2 = sim.simulate(cs, "async", epochs=40, staleness_limit=1)
    assert _rel(a2.throughput, s.throughput) < 0.05
    # staleness limit 0 degenerates to lock-step
    a0 = sim.simulate(c, "async", epochs=40, staleness_limit=0)
    assert a0.staleness_max == 0 and _rel(a0.throughput, s.throughput) < 0.05


def test_validation_and_fit_check():
    with pytest.raises(ConfigError):
        sim.LaneCosts(rollout_s=0.0, actor_s=1.0).validate()
    with pytest.raises(ConfigError):
        sim.simulate(sim.LaneCosts(1e-3, 1e-3), "pipelined", epochs=3)
    with pytest.raises(ConfigError):
        sim.simulate(sim.LaneCosts(1e-3, 1e-3), "async", epochs=3, queue_capacity=0)
    r = sim.simulate(sim.LaneCosts(1e-3, 2e-3, transitions_per_epoch=100), "sync", epochs=5)
    ok = sim.fit_check(r, {"mode": "sync", "throughput": r.throughput * 1.05,
                           "rollout_time": r.rollout_time, "actor_time": r.actor_time})
    assert ok["pass"] and abs(ok["throughput_dev"] - 0.05) < 1e-12
    bad = sim.fit_check(r, {"mode": "sync", "throughput": r.throughput * 1.5,
                            "rollout_time": r.rollout_time, "actor_time": r.actor_time})
    assert not bad["pass"]
    with pytest.raises(ConfigError):
        sim.fit_check(r, {"mode": "async", "throughput": 1.0, "rollout_time": 1.0,
                          "actor_time": 1.0})


def test_b200_costs_shapes():
    c = sim.b200_costs()  # C2/C4 token head: R = 28,672, V = 32,064, H = 4,096
    R, V, H = 28672, 32064, 4096
    gemm = 2.0 * R * H * V / 1692.6e12
    assert c.transitions_per_epoch == R
    assert gemm < c.rollout_s < gemm + 2e-3
    assert 2 * gemm < c.actor_s < 2 * gemm + 4e-3
    assert c.reduce_s == 0.0 and c.broadcast_s == 0.0 and c.shared_slots
    c8 = sim.b200_costs(nodes=8, replicas=6)
    assert c8.reduce_s > 0 and c8.broadcast_s > 0
    r = sim.simulate(c8, "async", epochs=10, nodes=8, per_node_slots=True)
    # a version still in flight when the next is published counts at publish
    # time (reference sim.py:244-247): limit + 1 with a non-zero broadcast
    assert r.throughput > 0 and r.staleness_max <= 2
