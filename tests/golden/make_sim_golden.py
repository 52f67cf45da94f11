"""Golden vectors for the swimlane discrete-event model.

Runs the REFERENCE simulator (dvla.sim.simulate, /root/reference/pkg/src)
on a grid of configurations and records, per case, the cost inputs the
reference derives (rollout / actor wall, transfer, broadcast and
gradient-reduce delays, whether sampler and trainer share a slot group)
next to its outputs.  `paper_2605_13276_b200.sim` must reproduce the outputs
from the inputs alone (tests/test_sim.py).  Run here, where /root/reference
exists; the JSON it writes is committed and travels.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_sim_golden.py
"""
import itertools
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from dvla import config as C  # noqa: E402
from dvla import sim as S  # noqa: E402


def case(strategy, ratio, mode, limit, qcap, nodes, t_infer, t_train, link_bw, link_lat,
         inter_bw, epochs, warm, n_envs):
    d = {
        "env": {"n_envs": n_envs, "horizon": 16, "step_cost_us": 0.0},
        "policy": {"hidden": 16, "chunk": 4},
        "grpo": {"group_size": 8, "micro_batch": 8},
        "placement": {"strategy": strategy, "slots": 8, "ratio": ratio, "nodes": nodes,
                      "link": {"latency_us": link_lat, "bandwidth_bps": link_bw},
                      "inter_node_link": {"latency_us": 5.0, "bandwidth_bps": inter_bw}},
        "runtime": {"mode": mode, "epochs": epochs, "staleness_limit": limit,
                    "queue_capacity": qcap, "t_infer_chunk_us": t_infer,
                    "t_train_us": t_train, "warmup_epochs": warm},
    }
    cfg = C.from_dict(d)
    roll_dom = tuple(s.slot_id for s in cfg.plan.group_of("rollout").slots)
    act_dom = tuple(s.slot_id for s in cfg.plan.group_of("actor").slots)
    res = S.simulate(cfg)
    return {
        "config": d,
        "inputs": {
            "rollout_s": S.rollout_wall_s(cfg), "actor_s": S.actor_wall_s(cfg),
            "transfer_s": S.transfer_delay_s(cfg), "broadcast_s": S.broadcast_delay_s(cfg),
            "reduce_s": S.grad_reduce_delay_s(cfg), "shared_slots": roll_dom == act_dom,
            "nodes": nodes, "epochs": epochs, "staleness_limit": limit,
            "queue_capacity": qcap, "warmup_epochs": warm, "mode": mode,
            "transitions_per_epoch": cfg.env.n_envs * cfg.env.horizon,
        },
        "outputs": {
            "throughput": res.throughput, "step_time": res.step_time,
            "rollout_time": res.rollout_time, "actor_time": res.actor_time,
            "transfer_time": res.transfer_time, "broadcast_time": res.broadcast_time,
            "bottleneck": res.bottleneck, "staleness_max": res.staleness_max,
            "wall": res.wall, "occupancy": res.occupancy,
            "ends": [r["end"] for r in res.epochs],
        },
    }


def main():
    out = []
    grid = itertools.product(
        [("disaggregated", "1:1"), ("disaggregated", "3:1"), ("colocated", "1:1"),
         ("hybrid", "1:1")],
        ["sync", "async"], [0, 1, 2], [1, 2], [1, 2],
        [(8.0, 2.0), (2.0, 9.0)], [(None, 0.0), (2e8, 20.0)])
    for (strategy, ratio), mode, limit, qcap, nodes, (ti, tt), (bw, lat) in grid:
        if mode == "sync" and (limit, qcap) != (1, 2):
            continue
        try:
            out.append(case(strategy, ratio, mode, limit, qcap, nodes, ti, tt, bw, lat,
                            1e9, 10, 1, 64))
        except C.ConfigError as e:  # e.g. a strategy that rejects a ratio
            print("skip", strategy, ratio, e)
    # long runs, more envs, no warm-up
    out.append(case("disaggregated", "1:1", "async", 1, 2, 1, 8.0, 2.0, None, 0.0, None, 40, 0,
                    256))
    out.append(case("colocated", "1:1", "async", 1, 2, 2, 5.0, 6.0, 1e8, 50.0, 1e8, 25, 2, 128))
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "sim_cases.json")
    with open(path, "w") as f:
        json.dump(out, f, sort_keys=True, separators=(",", ":"))
    print(len(out), "cases ->", path)


if __name__ == "__main__":
    main()
