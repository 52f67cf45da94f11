"""Per-rank body of tests/test_multigpu.py::test_disaggregated_worker (run
under torch.distributed.run): the disaggregated swimlane (learner ranks +
rollout ranks, NVLink weight replication every iteration, trajectories over
PeerChannels) with a checksum of every version on every receiver, a final
bitwise comparison of every rollout rank's replica with the learners'
weights, and a poisoned epoch quarantined on every learner."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    import faulthandler
    faulthandler.dump_traceback_later(int(os.environ.get("DVLA_HANG_DUMP_S", "200")), exit=False)
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    opts = dist.ProcessGroupNCCL.Options()
    opts.is_high_priority_stream = True
    dist.init_process_group("nccl", device_id=torch.device("cuda", local), pg_options=opts)
    rank, world = dist.get_rank(), dist.get_world_size()
    from paper_2605_13276_b200.disagg import default_learners, run_disaggregated
    from paper_2605_13276_b200.runtime import SwimlaneConfig
    L = [int(x) for x in os.environ["DVLA_DISAGG_LEARNERS"].split(",")] \
        if os.environ.get("DVLA_DISAGG_LEARNERS") else default_learners(world)
    cfg = SwimlaneConfig(n_groups=2, group_size=4, tokens=8, vocab=1024, action_bins=256,
                         hidden=64, epochs=5, seed=13)
    engine = os.environ.get("DVLA_DISAGG_ENGINE", "sm")
    res = run_disaggregated(cfg, learners=L, verify=True, body_bytes=3_000_000, engine=engine)
    assert res.checksum_mismatches == 0
    n = cfg.vocab * cfg.hidden
    if res.role == "learner":
        assert res.updates == 5 and res.quarantined == 0, (res.updates, res.quarantined)
        last = res.updates
        mine = res.policy.w16.reshape(-1).contiguous()
        if rank == L[0]:
            assert [r["version"] for r in res.replication] == list(range(6))
            assert all(r["gbs"] > 0 for r in res.replication)
    else:
        assert res.versions_received == 6, res.versions_received
        assert res.installed == sorted(res.installed) and res.installed[0] == 0
        # staleness gate: epoch e ran on a version published after epoch e - 2
        assert all(v >= e - 1 for e, v in enumerate(res.installed)), res.installed
        last = 5
        mine = res.replica_of(last)[: 2 * n].view(torch.bfloat16).contiguous()
    allw = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(world)]
    dist.all_gather(allw, mine)
    for r in range(1, world):
        assert torch.equal(allw[0].view(torch.int16), allw[r].view(torch.int16)), ("replica", r)
    dist.barrier()
    if rank == 0:
        print("DISAGG_OK", world, flush=True)

    # a poisoned epoch on every rollout rank: the learners quarantine it together
    cfg2 = SwimlaneConfig(n_groups=2, group_size=4, tokens=8, vocab=1024, action_bins=256,
                          hidden=64, epochs=4, seed=14)
    res2 = run_disaggregated(cfg2, learners=L, verify=True, poison_epochs={2},
                             engine="ce" if engine == "sm" else "sm")
    if res2.role == "learner":
        assert res2.quarantined == 1 and res2.updates == 3, (res2.quarantined, res2.updates)
    dist.barrier()
    if rank == 0:
        print("DISAGG_QUARANTINE_OK", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
