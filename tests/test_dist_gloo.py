"""World-size-2 host logic of the multi-GPU path, on CPU with the gloo backend.

Covers what does not need a GPU: the NCCL unique-id broadcast, the span/slice
ownership (every element of the padded buffer owned by exactly one rank, each
rank's shard a concatenation of its slices), the real-parameter prefix that
HostStore parks per rank (so per-boundary offload bytes equal the reference's
2 * P * itemsize, driver.py:318-322), and the phase plan agreeing on all ranks.
"""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_17849_b200 as P
        from paper_2511_17849_b200.engine import PierSchedule, bucket_layout
        from paper_2511_17849_b200.topology import broadcast_unique_id, owned_ranges, valid_shard_prefix

        out = {}
        uid = bytes(broadcast_unique_id(rank, world))
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        out["uid_same"] = all(i == ids[0] for i in ids) and len(uid) == 128
        cases = []
        for n_params, bucket in ((306_176, 4096), (1_557_611_200, 1 << 24), (4099, 64), (130, 64)):
            n_pad = P.padded_len(n_params, world)
            lay = bucket_layout(n_pad, world, bucket)
            mine = owned_ranges(lay, rank)
            allr = [None] * world
            dist.all_gather_object(allr, mine)
            valid = [None] * world
            dist.all_gather_object(valid, valid_shard_prefix(lay, rank, n_params))
            cases.append((n_params, n_pad, allr, valid))
        out["cases"] = cases
        plan = PierSchedule(P.ScheduleConfig(total_iters=160, sync_interval=8), "pier")
        evs = [(e.iteration, e.kind, e.mu, e.outer_lr) for e in
               (plan.event(t) for t in range(1, 161)) if e is not None]
        plans = [None] * world
        dist.all_gather_object(plans, evs)
        out["plans_agree"] = all(p == plans[0] for p in plans)
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_world2_host_logic(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert out["uid_same"]
    assert out["plans_agree"]
    for n_params, n_pad, allr, valid in out["cases"]:
        cover = sorted(rg for ranks in allr for rg in ranks)
        pos = 0
        for a, b in cover:          # disjoint, contiguous, covering [0, n_pad)
            assert a == pos and b > a
            pos = b
        assert pos == n_pad
        for r, ranks in enumerate(allr):
            shard = sum(b - a for a, b in ranks)
            assert shard == n_pad // world
            # the real-parameter prefix: exactly the owned elements below n_params
            real = sum(max(0, min(b, n_params) - a) for a, b in ranks)
            assert valid[r] == real
        assert sum(valid) == n_params  # parked bytes per boundary = 2 * P * 4 (driver.py:318-322)
