"""Multi-GPU parity worker (launched by tests/test_multigpu_gpu.py under torchrun):
one Pier group per GPU, NCCL outer step through PierEngine.

Checks, on every rank, written as JSON by rank 0:
  1. open loop, T=200 r=10, groups = world: the engine driven through the
     whole schedule reproduces the reference ENGINE's final anchor and outer
     momentum (golden open_loop_T200_r10_g{world}.npz): bitwise at 2 ranks
     (a two-term sum is order-free), <= 1e-5 max-rel otherwise (NCCL order);
  2. lazy-phase gradient mean (NCCL avg) vs the reference left fold.
"""

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2511_17849_b200 as P  # noqa: E402
from oracle import pier_oracle as O  # noqa: E402


def rel(x, y):
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    return float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-30)), \
        float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-30))


def main():
    out_path = sys.argv[1]
    bucket = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    comm = P.GroupComm(rank, world)
    res = {"world": world, "bucket": bucket}

    gold = os.path.join(ROOT, "tests", "golden", f"open_loop_T200_r10_g{world}.npz")
    if os.path.exists(gold):
        f = np.load(gold)
        n = f["theta0"].shape[0]
        sched = P.ScheduleConfig(total_iters=200, lazy_fraction=0.1, sync_interval=10)
        for reduce, offload in (("p2p", False), ("p2p", True), ("nccl", False), ("nccl", True)):
            eng = P.PierEngine(n, sched, comm=comm, theta0=torch.from_numpy(f["theta0"]).to(dev),
                               bucket_elems=bucket, offload=offload, reduce=reduce)
            k = 0
            for t in range(1, 201):
                if not eng.is_boundary(t):
                    continue
                anchor = eng.snapshot().cpu().numpy()
                lazy = t <= sched.lazy_end
                g = 0 if lazy else rank  # lazy phase: replicas identical (driver.py:412)
                eng.theta[:n].copy_(torch.from_numpy(O.open_loop_inputs(0, k, g, anchor)).to(dev))
                k += 1
                eng.boundary(t)
            th = eng.params().cpu().numpy()
            mo = eng.outer_momentum().cpu().numpy()
            tag = f"{reduce}_{'offload' if offload else 'resident'}"
            res[f"open_loop_{tag}"] = {
                "theta_bitwise": bool(np.array_equal(th.view(np.uint32), f["anchor"].view(np.uint32))),
                "mom_bitwise": bool(np.array_equal(mo.view(np.uint32), f["momentum"].view(np.uint32))),
                "theta_rel": rel(th, f["anchor"]), "mom_rel": rel(mo, f["momentum"]),
                "records": [(r.iteration, r.kind, r.mu, r.outer_lr) for r in eng.records],
                "counters": eng.host.counters(),
            }

    # lazy-phase gradient mean vs the reference left fold
    n = 1_000_003
    grads = [np.random.default_rng([5, r]).standard_normal(n).astype(np.float32) for r in range(world)]
    buf = torch.from_numpy(grads[rank]).to(dev)
    comm.allreduce_mean_(buf, 1 << 18)
    want = O.mean_left_fold(grads)
    got = buf.cpu().numpy()
    res["grad_mean"] = {"bitwise": bool(np.array_equal(got.view(np.uint32), want.view(np.uint32))),
                        "rel": rel(got, want)}
    npad = P.padded_len(n, world)
    sbuf, sid = comm.alloc_shared(npad)
    sbuf[:n].copy_(torch.from_numpy(grads[rank]).to(dev))
    comm.allreduce_mean_p2p_(sid, npad)
    got = sbuf[:n].cpu().numpy()
    res["grad_mean_p2p"] = {"bitwise": bool(np.array_equal(got.view(np.uint32), want.view(np.uint32))),
                            "rel": rel(got, want)}
    torch.cuda.synchronize()
    if rank == 0:
        with open(out_path, "w") as fh:
            json.dump(res, fh)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
