"""Sweep of the fused Pier round at XL size (run under torchrun):
persistent kernel CTA split (AdamW / exchange CTAs per SM) x bucket, plus the
two-stream variant, max-over-ranks ms/step."""

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17849_b200 as P  # noqa: E402
from paper_2511_17849_b200._lib import lib  # noqa: E402


def timed(eng, reps, dev):
    for k in range(2):
        eng.step(50_000 + 50 * k)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(reps):
        eng.step(50_100 + 50 * k)
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / reps], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    return float(ms.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--params", type=int, default=1_557_611_200)
    ap.add_argument("--reps", type=int, default=6)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    comm = P.GroupComm(rank, world)
    sched = P.ScheduleConfig(total_iters=100_000, sync_interval=50)
    for bucket in [int(x) for x in os.environ.get("BUCKETS", "4194304,16777216").split(",")]:
        eng = P.PierEngine(a.params, sched, comm=comm, bucket_elems=bucket)
        eng.grad.normal_(0, 1e-4)
        eng.theta.normal_(0, 0.02)
        splits = [tuple(int(v) for v in x.split(":")) for x in os.environ.get("SPLITS", "3:0").split(",")]
        for split in splits:
            lib.pier_round_split(*split)
            eng.round_impl = os.environ.get("IMPL", "persistent")
            ms = timed(eng, a.reps, dev)
            if rank == 0:
                print(json.dumps({"world": world, "bucket": bucket, "impl": "persistent", "split": split,
                                  "impl2": eng.round_impl, "ms_per_step": ms}), flush=True)
        if os.environ.get("STREAMS"):
            eng.round_impl = "streams"
            ms = timed(eng, a.reps, dev)
            if rank == 0:
                print(json.dumps({"world": world, "bucket": bucket, "impl": "streams", "ms_per_step": ms}),
                      flush=True)
        del eng
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
