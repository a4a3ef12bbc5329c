"""groups x dp x tp layouts on real ranks: per-iteration
device time of the three kinds of Pier iteration, GPT-2 XL sized model, one
rank per GPU under torchrun.

  lazy   t <= lazy_end: gradient mean over every replica of the rank's tensor
         shard (driver.py:372-374), clip + AdamW
  inner  outer phase, not a boundary: the mean over the group's dp replicas
         only (driver.py:375-378), clip + AdamW
  outer  outer boundary: inner step + mean over all replicas + outer step
         (driver.py:423-443)

Every rank holds its tensor shard of the model (shard_offsets, topology.py:
146-160): N params at tp = 1, N/2 at tp = 2.

  python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \\
      tools/layout_bench.py --layouts 2x2x1,2x1x2,4x1x1
"""

import argparse
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2511_17849_b200 as P  # noqa: E402

CONFIGS = {"small": 124_439_808, "medium": 354_823_168, "xl": 1_557_611_200, "7b": 6_658_596_864}


def timed(fn, steps):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    dist.barrier()
    ev[0].record()
    for k in range(steps):
        fn(k)
        ev[k + 1].record()
    torch.cuda.synchronize()
    ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(steps)]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, ms)
    return round(statistics.median(max(r[k] for r in out) for k in range(steps)), 3)   # max over ranks


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=sorted(CONFIGS), default="xl")
    ap.add_argument("--layouts", default="2x2x1,2x1x2,4x1x1")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--bf16", action="store_true", help="7B recipe: bf16 params and grads, fp32 master/m/v")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    comm = P.GroupComm(rank, world)
    n_full = CONFIGS[args.config]
    T, r = 100_000, 50
    sched = P.ScheduleConfig(total_iters=T, sync_interval=r)
    for lay in args.layouts.split(","):
        g, dp, tp = (int(x) for x in lay.split("x"))
        topo = P.Topology(groups=g, dp_per_group=dp, tp_size=tp)
        if topo.world_size != world:
            continue
        _, _, t = topo.coords(rank)
        lo, hi = P.shard_offsets(n_full, tp)[t]
        gen = torch.Generator(device=dev)
        gen.manual_seed(1234 + t)
        eng = P.PierEngine(hi - lo, sched, comm=comm, topology=topo, model_params=n_full, bucket_elems=1 << 21,
                           bf16_params=args.bf16)
        eng.theta[: hi - lo].normal_(0.0, 0.02, generator=gen)   # in place: no second copy of the model
        gen.manual_seed(1000 + rank)
        eng.grad[: hi - lo].normal_(0.0, 1e-4, generator=gen)
        res = {"layout": lay, "params_per_rank": hi - lo, "bf16": args.bf16, "lazy_sharded": eng.lazy_sharded}
        for k in range(2):
            eng.step(1001 + k)                                    # warm-up (lazy phase)
        res["lazy_ms"] = timed(lambda k: eng.step(1003 + k), args.steps)
        eng.gather_moments()
        for k in range(2):
            eng.step(50_001 + k)
        res["inner_ms"] = timed(lambda k: eng.step(50_003 + k), args.steps)
        eng.step(50_050)
        res["outer_ms"] = timed(lambda k: eng.step(50_100 + r * k), args.steps)
        if rank == 0:
            print(json.dumps(res), flush=True)
        eng.close()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
