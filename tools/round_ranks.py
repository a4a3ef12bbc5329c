"""The persistent round on n REAL GPUs (one rank per GPU, under torchrun):
live per-step timing of K4a + k_round<n> with BASELINE.md's synthetic inputs
(GPT-2 XL shaped flat fp32 set, schedule point T=100,000 r=50 t=50,000:
mu 0.9, lr 1.1), every rank's CUDA events printed as one JSON line.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/round_ranks.py

(Its DRAM traffic comes from tools/round_profile.py on one GPU: ncu on one rank
of the multi-process round does not complete, even with a one-pass metric set
and the other ranks unprofiled -- tools/exp/README.md.)
"""

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2511_17849_b200 as P  # noqa: E402

CONFIGS = {"small": 124_439_808, "medium": 354_823_168, "xl": 1_557_611_200}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=sorted(CONFIGS), default="xl")
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--bucket-mb", type=int, default=0, help="per-rank slice per span (0: bench.py's default)")
    ap.add_argument("--no-lazy-shard", action="store_true", help="m, v as plain device tensors (no sharded lazy phase)")
    ap.add_argument("--lazy-ctas", default="", help="comma list of CTAs/SM for the lazy-phase exchange kernels: "
                    "time lazy-phase iterations (pier_p2p_tune) instead of rounds")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    comm = P.GroupComm(rank, world)
    N = CONFIGS[args.config]
    bucket_mb = args.bucket_mb or (32 if world <= 2 else 8)
    sched = P.ScheduleConfig(total_iters=100_000, sync_interval=50)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234)
    theta0 = torch.randn(N, device=dev, generator=gen).mul_(0.02)
    eng = P.PierEngine(N, sched, comm=comm, bucket_elems=bucket_mb * (1 << 20) // 4, theta0=theta0,
                       lazy_shard=not args.no_lazy_shard)
    del theta0
    gen.manual_seed(1000 + rank)
    eng.theta[:N].add_(torch.randn(N, device=dev, generator=gen).mul_(1e-3))
    eng.mom.normal_(0.0, 1e-3, generator=gen)
    eng.grad[:N].normal_(0.0, 1e-4, generator=gen)
    eng.m[:N].normal_(0.0, 1e-4, generator=gen)
    torch.mul(eng.m, eng.m, out=eng.v).add_(1e-12)
    eng.opt_step = 10
    if args.lazy_ctas:
        from paper_2511_17849_b200._lib import lib
        res = {}
        for c in [int(x) for x in args.lazy_ctas.split(",")]:
            lib.pier_p2p_tune(c, -1, -1)
            for k in range(2):
                eng.inner_step(1000 + k)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
            dist.barrier()
            ev[0].record()
            for k in range(args.steps):
                eng.inner_step(1002 + k)
                ev[k + 1].record()
            torch.cuda.synchronize()
            res[c] = [round(ev[k].elapsed_time(ev[k + 1]), 3) for k in range(args.steps)]
        print(json.dumps({"rank": rank, "world": world, "lazy_sharded": eng.lazy_sharded, "lazy_ms_by_ctas": res}),
              flush=True)
    for k in range(2):                                   # warm-up
        eng.step(50_000 + 50 * k)
    torch.cuda.synchronize()
    dist.barrier()
    marks = []
    for k in range(args.steps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        eng.step(50_100 + 50 * k, mark=ev[1].record)
        ev[2].record()
        marks.append(ev)
    torch.cuda.synchronize()
    steps_ms = [e[0].elapsed_time(e[2]) for e in marks]
    rounds = sorted(e[1].elapsed_time(e[2]) for e in marks)
    out = {"rank": rank, "world": world, "config": args.config, "n_pad": eng.n_pad, "bucket_mb": bucket_mb,
           "lazy_shard": eng.lazy_sharded,
           "round_ms": [round(e[1].elapsed_time(e[2]), 3) for e in marks][:16],
           "step_ms": [round(x, 3) for x in steps_ms][:16],
           "round_ms_stats": {"n": len(rounds), "min": round(rounds[0], 3), "median": round(rounds[len(rounds) // 2], 3),
                              "p99": round(rounds[min(len(rounds) - 1, int(0.99 * len(rounds)))], 3),
                              "max": round(rounds[-1], 3)}}
    # every replica holds the same params after the outer steps (test_driver.py:249-258): a checksum per rank
    out["params_checksum"] = float(eng.params().double().sum().item())
    sums = [None] * world
    dist.all_gather_object(sums, out["params_checksum"])
    out["replicas_agree"] = len(set(sums)) == 1
    print(json.dumps(out), flush=True)
    eng.close()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
