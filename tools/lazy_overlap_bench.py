"""The lazy-phase step overlapped with a (synthetic) backward pass on real ranks.

Per iteration the gradient is produced in K chunks in backward order (highest
addresses first), each behind a block of bf16 GEMMs that keeps every SM busy
(the backward's compute), and the step runs after the last chunk:

  backward    a forward (GEMMs per chunk in forward order) + the backward
              (GEMMs + chunk writes in reverse order), no optimizer step
  plain       + inner_step (the one-call sharded step)
  overlap     the backward reports every chunk with grad_ready (copy-engine
              pulls of each completed span on a side stream), then inner_step
  overlap_ag  + defer_allgather: the step leaves the all-gather to the copy
              engines, the next forward waits per chunk (params_ready)

exposed = (plain | overlap | overlap_ag) - backward: the part of the step the
forward/backward does not hide.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
      tools/lazy_overlap_bench.py --gemms 64 --chunks 16
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

CONFIGS = {"small": 124_439_808, "medium": 354_823_168, "xl": 1_557_611_200}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=sorted(CONFIGS), default="xl")
    ap.add_argument("--gemms", type=int, default=64, help="8192^3 bf16 GEMMs per backward")
    ap.add_argument("--chunks", type=int, default=16)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--ctas", default="", help="comma list: CTAs/SM of the exchange kernels (pier_p2p_tune) to sweep")
    ap.add_argument("--layout", default="", help="groups x dp x tp, e.g. 2x2x1 (default: one group per rank)")
    ap.add_argument("--bf16", action="store_true", help="the 7B recipe (bf16 params and grads, fp32 master/m/v)")
    ap.add_argument("--phase", choices=("lazy", "outer"), default="lazy",
                    help="outer: inner iterations after the lazy phase (the dp-team step with dp > 1)")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    comm = P.GroupComm(rank, world)
    N = CONFIGS[args.config]
    topo = P.Topology(*(int(x) for x in args.layout.split("x"))) if args.layout else None
    eng = P.PierEngine(N, P.ScheduleConfig(total_iters=100_000, sync_interval=50), comm=comm, topology=topo,
                       bf16_params=args.bf16)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + rank)
    eng.theta[:N].normal_(0.0, 0.02, generator=gen)
    src = torch.empty(N, device=dev).normal_(0.0, 1e-4, generator=gen)      # the "gradient" each backward writes
    if args.bf16:
        src = src.to(torch.bfloat16)
    a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    b = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    c = torch.empty(8192, 8192, device=dev, dtype=torch.bfloat16)
    cuts = [N * k // args.chunks for k in range(args.chunks + 1)]
    per = max(1, args.gemms // args.chunks)
    t_iter = [1000 if args.phase == "lazy" else 50_001]

    def forward(wait):
        for k in range(args.chunks):                   # forward order: the params of chunk k first
            if wait:
                eng.params_ready(cuts[k], cuts[k + 1])
            for _ in range(max(1, per // 2)):
                torch.matmul(a, b, out=c)

    def backward(report):
        t = t_iter[0]
        for k in reversed(range(args.chunks)):
            for _ in range(per):
                torch.matmul(a, b, out=c)
            lo, hi = cuts[k], cuts[k + 1]
            eng.grad[lo:hi].copy_(src[lo:hi])
            if report:
                eng.grad_ready(t, lo, hi)

    def run(kind):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        dist.barrier()
        torch.cuda.synchronize()
        ev[0].record()
        eng.defer_allgather = kind == "overlap_ag" and not args.bf16
        for k in range(args.steps):
            forward(kind == "overlap_ag")
            backward(kind in ("overlap", "overlap_ag"))
            if kind != "backward":
                eng.inner_step(t_iter[0])
            t_iter[0] += 1
            if t_iter[0] % 50 == 0:                     # stay off the outer boundaries
                t_iter[0] += 1
            ev[k + 1].record()
        torch.cuda.synchronize()
        ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
        out = [None] * world
        dist.all_gather_object(out, ms)
        return round(statistics.median(max(r[k] for r in out) for k in range(args.steps)), 3)

    from paper_2511_17849_b200._lib import lib
    for ctas in [int(x) for x in args.ctas.split(",")] if args.ctas else [0]:
        if ctas:
            lib.pier_p2p_tune(ctas, -1, -1)
        for kind in ("backward", "plain", "overlap", "overlap_ag"):   # warm-up
            run(kind)
        res = {"world": world, "config": args.config + ("-bf16" if args.bf16 else ""),
               "layout": args.layout or f"{world}x1x1", "phase": args.phase,
               "gemms_bwd": args.gemms, "gemms_fwd": args.chunks * max(1, per // 2), "chunks": args.chunks,
               "ctas": ctas}
        for kind in ("backward", "plain", "overlap", "overlap_ag", "backward"):
            res[kind + "_ms"] = run(kind)
        for kind in ("plain", "overlap", "overlap_ag"):
            res[f"exposed_{kind}_ms"] = round(res[kind + "_ms"] - res["backward_ms"], 3)
        if rank == 0:
            print(json.dumps(res), flush=True)
    eng.close()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
