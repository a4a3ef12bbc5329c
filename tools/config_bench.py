"""Timing of BASELINE.json configs 2, 3 and 5 (the headline config 4 is bench.py).

  torchrun --nproc-per-node N tools/config_bench.py --config {small,medium,7b} [--offload] [--window K]

One timed unit = a window of K iterations ending in an outer boundary
(K-1 plain inner AdamW steps + 1 fused boundary step), so host offload of the
outer state (prefetched one iteration ahead, parked asynchronously) is measured
where it lives: during the inner loop.  Prints one JSON line on rank 0 with
ms per window and per step, params/s, and the exposed offload cost
(window time with offload minus without, when --compare-offload).

--fwd-ms X puts a synthetic forward/backward before every iteration: a chain
of bf16 8192^3 GEMMs calibrated to X ms on the compute stream (the model's
place in a real inner loop), so the offload copies have something to hide
behind -- e.g. ~35 ms for GPT-2 medium at 16K tokens, ~300 ms for the 7B at
8K tokens per GPU (6 * params * tokens at ~1 PFLOP/s).
"""

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17849_b200 as P  # noqa: E402

SIZES = {"small": 124_439_808, "medium": 354_823_168, "xl": 1_557_611_200, "7b": 6_658_596_864}


def run(args, offload, comm, rank, world, dev):
    n = SIZES[args.config]
    bf16 = args.config == "7b"
    sched = P.ScheduleConfig(total_iters=100_000, sync_interval=args.window)
    eng = P.PierEngine(n, sched, comm=comm, bucket_elems=1 << 22, offload=offload, bf16_params=bf16)
    gen = torch.Generator(device=dev)
    gen.manual_seed(7 + rank)
    if bf16:
        eng.grad.normal_(0.0, 1e-4, generator=gen)
    else:
        eng.grad[:n].normal_(0.0, 1e-4, generator=gen)
    eng.theta[:n].normal_(0.0, 0.02, generator=gen)
    t0 = 50_000

    fwd = _fwd_bwd(args.fwd_ms, dev)

    def window(k):
        base = t0 + args.window * k
        for t in range(base + 1, base + args.window + 1):
            fwd()
            eng.step(t, fuse=not args.unfused)

    for k in range(2):
        window(k)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(args.windows):
        window(2 + k)
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / args.windows], device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    counters = eng.host.counters()
    mem = torch.cuda.max_memory_allocated(dev) / 1e9
    del eng
    torch.cuda.empty_cache()
    return float(ms.item()), counters, mem


def _fwd_bwd(ms: float, dev):
    """A stand-in for the model's forward/backward: bf16 GEMMs for ~ms milliseconds."""
    if ms <= 0:
        return lambda: None
    a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    b = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    c = torch.empty_like(a)
    for _ in range(3):
        torch.mm(a, b, out=c)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        torch.mm(a, b, out=c)
    e1.record()
    torch.cuda.synchronize()
    reps = max(1, round(ms / (e0.elapsed_time(e1) / 10)))

    def run():
        for _ in range(reps):
            torch.mm(a, b, out=c)
    return run


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=sorted(SIZES), default="medium")
    ap.add_argument("--window", type=int, default=10)
    ap.add_argument("--windows", type=int, default=3)
    ap.add_argument("--offload", action="store_true")
    ap.add_argument("--compare-offload", action="store_true")
    ap.add_argument("--unfused", action="store_true", help="boundary iterations as inner step + boundary stage")
    ap.add_argument("--fwd-ms", type=float, default=0.0, help="synthetic forward/backward per iteration (ms)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dev = torch.device("cuda", torch.cuda.current_device())
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        comm = P.GroupComm(rank, world)
    out = {"config": args.config, "groups": world, "window": args.window, "params": SIZES[args.config],
           "fwd_ms_per_iteration": args.fwd_ms,
           "dtype": "bf16 params / fp32 master+states" if args.config == "7b" else "f32"}
    modes = [False, True] if args.compare_offload else [args.offload]
    for off in modes:
        ms, cnt, mem = run(args, off, comm, rank, world, dev)
        tag = "offload" if off else "resident"
        out[tag] = {"ms_per_window": ms, "ms_per_step": ms / args.window,
                    "params_per_s": world * SIZES[args.config] * args.window / (ms / 1e3),
                    "offload_counters": cnt, "peak_device_gb": mem}
    if args.compare_offload:
        out["offload_exposed_ms_per_boundary"] = out["offload"]["ms_per_window"] - out["resident"]["ms_per_window"]
    if rank == 0:
        print(json.dumps(out), flush=True)
    if comm is not None:
        comm.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
