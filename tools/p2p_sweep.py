"""Launch-parameter sweep of the fused peer-memory outer step (run under torchrun).

  torchrun --nproc-per-node N tools/p2p_sweep.py [--params 1557611200]

Prints, on rank 0, one line per (flags, ctas_per_sm, unroll): max-over-ranks
ms per call and the implied per-direction NVLink GB/s ((n-1)/n * 4N bytes).
flags: 3 = normal, 1 = remote loads only, 2 = remote stores only, 0 = local only.
"""

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17849_b200 as P  # noqa: E402
from paper_2511_17849_b200._lib import lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--params", type=int, default=1_557_611_200)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--bucket", type=int, default=0, help="per-rank slice of a span (0: one span)")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    comm = P.GroupComm(rank, world)
    npad = P.padded_len(a.params, world)
    theta, tid = comm.alloc_shared(npad)
    theta.normal_()
    shard = npad // world
    anchor = torch.randn(shard, device=dev)
    mom = torch.randn(shard, device=dev)
    bucket = a.bucket or shard  # default one span: contiguous shards
    rows = []
    flags_set = (3,) if a.quick else (3, 1, 2, 0)
    for flags in flags_set:
        for ctas in (2, 4, 8, 16, 1000):          # 1000 ~ one tile per CTA
            for unroll in ((0, 2) if a.quick else (0, 1, 2, 4)):   # 0: 256-bit vectors
                lib.pier_p2p_tune(ctas, unroll, flags)
                for _ in range(2):
                    comm.outer_step_p2p_(tid, anchor, mom, npad, bucket, 1.1, 0.9)
                torch.cuda.synchronize()
                dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.reps):
                    comm.outer_step_p2p_(tid, anchor, mom, npad, bucket, 1.1, 0.9)
                e1.record()
                torch.cuda.synchronize()
                ms = torch.tensor([e0.elapsed_time(e1) / a.reps], device=dev)
                dist.all_reduce(ms, op=dist.ReduceOp.MAX)
                ms = float(ms.item())
                gbs = (world - 1) / world * 4 * npad / (ms / 1e3) / 1e9
                rows.append({"flags": flags, "ctas": ctas, "unroll": unroll, "ms": ms, "nvlink_dir_gbs": gbs})
                if rank == 0:
                    print(json.dumps(rows[-1]), flush=True)
    # NCCL bucketed path for comparison
    lib.pier_p2p_tune(4, 0, 3)
    th2 = torch.randn(npad, device=dev)
    for b in (1 << 24, 1 << 26):
        for _ in range(2):
            P._lib.check(lib.pier_outer_step_sharded_f32(comm.handle, th2.data_ptr(), anchor.data_ptr(),
                                                         mom.data_ptr(), npad, b, 1.1, 0.9,
                                                         torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            P._lib.check(lib.pier_outer_step_sharded_f32(comm.handle, th2.data_ptr(), anchor.data_ptr(),
                                                         mom.data_ptr(), npad, b, 1.1, 0.9,
                                                         torch.cuda.current_stream().cuda_stream))
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / a.reps], device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        if rank == 0:
            print(json.dumps({"nccl_bucket": b, "ms": float(ms.item())}), flush=True)
    del theta
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
