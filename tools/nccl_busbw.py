"""NCCL reference point for the exchange: bus bandwidth of a plain
torch.distributed (NCCL) all-reduce and reduce-scatter + all-gather of the
GPT-2 XL fp32 buffer (4N bytes) on n GPUs of one box, nccl-tests definition:
busBW = 2(n-1)/n * bytes / time (all-reduce), (n-1)/n * bytes / time (RS, AG).

  torchrun --nproc-per-node N tools/nccl_busbw.py      (one JSON line on rank 0)

Compare with bench.py's k_round NVLink GB/s per direction, which uses the same
byte count for the pull-fold-update-push exchange.
"""

import json
import os

import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    n = 1_557_611_200 // world * world
    buf = torch.randn(n, device=dev)
    shard = torch.empty(n // world, device=dev)
    res = {"tool": "nccl_busbw", "n_gpus": world, "bytes": 4 * n, "nccl": ".".join(map(str, torch.cuda.nccl.version()))}

    def timed(fn, reps=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        dist.barrier(device_ids=[local])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / reps], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms = timed(lambda: dist.all_reduce(buf, op=dist.ReduceOp.AVG))
    res["allreduce_avg_ms"] = ms
    res["allreduce_busbw_GBps"] = 2 * (world - 1) / world * 4 * n / (ms * 1e-3) / 1e9
    ms_rs = timed(lambda: dist.reduce_scatter_tensor(shard, buf, op=dist.ReduceOp.AVG))
    ms_ag = timed(lambda: dist.all_gather_into_tensor(buf, shard))
    res["reduce_scatter_ms"], res["all_gather_ms"] = ms_rs, ms_ag
    res["rs_ag_busbw_GBps"] = 2 * (world - 1) / world * 4 * n / ((ms_rs + ms_ag) * 1e-3) / 1e9
    if rank == 0:
        print(json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
