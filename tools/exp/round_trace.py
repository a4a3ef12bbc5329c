"""Per-span timeline of the persistent round (diagnostic build: make EXTRA=-DPIER_ROUND_TRACE).
Run under torchrun; rank 0 prints: AdamW end, kernel end, and per span the
ready time (all ranks' AdamW done) and exchange-CTA-0 done time, relative to start."""
import ctypes as C
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2511_17849_b200 as P  # noqa: E402
from paper_2511_17849_b200._lib import lib  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    comm = P.GroupComm(rank, world)
    n = 1_557_611_200
    bucket = int(os.environ.get("BUCKET", 1 << 22))
    eng = P.PierEngine(n, P.ScheduleConfig(total_iters=100_000, sync_interval=50), comm=comm, bucket_elems=bucket)
    eng.grad.normal_(0, 1e-4)
    eng.theta.normal_(0, 0.02)
    for k in range(4):
        eng.step(50_000 + 50 * k)
    torch.cuda.synchronize()
    nsp = len(eng.layout)
    buf = (C.c_ulonglong * (3 + 2 * nsp))()
    fn = lib.pier_round_trace
    fn.argtypes = [C.c_void_p, C.c_int]
    assert fn(C.cast(buf, C.c_void_p), nsp) == 0
    t0 = buf[0]
    rel = lambda x: round((x - t0) / 1e6, 3)  # noqa: E731
    ready = [rel(buf[3 + i]) for i in range(nsp)]
    xdone = [rel(buf[3 + nsp + i]) for i in range(nsp)]
    out = {"rank": rank, "world": world, "spans": nsp, "adam_end_ms": rel(buf[1]), "end_ms": rel(buf[2]),
           "ready_ms": ready[::max(1, nsp // 24)], "xdone_ms": xdone[::max(1, nsp // 24)],
           "lag_ms_last": round(xdone[-1] - ready[-1], 3),
           "exchange_wait_ms": round(sum(max(0.0, ready[i] - (xdone[i - 1] if i else 0.0)) for i in range(nsp)), 3)}
    print(json.dumps(out), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
