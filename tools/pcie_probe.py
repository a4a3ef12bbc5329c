"""PCIe probe: pinned host <-> device copy bandwidth with 1, 2 and 4 concurrent
streams per direction, and both directions at once (context for the e2e path).
Under torchrun every rank copies at the same time on its own GPU (host-side
contention when several groups run step_host at once)."""

import json
import os

import torch


def run(nstreams, h2d, d2h, chunk=256 << 20, total=8 << 30):
    n = total // 4
    host_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
    host_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
    dev = torch.empty(n, dtype=torch.float32, device="cuda")
    dev2 = torch.empty(n, dtype=torch.float32, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(2 * nstreams)]
    ce = chunk // 4
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in streams:
            s.wait_event(e0)
        for k, a in enumerate(range(0, n, ce)):
            if h2d:
                with torch.cuda.stream(streams[k % nstreams]):
                    dev[a:a + ce].copy_(host_in[a:a + ce], non_blocking=True)
            if d2h:
                with torch.cuda.stream(streams[nstreams + k % nstreams]):
                    host_out[a:a + ce].copy_(dev2[a:a + ce], non_blocking=True)
        for s in streams:
            e1.wait(s) if False else torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return total / (ms / 1e3) / 1e9


def main():
    if "RANK" in os.environ:
        import torch.distributed as dist
        rank = int(os.environ["RANK"])
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
        dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
        out = {}
        for name, h2d, d2h in (("h2d", True, False), ("d2h", False, True), ("both_per_direction", True, True)):
            dist.barrier()
            gbs = torch.tensor([run(1, h2d, d2h)], device="cuda")
            allv = [torch.zeros_like(gbs) for _ in range(dist.get_world_size())]
            dist.all_gather(allv, gbs)
            out[name + "_per_rank"] = [round(float(x.item()), 2) for x in allv]
        if rank == 0:
            print(json.dumps({"world": dist.get_world_size(), **out}))
        dist.destroy_process_group()
        return
    out = {}
    for ns in (1, 2, 4):
        out[f"h2d_{ns}"] = run(ns, True, False)
        out[f"d2h_{ns}"] = run(ns, False, True)
        out[f"both_{ns}_per_direction"] = run(ns, True, True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
