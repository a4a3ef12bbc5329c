"""NVLink ceiling probe (one process, 2 GPUs): copy-engine peer copies one way
and both ways at once, to put the fused exchange kernels' GB/s in context."""

import json

import torch


def main():
    assert torch.cuda.device_count() >= 2
    nbytes = 4 << 30
    a0 = torch.empty(nbytes // 4, device="cuda:0")
    b0 = torch.empty(nbytes // 4, device="cuda:0")
    a1 = torch.empty(nbytes // 4, device="cuda:1")
    b1 = torch.empty(nbytes // 4, device="cuda:1")
    s0 = torch.cuda.Stream(device="cuda:0")
    s1 = torch.cuda.Stream(device="cuda:1")
    out = {}
    for mode in ("0->1", "1->0", "both"):
        for _ in range(2):
            for rep in range(3):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                with torch.cuda.device(0):
                    e0.record(s0)
                if mode in ("0->1", "both"):
                    with torch.cuda.stream(s0):
                        b1.copy_(a0, non_blocking=True)
                if mode in ("1->0", "both"):
                    with torch.cuda.stream(s1):
                        b0.copy_(a1, non_blocking=True)
                s0.wait_stream(s1)
                with torch.cuda.device(0):
                    e1.record(s0)
                torch.cuda.synchronize("cuda:0")
                torch.cuda.synchronize("cuda:1")
                ms = e0.elapsed_time(e1)
        out[mode] = {"ms": ms, "GB/s per direction": nbytes / (ms / 1e3) / 1e9}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
