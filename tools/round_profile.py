"""The persistent round kernel at n groups on ONE GPU (a VirtualGroup: every
rank's grid in one cooperative launch, k_round_multi<n>) -- live timing and an
ncu target for its DRAM traffic per parameter.

Every rank's HBM traffic lands on the one device here, so the kernel's DRAM
bytes / (n * n_pad) is the per-GPU HBM traffic of the multi-GPU round
(AdamW 28 + own slice pulled 4/n + peers' pulls of our slices 4(n-1)/n +
anchor/M read+write 16/n + incoming results 4 = 36 + 16/n B/param) -- each
GPU's HBM serves its peers' pulls and pushes exactly as the device does here.

  python tools/round_profile.py --n 4 [--config medium --steps 5]
  ncu --set full -k regex:k_round_multi --launch-skip 1 --launch-count 1 \\
      -o gpurun_out/round_n4 python tools/round_profile.py --n 4 --steps 1
"""

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2511_17849_b200 as P  # noqa: E402
from paper_2511_17849_b200._lib import lib  # noqa: E402

CONFIGS = {"small": 124_439_808, "medium": 354_823_168, "xl": 1_557_611_200}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4)
    ap.add_argument("--config", choices=sorted(CONFIGS), default="medium")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--bucket-mb", type=int, default=8)
    args = ap.parse_args()
    n, N = args.n, CONFIGS[args.config]
    sched = P.ScheduleConfig(total_iters=100_000, sync_interval=50)
    bucket = args.bucket_mb * (1 << 20) // 4
    T0 = 50_000

    def fn(comm):
        dev = torch.device("cuda", torch.cuda.current_device())
        gen = torch.Generator(device=dev)
        gen.manual_seed(1234)
        theta0 = torch.randn(N, device=dev, generator=gen).mul_(0.02)
        eng = P.PierEngine(N, sched, comm=comm, bucket_elems=bucket, theta0=theta0)
        del theta0
        gen.manual_seed(1000 + comm.rank)
        eng.theta[:N].add_(torch.randn(N, device=dev, generator=gen).mul_(1e-3))
        eng.mom.normal_(0.0, 1e-3, generator=gen)
        eng.grad[:N].normal_(0.0, 1e-4, generator=gen)
        eng.m[:N].normal_(0.0, 1e-4, generator=gen)
        torch.mul(eng.m, eng.m, out=eng.v).add_(1e-12)
        eng.opt_step = 10
        marks = []
        for k in range(args.steps + 1):              # step 0 = warm-up
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record()
            eng.step(T0 + 50 * k, mark=ev[1].record)  # K4a, then the persistent round
            ev[2].record()
            marks.append(ev)
        torch.cuda.synchronize()
        rnd = [e[1].elapsed_time(e[2]) for e in marks[1:]] or [marks[0][1].elapsed_time(marks[0][2])]
        out = {"rank": comm.rank, "n_pad": eng.n_pad, "round_ms": rnd}
        eng.close()
        return out

    with P.VirtualGroup(n) as vg:
        res = vg.run(fn)
    npad = res[0]["n_pad"]
    # all ranks' rounds are ONE launch; every rank's events bracket it on the shared stream
    ms = min(min(r["round_ms"]) for r in res)
    hbm_bpp = 36.0 + 16.0 / n
    total = n * hbm_bpp * npad
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6536.0
    print(json.dumps({"n": n, "config": args.config, "params": N, "n_pad": npad, "bucket_elems": bucket,
                      "virtual_round_ms": ms, "hbm_bytes_per_param_per_rank": hbm_bpp,
                      "algorithmic_bytes": total, "achieved_GBps": total / (ms / 1e3) / 1e9,
                      "frac_of_hbm_peak": total / (ms / 1e3) / 1e9 / peak,
                      "launches": int(lib.pier_launch_count())}), flush=True)


if __name__ == "__main__":
    main()
