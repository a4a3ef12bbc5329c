"""The sharded lazy-phase step (pier_lazy_step_p2p_f32) of n groups on ONE GPU
(a VirtualGroup) -- live timing and an ncu target for the DRAM traffic of its
two kernels per parameter.

Per rank and parameter of the full buffer (algorithmic):
  k_p2p_reduce<kP2pMeanOwn>: own slice read 4/n + the peers' pulls of our other
      slices served 4(n-1)/n + the mean of our slice written 4/n  = 4 + 4/n B
      (NVLink: 4(n-1)/n B pulled in, the same served out)
  k_lazy_adamw_push: AdamW on our slice (theta, g, m, v read, m, v written) 24/n
      + our slice's new theta stored locally 4/n + the peers' pushes landing
      4(n-1)/n  = 4 + 24/n B (NVLink: 4(n-1)/n B pushed out, the same in)
In a VirtualGroup every rank's traffic lands on the one device, so DRAM bytes /
(n * n_pad) is the per-GPU figure.

  python tools/lazy_profile.py --n 2
  ncu --set full -k regex:"k_p2p_reduce|k_lazy_adamw_push" --launch-skip 4 --launch-count 4 \\
      -o gpurun_out/lazy_n2 python tools/lazy_profile.py --n 2 --steps 2
"""

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2511_17849_b200 as P  # noqa: E402

CONFIGS = {"small": 124_439_808, "medium": 354_823_168, "xl": 1_557_611_200}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2)
    ap.add_argument("--config", choices=sorted(CONFIGS), default="medium")
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    n, N = args.n, CONFIGS[args.config]
    sched = P.ScheduleConfig(total_iters=100_000, sync_interval=50)

    def fn(comm):
        dev = torch.device("cuda", torch.cuda.current_device())
        gen = torch.Generator(device=dev)
        gen.manual_seed(1234)
        eng = P.PierEngine(N, sched, comm=comm, theta0=torch.randn(N, device=dev, generator=gen).mul_(0.02))
        gen.manual_seed(1000 + comm.rank)
        eng.grad[:N].normal_(0.0, 1e-4, generator=gen)
        marks = []
        for k in range(args.steps + 1):              # step 0 = warm-up
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            eng.inner_step(1000 + k)                 # t <= lazy_end (10,000): the sharded step
            ev[1].record()
            marks.append(ev)
        torch.cuda.synchronize()
        out = {"rank": comm.rank, "n_pad": eng.n_pad, "sharded": eng.lazy_sharded,
               "step_ms": [e[0].elapsed_time(e[1]) for e in marks[1:]]}
        eng.close()
        return out

    with P.VirtualGroup(n) as vg:
        res = vg.run(fn)
    npad = res[0]["n_pad"]
    ms = max(min(r["step_ms"]) for r in res)
    hbm_bpp = 8.0 + 28.0 / n
    print(json.dumps({"n": n, "config": args.config, "params": N, "n_pad": npad, "sharded": res[0]["sharded"],
                      "step_ms_all_ranks": ms, "hbm_B_per_param_per_rank": hbm_bpp,
                      "hbm_GBps_all_ranks": n * hbm_bpp * npad / (ms * 1e-3) / 1e9}))


if __name__ == "__main__":
    main()
