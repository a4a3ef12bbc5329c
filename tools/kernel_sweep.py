"""Single-GPU launch sweep of the streaming kernels at XL size: K4a (norm),
K4b (AdamW) and K5 (AdamW + outer step) vs the grid cap (CTAs per SM; -1 =
one tile per CTA, the default) and K5's 256-bit vectors per thread.
Prints GB/s of algorithmic traffic per configuration."""

import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17849_b200 as P  # noqa: E402
from paper_2511_17849_b200._lib import lib  # noqa: E402


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    n = 1_557_611_200
    f = dict(device="cuda", dtype=torch.float32)
    th, g, m, v, an, mo = (torch.randn(n, **f) * 0.01 for _ in range(6))
    v.abs_()
    ws = P.norm_workspace()
    P.grad_sqnorm_(g, 1.0, ws)
    cfg = P.AdamWConfig()
    hp = cfg.hyper(1e-3, 11)
    s = torch.cuda.current_stream().cuda_stream
    for ctas in (-1, 8, 32, 128):
        for u in (1, 2):
            lib.pier_kernel_tune(ctas, u)
            ms5 = timeit(lambda: lib.pier_adamw_outer_f32(th.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(),
                                                          an.data_ptr(), mo.data_ptr(), n, C.byref(hp),
                                                          ws.data_ptr(), 1.1, 0.9, s))
            row = {"ctas_per_sm": ctas, "k5_unroll": u, "k5_ms": ms5, "k5_GBps": 44 * n / ms5 / 1e6}
            if u == 2:
                msa = timeit(lambda: P.adamw_(th, g, m, v, 11, 1e-3, cfg, ws))
                msn = timeit(lambda: P.grad_sqnorm_(g, 1.0, ws))
                row.update({"k4b_ms": msa, "k4b_GBps": 28 * n / msa / 1e6,
                            "k4a_ms": msn, "k4a_GBps": 4 * n / msn / 1e6})
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
