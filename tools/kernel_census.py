"""Every single-GPU kernel of the library, timed live at one size against its
algorithmic bytes, one JSON line per kernel:

  python tools/kernel_census.py [--n N] [--reps K]       # default N = GPT-2 XL, 1,557,611,200

ms = mean of K launches bracketed by CUDA events after 2 warm-up launches (the
arrays are >> L2, so no flush); GB/s = bytes/param x N / time; frac against
MEASURED_PEAKS.json hbm_gbs.  `--ncu` runs each kernel twice at the given N
for an `ncu --set full -k regex:^k_` capture (tools/README.md).
"""

import argparse
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_17849_b200 as P  # noqa: E402
from paper_2511_17849_b200._lib import lib  # noqa: E402


def hbm_peak():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6536.0, "fallback"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_557_611_200)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ncu", action="store_true")
    ap.add_argument("--skip-mt", action="store_true", help="skip the multi-tensor (580-tensor list) kernels")
    ap.add_argument("--only-mt", action="store_true", help="only the multi-tensor kernels")
    args = ap.parse_args()
    n = args.n
    peak, src = hbm_peak()
    f32 = dict(device="cuda", dtype=torch.float32)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(0)
    th = torch.randn(n, generator=gen, **f32).mul_(0.02)
    an = th + torch.randn(n, generator=gen, **f32).mul_(1e-3)
    g = torch.randn(n, generator=gen, **f32).mul_(1e-4)      # XL: |g| ~ 3.9 > 1 -> clip active
    m = torch.randn(n, generator=gen, **f32).mul_(1e-4)
    v = (m * m).add_(1e-12)
    mo = torch.randn(n, generator=gen, **f32).mul_(1e-3)
    out = torch.empty(n, **f32)
    th16 = th.to(torch.bfloat16)
    g16 = g.to(torch.bfloat16)
    ws = P.norm_workspace()
    cfg = P.AdamWConfig()
    hp = cfg.hyper(1e-4, 11)
    s = torch.cuda.current_stream().cuda_stream
    parts = (C.c_void_p * 4)(th.data_ptr(), an.data_ptr(), m.data_ptr(), mo.data_ptr())
    p = lambda t: t.data_ptr()  # noqa: E731

    def ok(rc):
        if rc != 0:
            raise RuntimeError(lib.pier_last_error().decode())

    cases = [
        # (name, kernel, algorithmic bytes/param, launch)
        ("K4a grad_sqnorm_f32", "k_sqnorm", 4, lambda: ok(lib.pier_grad_sqnorm_f32(p(g), n, 1.0, p(ws), s))),
        ("K4b adamw_f32 (clip in flight)", "k_adamw", 28,
         lambda: ok(lib.pier_adamw_f32(p(th), p(g), p(m), p(v), n, C.byref(hp), p(ws), s))),
        ("K5 adamw_outer_f32", "k_adamw_outer", 44,
         lambda: ok(lib.pier_adamw_outer_f32(p(th), p(g), p(m), p(v), p(an), p(mo), n, C.byref(hp), p(ws),
                                             1.1, 0.9, s))),
        ("K3 outer_update_f32 (n=1, in place)", "k_outer_update", 24,
         lambda: ok(lib.pier_outer_update_f32(p(th), p(an), p(mo), p(th), n, 1.1, 0.9, 1, s))),
        ("K3b warmup_fold_f32", "k_warmup_fold", 20,
         lambda: ok(lib.pier_warmup_fold_f32(p(th), p(an), p(mo), n, 0.99, s))),
        ("K1 pseudograd_f32", "k_pseudograd", 12, lambda: ok(lib.pier_pseudograd_f32(p(th), p(an), p(out), n, s))),
        ("a1 fold_momentum_f32", "k_fold", 12,
         lambda: ok(lib.pier_fold_momentum_f32(p(mo), p(g), p(out), n, 0.9, s))),
        ("a2 outer_step_f32 (pure, snapshot form)", "k_outer_pure", 20,
         lambda: ok(lib.pier_outer_step_f32(p(mo), p(an), p(g), None, p(out), p(v), n, 1.1, 0.9, s))),
        ("K6 mean_left_fold_f32 (4 parts)", "k_mean_left_fold", 20,
         lambda: ok(lib.pier_mean_left_fold_f32(parts, 4, p(out), n, s))),
        ("K4c apply_clip_f32", "k_apply_clip", 8, lambda: ok(lib.pier_apply_clip_f32(p(g), p(out), n, p(ws), s))),
        ("bf16 grad_sqnorm_bf16", "k_sqnorm_bf16", 2, lambda: ok(lib.pier_grad_sqnorm_bf16(p(g16), n, 1.0, p(ws), s))),
        ("bf16 adamw_bf16_f32 (fp32 master, bf16 params/grads)", "k_adamw_bf16", 28,
         lambda: ok(lib.pier_adamw_bf16_f32(p(th), p(th16), p(g16), p(m), p(v), n, C.byref(hp), p(ws), s))),
        ("bf16 cast_bf16 (master -> live refresh)", "k_cast_bf16", 6,
         lambda: ok(lib.pier_cast_bf16(p(th), p(th16), n, s))),
    ]
    # the pure outer step overwrote v; keep it a valid second moment for the AdamW cases that follow it
    fix_v = lambda: torch.mul(m, m, out=v).add_(1e-12)  # noqa: E731

    def timed(fn, reps):
        for _ in range(1 if args.ncu else 2):
            fn()
        if args.ncu:
            fn()
            torch.cuda.synchronize()
            return None
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    rows = []
    for name, kern, bpp, fn in ([] if args.only_mt else cases):
        fix_v()
        ms = timed(fn, args.reps)
        if ms is not None:
            gbs = bpp * n / (ms * 1e-3) / 1e9
            rows.append({"kernel": name, "symbol": kern, "n": n, "bytes_per_param": bpp, "ms": round(ms, 4),
                         "GBps": round(gbs, 1), "frac_of_hbm_peak": round(gbs / peak, 3), "peak_source": src})
            print(json.dumps(rows[-1]), flush=True)

    if not args.skip_mt:
        # multi-tensor path: the GPT-2 XL tensor list (580 tensors, 4x MLP) as separate allocations
        del th16, g16, out
        d, V, L = 1600, 50257, 48
        shapes = [(V, d), (1024, d)]
        for _ in range(L):
            shapes += [(d,), (d,), (d, 3 * d), (3 * d,), (d, d), (d,), (d,), (d,), (d, 4 * d), (4 * d,), (4 * d, d), (d,)]
        shapes += [(d,), (d,)]
        params = [torch.empty(shp, **f32).normal_(0, 0.02, generator=gen) for shp in shapes]
        for q in params:
            q.grad = torch.empty_like(q).normal_(0, 1e-4, generator=gen)
        nmt = sum(q.numel() for q in params)
        opt = P.MultiTensorAdamW(params, cfg)
        opt._build()
        mt_cases = [
            ("MT grad_sqnorm_mt (580 tensors)", "k_sqnorm_mt", 4,
             lambda: ok(lib.pier_grad_sqnorm_mt(opt._list, 1.0, p(opt.ws), s))),
            ("MT adamw_mt (580 tensors)", "k_adamw_mt", 28,
             lambda: ok(lib.pier_adamw_mt(opt._list, C.byref(hp), p(opt.ws), s))),
        ]
        for name, kern, bpp, fn in mt_cases:
            ms = timed(fn, args.reps)
            if ms is not None:
                gbs = bpp * nmt / (ms * 1e-3) / 1e9
                rows.append({"kernel": name, "symbol": kern, "n": nmt, "bytes_per_param": bpp, "ms": round(ms, 4),
                             "GBps": round(gbs, 1), "frac_of_hbm_peak": round(gbs / peak, 3), "peak_source": src})
                print(json.dumps(rows[-1]), flush=True)
        opt.close()
    print(json.dumps({"launches": int(lib.pier_launch_count())}), flush=True)


if __name__ == "__main__":
    main()
