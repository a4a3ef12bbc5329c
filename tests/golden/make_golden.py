"""Generate the golden fixtures in this directory FROM THE REFERENCE ITSELF.

Run here (the reference is importable only in the build container):

    PYTHONDONTWRITEBYTECODE=1 PIER_REF_SRC=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Every fixture is the output of the unmodified reference package
(``pier.optim`` / ``pier.topology`` / ``pier.driver``) on seeded inputs; the
GPU box never reads ``/root/reference`` and uses only these files.

Fixtures:
  kernels.npz         adamw (3 chained steps, fp32+fp64), clip, fold,
                      outer_step (anchor + snapshot forms), allreduce_avg n=1..8
  schedules.json      inner_lr / outer_lr / momentum_mu tables for several T
  traces.json         boundary traces (iteration, phase, mu, outer_lr, comm,
                      offload counters) of real reference driver runs
  open_loop_*.npz     final anchor/momentum of the reference engine driven
                      open-loop (probe overwrites group params at boundaries)
  tiny_gpt.npz        config 1 (tiny GPT, 2 groups, r=8, T=160, fp32):
                      theta0, batches, val batches, reference loss curve
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, os.environ.get("PIER_REF_SRC", "/root/reference/pkg/src"))

import pier  # noqa: E402
from pier import optim, topology  # noqa: E402
from pier.config import load_config  # noqa: E402
from pier.driver import _Engine, run_training  # noqa: E402

N_KERNEL = 4099  # odd on purpose: exercises vector tails


def kernels():
    out = {}
    for dt in (np.float32, np.float64):
        tag = np.dtype(dt).name
        rng = np.random.default_rng([7, 1 if dt is np.float32 else 2])
        theta = (rng.standard_normal(N_KERNEL) * 0.02).astype(dt)
        m = (rng.standard_normal(N_KERNEL) * 1e-4).astype(dt)
        v = (m * m + dt(1e-12)).astype(dt)
        st = optim.AdamWState(m=m, v=v, step=10)
        cfg = optim.AdamWConfig()
        out[f"adamw_{tag}_theta0"] = theta
        out[f"adamw_{tag}_m0"] = m
        out[f"adamw_{tag}_v0"] = v
        lrs = [3e-3, 2.5e-3, 1e-4]
        for k, lr in enumerate(lrs):
            g = (rng.standard_normal(N_KERNEL) * 1e-3).astype(dt)
            g[::97] = 0.0  # exact zeros: pure-decay coordinates
            out[f"adamw_{tag}_g{k}"] = g
            theta, st = optim.adamw_step(theta, g, st, lr, cfg)
            out[f"adamw_{tag}_theta{k + 1}"] = theta
            out[f"adamw_{tag}_m{k + 1}"] = st.m
            out[f"adamw_{tag}_v{k + 1}"] = st.v
        out[f"adamw_{tag}_lrs"] = np.array(lrs)
        out[f"adamw_{tag}_step_final"] = np.array(st.step)

        # clip: one long vector (clipped), one short (untouched)
        gl = (rng.standard_normal(N_KERNEL) * 0.1).astype(dt)
        cl, nl = optim.clip_global_norm(gl, 1.0)
        gs = (rng.standard_normal(N_KERNEL) * 1e-3).astype(dt)
        cs, ns = optim.clip_global_norm(gs, 1.0)
        assert cs is gs
        out[f"clip_{tag}_long"] = gl
        out[f"clip_{tag}_long_out"] = cl
        out[f"clip_{tag}_long_norm"] = np.array(nl)
        out[f"clip_{tag}_short"] = gs
        out[f"clip_{tag}_short_norm"] = np.array(ns)

        # outer step + fold
        anchor = (rng.standard_normal(N_KERNEL) * 0.02).astype(dt)
        mom = (rng.standard_normal(N_KERNEL) * 1e-3).astype(dt)
        thetas = [(anchor + dt(1e-3) * rng.standard_normal(N_KERNEL).astype(dt)).astype(dt)
                  for _ in range(8)]
        out[f"outer_{tag}_anchor"] = anchor
        out[f"outer_{tag}_mom"] = mom
        for g_i, th in enumerate(thetas):
            out[f"outer_{tag}_theta{g_i}"] = th
        for n in range(1, 9):
            avg = topology.allreduce_avg(thetas[:n])
            out[f"mean_{tag}_n{n}"] = avg
        for mu, lr in ((0.99, 0.205), (0.9, 1.1), (0.9, 0.9), (0.0, 1.0), (0.95, 0.5)):
            key = f"{mu}_{lr}"
            for n in (1, 2, 3, 4, 8):
                avg = topology.allreduce_avg(thetas[:n])
                delta = avg - anchor
                st0 = optim.OuterState(momentum=mom, snapshot=anchor)
                th_new, st1 = optim.outer_step(st0, delta, lr, mu, anchor=avg)
                out[f"outer_{tag}_{key}_n{n}_theta"] = th_new
                out[f"outer_{tag}_{key}_n{n}_mom"] = st1.momentum
            th_s, st_s = optim.outer_step(optim.OuterState(momentum=mom, snapshot=anchor),
                                          thetas[0] - anchor, lr, mu)
            out[f"outer_{tag}_{key}_snapform_theta"] = th_s
            out[f"outer_{tag}_{key}_snapform_mom"] = st_s.momentum
            out[f"fold_{tag}_{key}"] = optim.fold_momentum(mom, thetas[0] - anchor, mu)
    np.savez_compressed(HERE / "kernels.npz", **out)


def schedules():
    tab = {}
    for T in (60, 160, 800, 1000, 1234, 3000, 100000):
        s = optim.ScheduleConfig(total_iters=T, sync_interval=min(20, T - 1))
        ts = sorted(set(list(range(0, min(T, 400) + 1)) + [T // 10 - 1, T // 10, T // 10 + 1,
                    (15 * T) // 100 - 1, (15 * T) // 100, T // 5 - 1, T // 5, T // 5 + 1,
                    (8 * T) // 10 - 1, (8 * T) // 10, T - 1, T, 12050, 50000, 90000]))
        ts = [t for t in ts if 0 <= t <= T]
        rows = []
        for t in ts:
            try:
                olr = optim.outer_lr(t, s)
            except ValueError:
                olr = None
            rows.append([t, optim.inner_lr(t, s), olr, optim.momentum_mu(t, T)])
        tab[str(T)] = {"lazy_end": s.lazy_end, "warmup_iters": s.warmup_iters, "rows": rows}
    (HERE / "schedules.json").write_text(json.dumps(tab))


TINY = dict(vocab_size=64, embed_dim=16, num_layers=1, num_heads=2, seq_len=16, global_batch=8,
            corpus_tokens=8192, val_tokens=2048, val_batches=1, val_batch_size=8,
            precision="single", dp_per_group=1, tp_size=1)

TRACE_CASES = [
    dict(mode="pier", total_iters=60, sync_interval=10, lazy_fraction=0.5, groups=2),
    dict(mode="diloco_baseline", total_iters=60, sync_interval=10, lazy_fraction=0.5, groups=2),
    dict(mode="pier", total_iters=160, sync_interval=8, lazy_fraction=0.1, groups=2),
    dict(mode="pier", total_iters=800, sync_interval=8, lazy_fraction=0.1, groups=2),
    dict(mode="pier", total_iters=1000, sync_interval=20, lazy_fraction=0.1, groups=2),
    dict(mode="pier", total_iters=1000, sync_interval=10, lazy_fraction=0.1, groups=4),
    dict(mode="pier", total_iters=60, sync_interval=10, lazy_fraction=0.5, groups=2,
         offload_enabled=True),
    dict(mode="pier", total_iters=40, sync_interval=20, lazy_fraction=0.0, groups=2,
         outer_lr_fixed=1.0),
]


def traces():
    out = []
    for case in TRACE_CASES:
        cfg = load_config(**{**TINY, **case})
        res = run_training(cfg)
        recs = [r.to_dict() for r in res.records]
        out.append({
            "case": case,
            "records": [{k: r[k] for k in ("iter", "phase", "mu", "outer_lr", "comm_bytes")}
                        for r in recs],
            "warmup_folds": res.warmup_folds,
            "outer_events": res.comm.outer_events,
            "outer_bytes": res.comm.outer_bytes,
            "offload": res.offload,
            "param_count": int(res.final_params.shape[0]),
            "lazy_end": cfg.schedule_config().lazy_end,
        })
    (HERE / "traces.json").write_text(json.dumps(out))


def open_loop(T: int, r: int, groups: int, seed: int = 0, dp: int = 1):
    """Reference engine driven open-loop: at every boundary k, before the
    boundary stage runs, each worker's params are overwritten with
    ``anchor + 1e-3 * N(0,1)`` from ``default_rng([seed, 300, k, g])`` (g = the
    worker's group, so the dp replicas of a group stay identical)."""
    cfg = load_config(**{**TINY, "mode": "pier", "total_iters": T, "sync_interval": r,
                         "lazy_fraction": 0.1, "groups": groups, "seed": seed,
                         "global_batch": 48, "dp_per_group": dp})
    k_of = {t: k for k, t in enumerate(range(r, T + 1, r))}

    def probe(engine, t, stage):
        if stage != "after_inner" or t not in k_of:
            return
        anchor = engine.outer.snapshot
        k = k_of[t]
        for w in engine.workers:
            rng = np.random.default_rng([seed, 300, k, w.group])
            w.params = anchor + anchor.dtype.type(1e-3) * rng.standard_normal(
                anchor.shape[0], dtype=anchor.dtype)

    eng = _Engine(cfg, probe=probe)
    theta0 = eng.outer.snapshot.copy()
    res = eng.run()
    tag = f"open_loop_T{T}_r{r}_g{groups}" + (f"_dp{dp}" if dp > 1 else "")
    np.savez_compressed(HERE / f"{tag}.npz", theta0=theta0,
                        anchor=res.final_params, momentum=res.outer_momentum,
                        folds=np.array(res.warmup_folds), outer=np.array(res.comm.outer_events))


def tiny_gpt():
    """BASELINE.json config 1 on the reference (fp32): the closed-loop oracle."""
    cfg = load_config(mode="pier", groups=2, sync_interval=8, total_iters=160,
                      precision="single", lazy_fraction=0.1)
    from pier import data as D
    from pier.model import init_params

    eng = _Engine(cfg)
    batches = np.stack([
        D.sample_global_batch(eng.train_corpus, cfg.seed, t, cfg.global_batch, cfg.seq_len)
        for t in range(1, cfg.total_iters + 1)])
    res = eng.run()
    res.write(HERE / "tiny_gpt_artifacts")   # the reference's trajectory.jsonl / params.bin / summary.json
    recs = [r.to_dict() for r in res.records]
    theta0 = init_params(cfg.model_config(), np.random.default_rng([cfg.seed, 100]))
    np.savez_compressed(
        HERE / "tiny_gpt.npz",
        theta0=theta0, batches=batches.astype(np.uint8),
        val=np.stack(eng.val_batches).astype(np.uint8),
        train_loss=np.array([r["train_loss"] if r["train_loss"] is not None else np.nan for r in recs]),
        val_loss=np.array([r["val_loss"] if r["val_loss"] is not None else np.nan for r in recs]),
        iters=np.array([r["iter"] for r in recs]),
        final_params=res.final_params, momentum=res.outer_momentum,
        warmup_folds=np.array(res.warmup_folds))


if __name__ == "__main__":
    what = sys.argv[1:] or ["kernels", "schedules", "traces", "open_loop", "tiny_gpt"]
    print("reference pier", pier.__version__, "numpy", np.__version__)
    if "kernels" in what:
        kernels()
    if "schedules" in what:
        schedules()
    if "traces" in what:
        traces()
    if "open_loop" in what:
        for T, r, g in ((200, 10, 1), (200, 10, 2), (200, 10, 3), (1000, 10, 2), (1000, 10, 8),
                        (200, 10, 4), (200, 10, 8)):
            open_loop(T, r, g)
        open_loop(200, 10, 2, dp=2)
    if "open_loop_dp" in what:
        open_loop(200, 10, 2, dp=2)
    if "tiny_gpt" in what:
        tiny_gpt()
    print("done")
