"""Closed-loop desk runs on one GPU: the reference's
``run_training`` for its tiny transformer (driver.py:465-474, 531-573) with the
gradients computed on the GPU (``tinygpt``) and every optimizer operation on
this package's kernels; G groups live on the one GPU as virtual groups
(left-fold means by K6), exactly the reference's sequential worker order.
Writes the reference's artifacts (trajectory.jsonl, params.bin, summary.json).
"""

from __future__ import annotations

import math
from dataclasses import asdict, dataclass, field
from pathlib import Path

import numpy as np
import torch

from . import _dev, artifacts, tinygpt
from .engine import PierSchedule
from .errors import NumericError
from .optim import (AdamWConfig, ScheduleConfig, adamw_, grad_sqnorm_, inner_lr, norm_workspace, outer_update_,
                    warmup_fold_)
from .topology import allreduce_avg, ring_allreduce_bytes

FORMAT_VERSION = 1  # driver.py:71


@dataclass
class DeskConfig:
    """The hot-path and model fields of the reference's RunConfig (config.py:32-85)."""

    mode: str = "pier"
    seed: int = 0
    vocab_size: int = 256
    embed_dim: int = 128
    num_layers: int = 2
    num_heads: int = 4
    seq_len: int = 64
    total_iters: int = 3000
    lazy_fraction: float = 0.1
    sync_interval: int = 20
    inner_warmup_fraction: float = 0.02
    inner_lr_peak: float = 3e-3
    inner_lr_min: float = 3e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.1
    clip_norm: float = 1.0
    groups: int = 4
    outer_lr_fixed: float | None = None
    outer_mu_fixed: float | None = None

    def model(self) -> dict:
        return dict(vocab=self.vocab_size, d=self.embed_dim, heads=self.num_heads, layers=self.num_layers,
                    seq=self.seq_len)


@dataclass
class DeskResult:
    config: dict
    records: list = field(default_factory=list)
    final_params: torch.Tensor | None = None
    outer_momentum: torch.Tensor | None = None
    warmup_folds: int = 0
    comm: dict = field(default_factory=dict)

    def write(self, out_dir) -> None:
        out = Path(out_dir)
        out.mkdir(parents=True, exist_ok=True)
        header = {"record": "header", "format_version": FORMAT_VERSION, "mode": self.config["mode"],
                  "seed": self.config["seed"], "world_size": self.config["groups"],
                  "topology": {"groups": self.config["groups"], "dp_per_group": 1, "tp_size": 1},
                  "config": self.config}
        artifacts.write_jsonl(out / artifacts.TRAJECTORY_NAME, [header] + self.records)
        artifacts.write_params(out / artifacts.PARAMS_NAME, self.final_params)
        last_train = next((r["train_loss"] for r in reversed(self.records) if r["train_loss"] is not None), None)
        last_val = next((r["val_loss"] for r in reversed(self.records) if r["val_loss"] is not None), None)
        artifacts.write_json(out / artifacts.SUMMARY_NAME, {
            "record": "summary", "format_version": FORMAT_VERSION, "mode": self.config["mode"],
            "seed": self.config["seed"], "iters": self.config["total_iters"],
            "param_count": int(self.final_params.numel()), "final_train_loss": last_train,
            "final_val_loss": last_val, "comm": self.comm, "warmup_folds": self.warmup_folds,
            "config": self.config})


class _WorkerView:
    """One replica as a probe sees it (the reference's ``_Worker``: ``params``, ``opt``)."""

    def __init__(self, g, th, m, v, step):
        self.replica, self._th, self._m, self._v, self._step = g, th, m, v, step

    @property
    def params(self):
        return self._th.cpu().numpy()

    @property
    def opt(self):
        from .optim import AdamWState
        return AdamWState(m=self._m.cpu().numpy(), v=self._v.cpu().numpy(), step=self._step())


class _OuterView:
    def __init__(self, anchor, mom, mu):
        self._a, self._m, self.mu = anchor, mom, mu

    @property
    def snapshot(self):
        return self._a.cpu().numpy()

    @property
    def momentum(self):
        return self._m.cpu().numpy()


class DeskView:
    """What ``probe(engine, t, stage)`` receives -- the attributes reference
    probes read from its ``_Engine`` (test_driver.py:154-156, 252-266):
    ``workers[i].params`` / ``.opt``, ``outer.snapshot`` / ``.momentum``
    (None for the synchronous baseline), ``records``, ``warmup_folds``.
    Arrays are host copies (the reference hands out its NumPy arrays)."""

    def __init__(self, workers, outer, res):
        self.workers, self.outer, self._res = workers, outer, res

    @property
    def records(self):
        return self._res.records

    @property
    def warmup_folds(self):
        return self._res.warmup_folds


def run_desk(cfg: DeskConfig, batch_source, val_batches, theta0=None, device=None, probe=None,
             stop_after: int | None = None) -> DeskResult:
    """``batch_source(t, group) -> (rows, seq_len+1)`` int tokens; ``val_batches``:
    list of (rows, seq_len+1) arrays.  fp32 ("single" precision) throughout.
    ``probe(view, t, stage)`` runs after the inner stages ("after_inner") and
    after the boundary stage ("after_boundary") of every iteration, like the
    reference's (driver.py:472-473, 460-461); ``stop_after`` ends the run early
    (driver.py:531-573)."""
    dev = device or _dev.require_cuda()
    mcfg = cfg.model()
    sched = ScheduleConfig(total_iters=cfg.total_iters, lazy_fraction=cfg.lazy_fraction,
                           sync_interval=cfg.sync_interval, inner_warmup_fraction=cfg.inner_warmup_fraction,
                           inner_lr_peak=cfg.inner_lr_peak, inner_lr_min=cfg.inner_lr_min)
    plan = PierSchedule(sched, cfg.mode, cfg.outer_lr_fixed, cfg.outer_mu_fixed)
    acfg = AdamWConfig(beta1=cfg.beta1, beta2=cfg.beta2, eps=cfg.eps, weight_decay=cfg.weight_decay,
                       clip_norm=cfg.clip_norm)
    if theta0 is None:   # driver.py:264
        theta0 = tinygpt.init_params(mcfg["vocab"], mcfg["d"], mcfg["layers"], mcfg["seq"],
                                     np.random.default_rng([cfg.seed, 100]))
    th0 = torch.as_tensor(np.asarray(theta0, dtype=np.float32)).to(dev)
    n, G = th0.numel(), cfg.groups
    th = [th0.clone() for _ in range(G)]
    m = [torch.zeros(n, device=dev) for _ in range(G)]
    v = [torch.zeros(n, device=dev) for _ in range(G)]
    grads = [torch.zeros(n, device=dev) for _ in range(G)]
    ws = [norm_workspace(dev) for _ in range(G)]
    synchronous = plan.synchronous
    anchor = None if synchronous else th0.clone()
    mom = None if synchronous else torch.zeros(n, device=dev)
    vals = [torch.as_tensor(np.asarray(b, dtype=np.int64)).to(dev) for b in val_batches]
    payload = float(n * 4)
    res = DeskResult(config=asdict(cfg))
    inner_b = outer_b = 0.0
    inner_ev = outer_ev = 0

    def evaluate(theta):  # driver.py:580-585
        with torch.no_grad():
            return float(sum(float(tinygpt.loss_fn(theta, b, mcfg).item()) for b in vals) / len(vals))

    res.records.append({"record": "iter", "iter": 0, "phase": plan.phase(0), "train_loss": None,
                        "val_loss": evaluate(th[0]), "inner_lr": inner_lr(0, sched), "outer_lr": None,
                        "mu": None, "comm_bytes": 0.0})
    step_of = {"t": 0}
    view = DeskView([_WorkerView(g, th[g], m[g], v[g], lambda: step_of["t"]) for g in range(G)],
                    None if synchronous else _OuterView(anchor, mom, 0.9), res)
    last = cfg.total_iters if stop_after is None else min(stop_after, cfg.total_iters)
    for t in range(1, last + 1):
        step_of["t"] = t
        losses = [tinygpt.loss_and_grad(th[g], torch.as_tensor(np.asarray(batch_source(t, g), dtype=np.int64)).to(dev),
                                        mcfg, grads[g]) for g in range(G)]
        if not all(np.isfinite(losses)):                        # driver.py:364-368
            raise NumericError(f"non-finite training loss ({losses}) at iteration {t}", iteration=t)
        comm_t = 0.0
        if G > 1 and plan.syncs_gradients(t):                  # driver.py:380-393
            mean = allreduce_avg(grads)
            for g in range(G):
                grads[g].copy_(mean)
            comm_t += ring_allreduce_bytes(payload, G)
            inner_b += comm_t
            inner_ev += 1
        lr = inner_lr(t, sched)
        for g in range(G):                                     # driver.py:395-399
            grad_sqnorm_(grads[g], acfg.clip_norm, ws[g])
            adamw_(th[g], grads[g], m[g], v[g], t, lr, acfg, ws[g])
        if probe is not None:
            probe(view, t, "after_inner")
        ev = plan.event(t)                                     # driver.py:404-443
        rec_lr = rec_mu = None
        if ev is not None and ev.kind == "fold":
            warmup_fold_(th[0], anchor, mom, ev.mu)
            res.warmup_folds += 1
            rec_mu = ev.mu
        elif ev is not None and ev.kind == "anchor":
            anchor.copy_(th[0])
        elif ev is not None:
            avg = allreduce_avg(th)
            outer_update_(avg, anchor, mom, ev.outer_lr, ev.mu)
            for g in range(G):
                th[g].copy_(avg)
            ob = ring_allreduce_bytes(payload, G)
            comm_t += ob
            outer_b += ob
            outer_ev += 1
            rec_lr, rec_mu = ev.outer_lr, ev.mu
        val = evaluate(th[0]) if (t % cfg.sync_interval == 0 or t == cfg.total_iters) else None
        res.records.append({"record": "iter", "iter": t, "phase": plan.phase(t),
                            "train_loss": float(sum(losses) / len(losses)), "val_loss": val,
                            "inner_lr": lr, "outer_lr": rec_lr, "mu": rec_mu, "comm_bytes": comm_t})
        if probe is not None:
            probe(view, t, "after_boundary")
    res.final_params = th[0]
    res.outer_momentum = mom
    res.comm = {"inner_bytes": inner_b, "outer_bytes": outer_b, "total_bytes": inner_b + outer_b,
                "inner_events": inner_ev, "outer_events": outer_ev}
    return res


# ---------------------------------------------------------------------------
# the reference's entry points (driver.py:588-621) over run_desk
# ---------------------------------------------------------------------------

def _desk_config(cfg) -> DeskConfig:
    """A DeskConfig from a DeskConfig or any object with the reference RunConfig's
    field names (config.py:32-85; unknown fields are ignored)."""
    if isinstance(cfg, DeskConfig):
        return cfg
    from dataclasses import fields
    kw = {f.name: getattr(cfg, f.name) for f in fields(DeskConfig) if hasattr(cfg, f.name)}
    if getattr(cfg, "dp_per_group", 1) != 1 or getattr(cfg, "tp_size", 1) != 1:
        from .errors import ConfigError
        raise ConfigError("the desk runs one replica per group; dp/tp layouts run on PierEngine "
                          "(one rank per replica shard, or a VirtualGroup on one GPU)")
    return DeskConfig(**kw)


def run_training(cfg, *, batch_source, val_batches=(), probe=None, theta0=None) -> DeskResult:
    """``driver.py:588-590``: run ``cfg.mode`` to completion.  ``batch_source(t,
    group, dp)`` as in the reference (the reference's synthetic corpus is its data
    pipeline, out of scope here, so the batches are the caller's)."""
    dcfg = _desk_config(cfg)
    vals = list(val_batches) or [batch_source(0, 0, 0)]
    return run_desk(dcfg, lambda t, g: batch_source(t, g, 0), vals, theta0=theta0, probe=probe)


def run_pier(cfg, **kwargs) -> DeskResult:                 # driver.py:593-594
    from dataclasses import replace
    return run_training(replace(_desk_config(cfg), mode="pier"), **kwargs)


def run_adamw_baseline(cfg, **kwargs) -> DeskResult:       # driver.py:597-598
    from dataclasses import replace
    return run_training(replace(_desk_config(cfg), mode="adamw_baseline"), **kwargs)


def run_diloco_baseline(cfg, **kwargs) -> DeskResult:      # driver.py:601-602
    from dataclasses import replace
    return run_training(replace(_desk_config(cfg), mode="diloco_baseline"), **kwargs)


def momentum_warmup_phase(cfg, *, batch_source, val_batches=(), probe=None, theta0=None):
    """``driver.py:605-621``: only the lazy-start phase of a Pier run.  Returns
    ``(theta, momentum, optimizer_states, records)`` at the phase boundary (host
    arrays, like the reference's)."""
    from dataclasses import replace
    dcfg = replace(_desk_config(cfg), mode="pier")
    lazy_end = int(math.floor(dcfg.lazy_fraction * dcfg.total_iters))
    captured = {}

    def grab(view, t, stage):
        if probe is not None:
            probe(view, t, stage)
        if t == lazy_end and stage == "after_boundary":
            captured["opt"] = [w.opt for w in view.workers]
            captured["theta"] = view.workers[0].params
            captured["momentum"] = view.outer.momentum

    vals = list(val_batches) or [batch_source(0, 0, 0)]
    res = run_desk(dcfg, lambda t, g: batch_source(t, g, 0), vals, theta0=theta0, probe=grab, stop_after=lazy_end)
    if not captured:          # no lazy phase (lazy_end = 0): the initial state
        from .optim import AdamWState
        n = res.final_params.numel()
        zeros = np.zeros(n, np.float32)
        return (res.final_params.cpu().numpy(), res.outer_momentum.cpu().numpy(),
                [AdamWState(m=zeros.copy(), v=zeros.copy(), step=0) for _ in range(dcfg.groups)], res.records)
    return captured["theta"], captured["momentum"], captured["opt"], res.records
