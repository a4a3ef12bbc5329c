"""The reference's driver entry points over the GPU desk run (driver.py:588-621):
``run_training(cfg, batch_source=, probe=)``, ``run_pier`` /
``run_adamw_baseline`` / ``run_diloco_baseline`` and ``momentum_warmup_phase``,
with the probe hook the reference's tests use (test_driver.py:149-162,
:261-276).  Batches come from the golden tiny-GPT fixture (the reference's
synthetic corpus is its data pipeline, out of scope)."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2511_17849_b200")


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _source():
    f = np.load(os.path.join(GOLDEN, "tiny_gpt.npz"))
    batches = f["batches"].astype(np.int64)
    per = batches.shape[1] // 2
    return (lambda t, g, dp: batches[max(t, 1) - 1, g * per:(g + 1) * per]), list(f["val"].astype(np.int64))


def test_warmup_two_interval_hand_formula():
    """test_driver.py:149-162: two folds with mu 0.9 -> M = 0.9*d1 + d2 (fp32, one
    rounding per op: bitwise)."""
    from paper_2511_17849_b200.desk import DeskConfig, momentum_warmup_phase

    src, val = _source()
    cfg = DeskConfig(groups=2, total_iters=40, lazy_fraction=0.5, sync_interval=10)
    snaps = {}

    def probe(view, t, stage):
        if t == 1 and stage == "after_inner":
            snaps[0] = view.outer.snapshot                   # theta0 (no boundary yet)
        if stage == "after_boundary" and t in (10, 20):
            snaps[t] = view.workers[0].params

    theta, momentum, opts, records = momentum_warmup_phase(cfg, batch_source=src, val_batches=val, probe=probe)
    f32 = np.float32
    d1, d2 = snaps[10] - snaps[0], snaps[20] - snaps[10]
    want = f32(0.9) * d1 + d2
    assert np.array_equal(momentum.view(np.uint32), want.view(np.uint32))
    assert np.array_equal(theta, snaps[20]) and records[-1]["iter"] == 20
    assert len(opts) == 2 and all(o.step == 20 for o in opts)


def test_no_lazy_phase_returns_initial_state():
    """test_driver.py:138-146: lazy_fraction 0 -> zero momentum, theta0."""
    from paper_2511_17849_b200.desk import DeskConfig, momentum_warmup_phase

    src, val = _source()
    cfg = DeskConfig(groups=2, total_iters=40, lazy_fraction=0.0, sync_interval=20, outer_lr_fixed=1.0)
    seen = {}
    theta, momentum, _, records = momentum_warmup_phase(
        cfg, batch_source=src, val_batches=val, probe=lambda v, t, s: seen.setdefault("called", True))
    assert np.all(momentum == 0.0) and records[-1]["iter"] == 0 and not seen
    from paper_2511_17849_b200 import tinygpt
    theta0 = tinygpt.init_params(256, 128, 2, 64, np.random.default_rng([0, 100]))
    assert np.array_equal(theta, np.asarray(theta0, dtype=np.float32))


def test_snapshot_frozen_between_boundaries_and_probe_order():
    """test_driver.py:261-276 (values): the anchor changes exactly at boundary
    iterations; the probe sees after_inner then after_boundary for every t."""
    from paper_2511_17849_b200.desk import DeskConfig, run_training

    src, val = _source()
    cfg = DeskConfig(groups=2, total_iters=60, lazy_fraction=0.5, sync_interval=10)
    by_iter, stages = {}, []

    def probe(view, t, stage):
        stages.append((t, stage))
        if stage == "after_inner":
            by_iter[t] = view.outer.snapshot

    res = run_training(cfg, batch_source=src, val_batches=val, probe=probe)
    assert stages == [(t, s) for t in range(1, 61) for s in ("after_inner", "after_boundary")]
    for t in range(2, 61):
        changed = not np.array_equal(by_iter[t], by_iter[t - 1])
        assert changed == ((t - 1) % 10 == 0), t
    assert [r["iter"] for r in res.records] == list(range(0, 61))


def test_baseline_entry_points():
    """run_adamw_baseline has no outer state and no folds; run_diloco_baseline
    re-anchors without folding and steps with the fixed 0.7 / 0.9 (config.py:28-29)."""
    from paper_2511_17849_b200.desk import DeskConfig, run_adamw_baseline, run_diloco_baseline

    src, val = _source()
    cfg = DeskConfig(groups=2, total_iters=40, lazy_fraction=0.5, sync_interval=10)
    outs = []
    res = run_adamw_baseline(cfg, batch_source=src, val_batches=val,
                             probe=lambda v, t, s: outs.append(v.outer is None))
    assert all(outs) and res.warmup_folds == 0 and res.outer_momentum is None
    res = run_diloco_baseline(cfg, batch_source=src, val_batches=val)
    assert res.warmup_folds == 0
    outer = [(r["iter"], r["outer_lr"], r["mu"]) for r in res.records if r["outer_lr"] is not None]
    assert outer == [(30, 0.7, 0.9), (40, 0.7, 0.9)]
