"""BASELINE config 1, closed loop: tiny GPT (2 layers, d=128), 2 groups x 8
inner AdamW steps, lazy start -> momentum warmup -> decay, T=160, fp32.

`paper_2511_17849_b200.desk.run_desk` computes the gradients on the GPU
(`tinygpt`, the reference desk model in torch) and runs every optimizer
operation -- lazy-phase gradient mean (K6), clip + AdamW (K4a/K4b), warmup
folds (K3b), the mean of the groups (K6) and the outer step (K3) -- on this
repo's kernels.  Against the reference's own run (tests/golden/tiny_gpt.npz and
its artifacts): loss curve within 1e-4 (BASELINE.json north_star), phase
schedule and comm accounting exact, artifacts in the same byte formats."""

import json
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


def test_tiny_gpt_closed_loop_loss_curve_and_artifacts(tmp_path):
    from paper_2511_17849_b200 import artifacts
    from paper_2511_17849_b200.desk import DeskConfig, run_desk

    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    f = np.load(os.path.join(GOLDEN, "tiny_gpt.npz"))
    cfg = DeskConfig(groups=2, sync_interval=8, total_iters=160, lazy_fraction=0.1)
    batches = f["batches"].astype(np.int64)
    per = batches.shape[1] // cfg.groups
    res = run_desk(cfg, lambda t, g: batches[t - 1, g * per:(g + 1) * per], list(f["val"].astype(np.int64)))

    train = np.array([r["train_loss"] for r in res.records[1:]])
    err = float(np.max(np.abs(train - f["train_loss"][1:])))
    assert err <= 1e-4, f"train-loss curve max |diff| {err:.3e}"
    ref_val = f["val_loss"]
    verr = max(abs(r["val_loss"] - ref_val[i]) for i, r in enumerate(res.records) if r["val_loss"] is not None)
    assert verr <= 1e-4, f"val-loss max |diff| {verr:.3e}"
    assert res.warmup_folds == int(f["warmup_folds"]) == 2
    rel = float(np.linalg.norm(res.final_params.cpu().numpy() - f["final_params"]) / np.linalg.norm(f["final_params"]))
    assert rel <= 1e-3, rel   # closed loop amplifies ulp noise: loose bound on params
    print(f"tiny-GPT closed loop: train-loss max diff {err:.2e}, val max diff {verr:.2e}, params l2-rel {rel:.2e}")

    # artifacts: same files, same record structure, schedule/comm fields exact, same params.bin format
    res.write(tmp_path)
    ref_dir = os.path.join(GOLDEN, "tiny_gpt_artifacts")
    ours = [json.loads(x) for x in open(tmp_path / "trajectory.jsonl")]
    refs = [json.loads(x) for x in open(os.path.join(ref_dir, "trajectory.jsonl"))]
    assert len(ours) == len(refs)
    for a, b in zip(ours[1:], refs[1:]):
        assert list(a) == list(b)
        for k in ("record", "iter", "phase", "inner_lr", "outer_lr", "mu", "comm_bytes"):
            assert a[k] == b[k], (k, a, b)
    theta_ref = artifacts.read_params(os.path.join(ref_dir, "params.bin"))
    theta_ours = artifacts.read_params(tmp_path / "params.bin")
    assert theta_ours.dtype == theta_ref.dtype and theta_ours.shape == theta_ref.shape
    raw_ref = open(os.path.join(ref_dir, "params.bin"), "rb").read(20)
    assert open(tmp_path / "params.bin", "rb").read(20) == raw_ref   # identical header bytes
    s_ours = json.load(open(tmp_path / "summary.json"))
    s_ref = json.load(open(os.path.join(ref_dir, "summary.json")))
    assert s_ours["comm"] == s_ref["comm"] and s_ours["warmup_folds"] == s_ref["warmup_folds"]


def test_divergence_raises_numeric_error_with_iteration():
    """test_driver.py:370-380: a diverging run raises NumericError carrying the
    iteration (driver.py:364-368); the engine's own guard reports a non-finite
    gradient norm the same way."""
    from paper_2511_17849_b200.desk import DeskConfig, run_desk

    f = np.load(os.path.join(GOLDEN, "tiny_gpt.npz"))
    cfg = DeskConfig(groups=2, sync_interval=8, total_iters=160, lazy_fraction=0.1, inner_lr_peak=1e200,
                     clip_norm=1e300, weight_decay=0.0)
    batches = f["batches"].astype(np.int64)
    per = batches.shape[1] // cfg.groups
    with pytest.raises(P.NumericError) as exc:
        run_desk(cfg, lambda t, g: batches[t - 1, g * per:(g + 1) * per], list(f["val"].astype(np.int64)))
    assert exc.value.iteration is not None and str(exc.value.iteration) in str(exc.value)

    eng = P.PierEngine(4099, P.ScheduleConfig(total_iters=100, sync_interval=10), check_finite=True)
    eng.grad[7] = float("nan")
    eng.inner_step(10)
    with pytest.raises(P.NumericError) as exc:
        eng.boundary(10)
    assert exc.value.iteration == 10
