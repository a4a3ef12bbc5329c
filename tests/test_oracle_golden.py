"""Pin the CPU oracle against the reference's own outputs (CPU only).

The fixtures were produced by the unmodified reference (tests/golden/make_golden.py);
the oracle must reproduce them bit for bit -- except the BLAS dot in the clip
norm, whose summation order is implementation-defined (reference
``optim.py:76``), which is pinned within 2 ulp.
"""

import json
import os

import numpy as np
import pytest

from oracle import pier_oracle as O

from conftest import GOLDEN

K = np.load(os.path.join(GOLDEN, "kernels.npz"))
TAGS = ("float32", "float64")
MU_LR = ((0.99, 0.205), (0.9, 1.1), (0.9, 0.9), (0.0, 1.0), (0.95, 0.5))


@pytest.mark.parametrize("tag", TAGS)
def test_adamw_chain_bitwise(tag):
    th, m, v = K[f"adamw_{tag}_theta0"], K[f"adamw_{tag}_m0"], K[f"adamw_{tag}_v0"]
    step = 10
    for k, lr in enumerate(K[f"adamw_{tag}_lrs"]):
        th, m, v, step = O.adamw(th, K[f"adamw_{tag}_g{k}"], m, v, step, float(lr))
        assert np.array_equal(th, K[f"adamw_{tag}_theta{k + 1}"])
        assert np.array_equal(m, K[f"adamw_{tag}_m{k + 1}"])
        assert np.array_equal(v, K[f"adamw_{tag}_v{k + 1}"])
        assert th.dtype == np.dtype(tag)
    assert step == int(K[f"adamw_{tag}_step_final"])


@pytest.mark.parametrize("tag", TAGS)
def test_clip(tag):
    g = K[f"clip_{tag}_long"]
    out, nrm = O.clip_global_norm(g, 1.0)
    ref_n = float(K[f"clip_{tag}_long_norm"])
    assert abs(nrm - ref_n) <= 2 * np.spacing(np.dtype(tag).type(ref_n))
    np.testing.assert_allclose(out, K[f"clip_{tag}_long_out"], rtol=4 * np.finfo(tag).eps)
    gs = K[f"clip_{tag}_short"]
    o2, n2 = O.clip_global_norm(gs, 1.0)
    assert o2 is gs
    assert n2 == pytest.approx(float(K[f"clip_{tag}_short_norm"]), rel=4 * np.finfo(tag).eps)


@pytest.mark.parametrize("tag", TAGS)
def test_mean_left_fold_bitwise(tag):
    ths = [K[f"outer_{tag}_theta{i}"] for i in range(8)]
    for n in range(1, 9):
        assert np.array_equal(O.mean_left_fold(ths[:n]), K[f"mean_{tag}_n{n}"])


@pytest.mark.parametrize("tag", TAGS)
@pytest.mark.parametrize("mu,lr", MU_LR)
def test_outer_and_fold_bitwise(tag, mu, lr):
    anchor, mom = K[f"outer_{tag}_anchor"], K[f"outer_{tag}_mom"]
    ths = [K[f"outer_{tag}_theta{i}"] for i in range(8)]
    key = f"{mu}_{lr}"
    for n in (1, 2, 3, 4, 8):
        avg = O.mean_left_fold(ths[:n])
        th, M = O.outer_anchor_form(avg, anchor, mom, lr, mu)
        assert np.array_equal(th, K[f"outer_{tag}_{key}_n{n}_theta"])
        assert np.array_equal(M, K[f"outer_{tag}_{key}_n{n}_mom"])
    th, M = O.outer_snapshot_form(anchor, mom, ths[0] - anchor, lr, mu)
    assert np.array_equal(th, K[f"outer_{tag}_{key}_snapform_theta"])
    assert np.array_equal(M, K[f"outer_{tag}_{key}_snapform_mom"])
    assert np.array_equal(O.fold(mom, ths[0] - anchor, mu), K[f"fold_{tag}_{key}"])
    # the warmup-fold form used by the driver (driver.py:415-420)
    M2, a2 = O.warmup_fold(ths[0], anchor, mom, mu)
    assert np.array_equal(M2, K[f"fold_{tag}_{key}"])
    assert np.array_equal(a2, ths[0])


def test_schedules_exact():
    tab = json.load(open(os.path.join(GOLDEN, "schedules.json")))
    for T, entry in tab.items():
        T = int(T)
        s = O.Sched(total_iters=T, sync_interval=min(20, T - 1))
        assert s.lazy_end == entry["lazy_end"]
        assert s.warmup_iters == entry["warmup_iters"]
        for t, ilr, olr, mu in entry["rows"]:
            assert O.inner_lr(t, s) == ilr
            assert O.momentum_mu(t, T) == mu
            if olr is None:
                with pytest.raises(ValueError):
                    O.outer_lr(t, s)
            else:
                assert O.outer_lr(t, s) == olr


def test_boundary_traces_exact():
    """Fold/outer iterations and every (mu, lr) pair equal the reference driver's."""
    for case in json.load(open(os.path.join(GOLDEN, "traces.json"))):
        c = case["case"]
        s = O.Sched(total_iters=c["total_iters"], lazy_fraction=c["lazy_fraction"],
                    sync_interval=c["sync_interval"])
        evs = {e.t: e for e in O.boundary_events(s, c["mode"], lr_fixed=c.get("outer_lr_fixed"))}
        assert s.lazy_end == case["lazy_end"]
        folds = 0
        outers = 0
        for rec in case["records"][1:]:
            t = rec["iter"]
            e = evs.get(t)
            if e is None:
                assert rec["mu"] is None and rec["outer_lr"] is None
                continue
            if e.kind == "outer":
                outers += 1
                assert rec["outer_lr"] == e.lr and rec["mu"] == e.mu, (c, t)
            else:
                folds += e.kind == "fold"
                assert rec["outer_lr"] is None and rec["mu"] == e.mu, (c, t)
            assert rec["phase"] == ("lazy_start" if t <= s.lazy_end
                                    else ("pier" if c["mode"] == "pier" else "diloco"))
        assert folds == case["warmup_folds"]
        assert outers == case["outer_events"]
        P = case["param_count"]
        assert case["outer_bytes"] == pytest.approx(
            outers * O.ring_bytes(P * 4.0, c["groups"]), rel=1e-12)


def test_offload_counters_match_reference_trace():
    case = [c for c in json.load(open(os.path.join(GOLDEN, "traces.json")))
            if c["case"].get("offload_enabled")][0]
    P = case["param_count"]
    world = case["case"]["groups"]
    led = O.HostLedger(enabled=True)
    snap = np.zeros(P, np.float32)
    mom = np.zeros(P, np.float32)

    def park():
        for r, (a, b) in enumerate(O.shard_ranges(P, world)):
            led.store(("snapshot", r), snap[a:b])
            led.store(("momentum", r), mom[a:b])

    def fetch():
        for r in range(world):
            led.load(("snapshot", r))
        for r in range(world):
            led.load(("momentum", r))

    park()  # driver.py:308-309
    s = O.Sched(total_iters=case["case"]["total_iters"], lazy_fraction=case["case"]["lazy_fraction"],
                sync_interval=case["case"]["sync_interval"])
    for _ in O.boundary_events(s, "pier"):
        fetch()
        park()
    off = case["offload"]
    assert led.to_host == off["to_host_bytes"]
    assert led.from_host == off["from_host_bytes"]
    assert led.stores == off["store_events"]
    assert led.loads == off["load_events"]
    with pytest.raises(O.ProtocolViolation):
        led.store(("snapshot", 0), snap)


@pytest.mark.parametrize("T,g", [(200, 1), (200, 2), (200, 3), (200, 4), (200, 8), (1000, 2), (1000, 8)])
def test_open_loop_bitwise(T, g):
    f = np.load(os.path.join(GOLDEN, f"open_loop_T{T}_r10_g{g}.npz"))
    s = O.Sched(total_iters=T, lazy_fraction=0.1, sync_interval=10)
    anchor, M, evs = O.open_loop_run(s, f["theta0"], g, seed=0)
    assert sum(e.kind == "fold" for e in evs) == int(f["folds"])
    assert sum(e.kind == "outer" for e in evs) == int(f["outer"])
    assert np.array_equal(anchor, f["anchor"])
    assert np.array_equal(M, f["momentum"])


def test_open_loop_dp2_bitwise():
    """groups=2 x dp_per_group=2: the outer mean folds all 4 replicas (driver.py:428)."""
    f = np.load(os.path.join(GOLDEN, "open_loop_T200_r10_g2_dp2.npz"))
    s = O.Sched(total_iters=200, lazy_fraction=0.1, sync_interval=10)
    anchor, M, _ = O.open_loop_run(s, f["theta0"], 2, seed=0, dp=2)
    assert np.array_equal(anchor, f["anchor"]) and np.array_equal(M, f["momentum"])


def test_shard_ranges_and_ring_bytes():
    assert O.shard_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert O.ring_bytes(100.0, 4) == 150.0
    assert O.ring_bytes(100.0, 1) == 0.0


def test_chunked_equals_unchunked():
    rng = np.random.default_rng(0)
    a = rng.standard_normal(10007).astype(np.float32)
    b = rng.standard_normal(10007).astype(np.float32)
    c = rng.standard_normal(10007).astype(np.float32)
    want = O.outer_anchor_form(a, b, c, 0.9, 0.99)
    got = O.chunked(lambda x, y, z: O.outer_anchor_form(x, y, z, 0.9, 0.99), [a, b, c], 4, 1000)
    assert all(np.array_equal(w, g) for w, g in zip(want, got))


def test_hash_inputs_torch_equals_numpy_and_subset_runs_are_exact():
    """The counter-based open-loop inputs (oracle.hash_values) computed with torch
    int64 ops (what the GPU test runs) equal NumPy's uint64 ones bit for bit, and
    an open-loop run over a subset of elements equals that subset of the full
    run (the boundary stage is elementwise) -- the basis of the full-size
    sampled parity test (tests/test_open_loop_sizes_gpu.py)."""
    from group_checks import torch_hash_values

    n = 200_003
    for key in (O.hash_key(4, -1, 0), O.hash_key(4, 57, 7), O.hash_key(99, 3, 1)):
        t = torch_hash_values(key, n, O.NOISE_SCALE, "cpu", chunk=1 << 16).numpy()
        c = O.hash_values(key, np.arange(n), O.NOISE_SCALE)
        assert np.array_equal(t.view(np.uint32), c.view(np.uint32))
    s = O.Sched(total_iters=200, lazy_fraction=0.1, sync_interval=10)
    idx = np.arange(n)
    theta0 = O.hash_values(O.hash_key(4, -1, 0), idx, O.THETA0_SCALE)
    full = O.open_loop_run(s, theta0, 3, 4, inputs=lambda sd, k, g, a: O.hash_inputs(sd, k, g, a, idx))
    sub = idx[::37]
    part = O.open_loop_run(s, theta0[sub], 3, 4, inputs=lambda sd, k, g, a: O.hash_inputs(sd, k, g, a, sub))
    assert np.array_equal(full[0][sub], part[0]) and np.array_equal(full[1][sub], part[1])
