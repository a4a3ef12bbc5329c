"""CPU-only checks of the product's host logic and of the C-ABI library
(loads, exports every declared symbol, exact host schedule) -- no GPU work."""

import ctypes as C
import json
import os
import re

import numpy as np
import pytest

import paper_2511_17849_b200 as P
from paper_2511_17849_b200 import _lib
from paper_2511_17849_b200.engine import PierSchedule, bucket_layout, validate_run

from conftest import GOLDEN, ROOT

HEADER = os.path.join(ROOT, "include", "pier_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pier_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported_and_bound():
    syms = declared_symbols()
    assert len(syms) > 40
    lib = C.CDLL(_lib.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/pier_b200.h but not exported"
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_mapping_without_gpu():
    # argument validation happens before any CUDA call
    assert _lib.lib.pier_pseudograd_f32(None, None, None, 10, None) == _lib.PIER_EINVAL
    with pytest.raises(P.ConfigError):
        _lib.check(_lib.lib.pier_pseudograd_f32(None, None, None, 10, None), "x")
    assert "pseudograd" in _lib.last_error()
    assert _lib.lib.pier_mean_left_fold_f32(None, 0, None, 4, None) == _lib.PIER_EINVAL
    out = C.c_double()
    assert _lib.lib.pier_outer_lr(10, 3000, C.byref(out)) == _lib.PIER_EINVAL
    # the persistent rounds reject a missing communicator / gradient before touching the device
    hp = _lib.PierAdamW(1e-3, 0.9, 0.999, 1e-8, 0.1, 1)
    for fn in (_lib.lib.pier_round_fused_f32, _lib.lib.pier_round_fused_bf16_f32):
        assert fn(None, 0, None, None, None, None, None, 64, 8, C.byref(hp), None, 1.0, 0.9, None) == _lib.PIER_EINVAL
        assert "round_fused" in _lib.last_error()


def test_schedules_match_reference_tables():
    tab = json.load(open(os.path.join(GOLDEN, "schedules.json")))
    for T, entry in tab.items():
        T = int(T)
        s = P.ScheduleConfig(total_iters=T, sync_interval=min(20, T - 1))
        assert s.lazy_end == entry["lazy_end"] and s.warmup_iters == entry["warmup_iters"]
        for t, ilr, olr, mu in entry["rows"]:
            assert P.inner_lr(t, s) == ilr
            assert P.momentum_mu(t, T) == mu
            assert _lib.lib.pier_momentum_mu(t, T) == mu          # C-ABI restatement
            out = C.c_double()
            rc = _lib.lib.pier_outer_lr(t, T, C.byref(out))
            if olr is None:
                with pytest.raises(ValueError):
                    P.outer_lr(t, s)
                assert rc == _lib.PIER_EINVAL
            else:
                assert P.outer_lr(t, s) == olr
                assert rc == 0 and out.value == olr


def test_acceptance_criterion_5_schedule_exactness():
    """test_acceptance.py:152-169: mu and the outer LR at the phase boundaries of
    T = 3000, exactly (Python host functions and their C-ABI restatements)."""
    sched = P.ScheduleConfig(total_iters=3000)
    mu_expected = {300: 0.99, 301: 0.99, 449: 0.99, 450: 0.95, 599: 0.95,
                   600: 0.9, 2399: 0.9, 2400: 0.9, 3000: 0.9}
    lr_expected = {300: 0.0, 301: 1.0 / 300.0, 449: 149.0 / 300.0, 450: 0.5,
                   599: 299.0 / 300.0, 600: 1.1, 2399: 1.1, 2400: 0.9, 3000: 0.9}
    for t, want in mu_expected.items():
        assert P.momentum_mu(t, 3000) == want and _lib.lib.pier_momentum_mu(t, 3000) == want, t
    for t, want in lr_expected.items():
        out = C.c_double()
        assert P.outer_lr(t, sched) == want, t
        assert _lib.lib.pier_outer_lr(t, 3000, C.byref(out)) == 0 and out.value == want, t


def test_engine_plan_matches_reference_driver_traces():
    for case in json.load(open(os.path.join(GOLDEN, "traces.json"))):
        c = case["case"]
        sched = P.ScheduleConfig(total_iters=c["total_iters"], lazy_fraction=c["lazy_fraction"],
                                 sync_interval=c["sync_interval"])
        plan = PierSchedule(sched, c["mode"], outer_lr_fixed=c.get("outer_lr_fixed"))
        folds = outers = 0
        for rec in case["records"]:
            t = rec["iter"]
            assert plan.phase(t) == rec["phase"]
            if t == 0:
                continue
            ev = plan.event(t)
            if ev is None or ev.kind == "anchor":
                assert rec["mu"] is None and rec["outer_lr"] is None
            else:
                assert ev.mu == rec["mu"] and ev.outer_lr == rec["outer_lr"], (c, t)
                folds += ev.kind == "fold"
                outers += ev.kind == "outer"
            # ring-formula byte accounting of the outer exchange (driver.py:430)
            if ev is not None and ev.kind == "outer":
                want = P.ring_allreduce_bytes(case["param_count"] * 4.0, c["groups"])
                assert rec["comm_bytes"] >= want
        assert folds == case["warmup_folds"] and outers == case["outer_events"]


def test_run_validation_mirrors_reference():
    with pytest.raises(P.ConfigError):   # lazy_end % r != 0 (config.py:149-153)
        validate_run(P.ScheduleConfig(total_iters=100, sync_interval=7), "pier", None, None)
    with pytest.raises(P.ConfigError):   # lazy < 0.1 without fixed outer LR (config.py:178-184)
        validate_run(P.ScheduleConfig(total_iters=100, lazy_fraction=0.0, sync_interval=10), "pier", None, None)
    validate_run(P.ScheduleConfig(total_iters=100, lazy_fraction=0.0, sync_interval=10), "pier", 1.0, None)
    validate_run(P.ScheduleConfig(total_iters=100, lazy_fraction=0.0, sync_interval=10), "diloco_baseline",
                 None, None)
    with pytest.raises(P.ConfigError):
        validate_run(P.ScheduleConfig(total_iters=100, sync_interval=10), "bogus", None, None)
    with pytest.raises(P.ConfigError):
        validate_run(P.ScheduleConfig(total_iters=100, sync_interval=10), "pier", -1.0, None)
    with pytest.raises(P.ConfigError):
        P.AdamWConfig(beta1=1.0)
    with pytest.raises(P.ConfigError):
        P.AdamWConfig(eps=0.0)
    with pytest.raises(P.ConfigError):
        P.ScheduleConfig(total_iters=100, sync_interval=100)
    with pytest.raises(P.ConfigError):
        P.ScheduleConfig(inner_lr_min=1.0, inner_lr_peak=0.1)


def test_diloco_plan_fixed_coefficients_and_no_folds():
    plan = PierSchedule(P.ScheduleConfig(total_iters=60, lazy_fraction=0.5, sync_interval=10), "diloco_baseline")
    evs = [plan.event(t) for t in range(1, 61)]
    evs = [e for e in evs if e is not None]
    assert [e.kind for e in evs] == ["anchor"] * 3 + ["outer"] * 3
    assert all(e.mu == 0.9 and e.outer_lr == 0.7 for e in evs if e.kind == "outer")


@pytest.mark.parametrize("n_params,nranks,bucket", [(1000, 1, 64), (306176, 2, 1 << 12), (124439808, 8, 1 << 22),
                                                    (1557611200, 8, 1 << 24), (4096, 8, 64), (1024, 3, 128)])
def test_bucket_layout_partitions_buffer(n_params, nranks, bucket):
    n_pad = P.padded_len(n_params, nranks)
    assert n_pad >= n_params and n_pad % (nranks * 64) == 0 and n_pad - n_params < nranks * 64
    lay = bucket_layout(n_pad, nranks, bucket)
    # spans tile [0, n_pad); each rank's slices tile its shard [0, n_pad / nranks)
    off = 0
    sh = 0
    for span_off, sl, shard_off in lay:
        assert span_off == off and shard_off == sh and sl % 16 == 0 and sl <= bucket
        off += sl * nranks
        sh += sl
    assert off == n_pad and sh == n_pad // nranks


def test_topology_and_shards_match_reference_semantics():
    topo = P.Topology(groups=2, dp_per_group=2, tp_size=2)
    assert topo.world_size == 8 and topo.num_replicas == 4
    for r in range(8):
        assert topo.rank(*topo.coords(r)) == r
    assert topo.outer_participant_ranks(1) == [1, 3, 5, 7]
    assert P.shard_offsets(10, 3) == [(0, 4), (4, 7), (7, 10)]
    x = np.arange(1031.0)
    for tp in (1, 2, 3, 7):
        assert np.array_equal(P.concat_shards(P.shard_views(x, tp)), x)
    assert P.ring_allreduce_bytes(100.0, 4) == 150.0 and P.ring_allreduce_bytes(100.0, 1) == 0.0
    with pytest.raises(P.ConfigError):
        P.Topology(groups=0)


def test_host_store_disabled_rejects_load():
    hs = P.HostStore(enabled=False)
    hs.store(("snapshot", 0), None)  # ignored when disabled (driver.py:134-135)
    with pytest.raises(P.ProtocolError):
        hs.load(("snapshot", 0))


def test_engine_rejects_non_bitwise_exchanges_beyond_two_groups():
    """The ring / in-switch sums are not the reference's ascending left fold
    (topology.py:113-121): the engine accepts them only where they are bitwise
    (2 groups) and never on a virtual group, which has no NCCL."""
    from types import SimpleNamespace

    sched = P.ScheduleConfig(total_iters=100, sync_interval=10)
    for reduce in ("nccl", "nvls"):
        for world in (3, 4, 8):
            with pytest.raises(P.ConfigError, match="left fold"):
                P.PierEngine(1024, sched, comm=SimpleNamespace(rank=0, world_size=world, virtual=False),
                             reduce=reduce)
        with pytest.raises(P.ConfigError, match="VirtualGroup"):
            P.PierEngine(1024, sched, comm=SimpleNamespace(rank=0, world_size=2, virtual=True), reduce=reduce)


def test_virtual_group_entry_points_validate_without_gpu():
    lib = _lib.lib
    arr = (C.c_void_p * 9)()
    assert lib.pier_vgroup_create(0, arr) == _lib.PIER_EINVAL
    assert lib.pier_vgroup_create(9, arr) == _lib.PIER_EINVAL
    assert lib.pier_vgroup_abort(None) == _lib.PIER_EINVAL
    assert lib.pier_comm_is_virtual(None) == 0
    assert lib.pier_comm_set_timeout(None, 1.0) == _lib.PIER_EINVAL
    assert lib.pier_allreduce_mean_p2p_bf16(None, 0, 64, None) == _lib.PIER_EINVAL
    assert lib.pier_norm_allreduce_team(None, None, 0, None, 1.0, None) == _lib.PIER_EINVAL


def test_sharded_step_entry_points_validate_without_gpu():
    """The sharded-step C-ABI (lazy phase / dp teams / overlap / deferred all-gather) refuses
    a missing communicator or buffers before touching the device, with a message."""
    lib = _lib.lib
    hp = _lib.PierAdamW(1e-3, 0.9, 0.999, 1e-8, 0.1, 1)
    E = _lib.PIER_EINVAL
    assert lib.pier_lazy_step_p2p_f32(None, 0, 1, None, None, 64, 0, C.byref(hp), 1.0, None, None) == E
    assert lib.pier_lazy_step_p2p_team_f32(None, 0, 1, None, 0, None, 0, None, None, 64, 0, C.byref(hp), 1.0,
                                           None, None) == E
    assert lib.pier_lazy_step_p2p_bf16(None, 0, 1, 2, None, None, 64, 0, C.byref(hp), 1.0, None, None) == E
    assert lib.pier_lazy_pull_span_p2p_f32(None, 0, None, 0, None, 64, 0, 0, None) == E
    assert lib.pier_lazy_pull_span_p2p_bf16(None, 0, None, 64, 0, 0, None) == E
    assert lib.pier_lazy_finish_staged_p2p_f32(None, 0, 1, None, 0, None, 0, None, None, None, 64, 0, C.byref(hp),
                                               1.0, None, 1, None) == E
    assert lib.pier_lazy_finish_staged_p2p_bf16(None, 0, 1, 2, None, None, None, 64, 0, C.byref(hp), 1.0, None,
                                                None) == E
    assert lib.pier_allgather_span_p2p_f32(None, 0, None, 0, 64, 0, 0, None) == E
    assert lib.pier_gather_p2p_f32(None, 0, 64, 0, None) == E
    assert lib.pier_gather_p2p_team_f32(None, 0, None, 0, 64, 0, None) == E
    assert "unknown" in _lib.last_error()


def test_group_aborted_maps_to_its_exception():
    with pytest.raises(_lib.GroupAborted):
        _lib.check(_lib.PIER_EABORTED, "x")


def test_span_tracker_reports_each_span_once():
    """grad_ready's host logic: disjoint ranges in any order complete every span exactly once
    (padding final from the start), overlaps are refused, the rest comes in backward order."""
    from paper_2511_17849_b200.engine import SpanTracker

    rng = np.random.default_rng(3)
    for num, npad, span in ((1000, 1024, 128), (4099, 4352, 1024), (50, 256, 64), (7, 64, 64)):
        cuts = sorted({0, num, *rng.integers(0, num + 1, size=9).tolist()})
        pieces = list(zip(cuts[:-1], cuts[1:]))
        rng.shuffle(pieces)
        st = SpanTracker(num, npad, span)
        seen = []
        for lo, hi in pieces:
            seen += st.report(lo, hi)
        nspans = -(-npad // span)
        real = {k for k in range(nspans) if k * span < num}
        assert set(seen) == real and len(seen) == len(real)      # every span holding real params, once
        assert st.rest() == sorted(set(range(nspans)) - real, reverse=True)
        assert st.rest() == []
    st = SpanTracker(1000, 1024, 128)
    st.report(0, 200)
    with pytest.raises(P.ConfigError):
        st.report(100, 300)


def test_stand_in_ranks_pick_one_replica_per_group():
    """The dp > 1 outer exchange folds in, for every participant, the replica of its group
    with the caller's dp index (same tensor shard): one distinct source per group, in the
    participants' ascending order, and the caller's own group served by the caller."""
    for g, dp, tp in ((2, 2, 1), (2, 2, 2), (4, 2, 1), (2, 4, 1), (3, 1, 2)):
        topo = P.Topology(groups=g, dp_per_group=dp, tp_size=tp)
        for rank in range(topo.world_size):
            gr, d, t = topo.coords(rank)
            team = topo.outer_participant_ranks(t)
            reps = topo.stand_in_ranks(rank)
            assert len(reps) == len(team)
            for q, s_ in zip(team, reps):
                assert topo.coords(s_) == (topo.coords(q)[0], d, t)
            assert len(set(reps)) == g                        # one pull per group
            assert all(reps[i] == reps[i - 1] or topo.coords(team[i])[0] != topo.coords(team[i - 1])[0]
                       for i in range(1, len(reps)))          # a group's terms are consecutive
            assert rank in reps                               # our group's copy is our own
