"""The persistent round kernel (csrc/pier_round.cu, k_round<n>) for every group
count 2..8 on ONE GPU: n virtual ranks whose "peer" buffers live on the same
device (pier_round_virtual_f32).  A 4-GPU box cannot launch the 8-group
instantiation the 8-GPU scaling run uses; this runs it, bitwise against the
oracle (per-group clip + AdamW, ascending left-fold mean, anchor-form outer
step, driver.py:395-440), for two consecutive rounds and a round with a
different span count on the same signal blocks (booked counters)."""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import pier_oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2511_17849_b200")


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _ptrs(ts):
    return (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


def _shard(full, layout, q):
    return np.concatenate([full[off + q * sl: off + (q + 1) * sl] for off, sl, _ in layout])


def _full(shards, layout, n_pad):
    out = np.zeros(n_pad, np.float32)
    for q, sh_arr in enumerate(shards):
        for off, sl, sh in layout:
            out[off + q * sl: off + (q + 1) * sl] = sh_arr[sh: sh + sl]
    return out


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 7, 8])
def test_round_kernel_virtual_ranks_bitwise(n):
    from paper_2511_17849_b200._lib import lib
    from paper_2511_17849_b200.engine import bucket_layout

    num = 70_001
    n_pad = P.padded_len(num, n)
    rng = np.random.default_rng([21, n])
    f32 = np.float32
    theta = [np.zeros(n_pad, f32) for _ in range(n)]
    grads = [np.zeros(n_pad, f32) for _ in range(n)]
    ms = [np.zeros(n_pad, f32) for _ in range(n)]
    vs = [np.zeros(n_pad, f32) for _ in range(n)]
    anchor = np.zeros(n_pad, f32)
    anchor[:num] = (rng.standard_normal(num) * 0.02).astype(f32)
    mom = np.zeros(n_pad, f32)
    mom[:num] = (rng.standard_normal(num) * 1e-3).astype(f32)
    for q in range(n):
        theta[q][:num] = anchor[:num] + (rng.standard_normal(num) * 1e-3).astype(f32)
        ms[q][:num] = (rng.standard_normal(num) * 1e-4).astype(f32)
        vs[q][:num] = ms[q][:num] * ms[q][:num] + f32(1e-12)
    T = [torch.from_numpy(x.copy()).cuda() for x in theta]
    M = [torch.from_numpy(x.copy()).cuda() for x in ms]
    V = [torch.from_numpy(x.copy()).cuda() for x in vs]
    G = [torch.zeros(n_pad, device="cuda") for _ in range(n)]
    sig = [torch.zeros(lib.pier_round_sig_bytes() // 4, dtype=torch.int32, device="cuda") for _ in range(n)]
    ws = [P.norm_workspace() for _ in range(n)]
    streams = [torch.cuda.Stream() for _ in range(n)]
    cfg = P.AdamWConfig()
    state = {"anchor": anchor, "mom": mom}
    step = 10

    # two rounds with 1024-element slices, then one with 512 (more spans, same signal blocks)
    for rnd, (bucket, lr, mu, clip_scale) in enumerate(((1024, 1.1, 0.9, 1e-2), (1024, 0.205, 0.99, 1.0),
                                                         (512, 0.9, 0.9, 5.0))):
        layout = bucket_layout(n_pad, n, bucket)
        for q in range(n):
            g = np.zeros(n_pad, f32)
            g[:num] = (rng.standard_normal(num) * clip_scale / np.sqrt(num)).astype(f32)
            grads[q] = g
            G[q].copy_(torch.from_numpy(g))
        AN = [torch.from_numpy(_shard(state["anchor"], layout, q)).cuda() for q in range(n)]
        MO = [torch.from_numpy(_shard(state["mom"], layout, q)).cuda() for q in range(n)]
        for q in range(n):
            P.grad_sqnorm_(G[q], cfg.clip_norm, ws[q])
        torch.cuda.synchronize()
        step += 1
        hp = cfg.hyper(2e-3, step)
        rc = lib.pier_round_virtual_f32(n, _ptrs(T), _ptrs(G), _ptrs(M), _ptrs(V), _ptrs(AN), _ptrs(MO),
                                        _ptrs(sig), n_pad, bucket, C.byref(hp), _ptrs(ws), lr, mu, 6, 4,
                                        (C.c_void_p * n)(*[s.cuda_stream for s in streams]))
        assert rc == 0, P._lib.last_error()
        torch.cuda.synchronize()

        # oracle: every group's clip + AdamW, the ascending mean, the outer step
        after = []
        for q in range(n):
            rec = P.read_clip(ws[q])
            gc = grads[q] * f32(rec.scale) if rec.clipped else grads[q]
            th2, m2, v2, _ = O.adamw(theta[q], gc, ms[q], vs[q], step - 1, 2e-3)
            ms[q], vs[q] = m2, v2
            after.append(th2)
        avg = O.mean_left_fold(after)
        th_new, mom_new = O.outer_anchor_form(avg, state["anchor"], state["mom"], lr, mu)
        for q in range(n):
            theta[q] = th_new.copy()
            assert np.array_equal(T[q].cpu().numpy().view(np.uint32), th_new.view(np.uint32)), (rnd, q)
            assert np.array_equal(M[q].cpu().numpy().view(np.uint32), ms[q].view(np.uint32)), (rnd, q)
            assert np.array_equal(V[q].cpu().numpy().view(np.uint32), vs[q].view(np.uint32)), (rnd, q)
        got_an = _full([a.cpu().numpy() for a in AN], layout, n_pad)
        got_mo = _full([a.cpu().numpy() for a in MO], layout, n_pad)
        assert np.array_equal(got_an.view(np.uint32), th_new.view(np.uint32)), rnd
        assert np.array_equal(got_mo.view(np.uint32), mom_new.view(np.uint32)), rnd
        state = {"anchor": th_new, "mom": mom_new}
        if rnd == 0:
            assert any(P.read_clip(w).clipped for w in ws) is False
        if rnd == 2:
            assert all(P.read_clip(w).clipped for w in ws)   # the clip path inside the round


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("outer", [0, 1], ids=["grad_mean", "outer_step"])
def test_p2p_kernel_virtual_ranks_bitwise(n, outer):
    """k_p2p_reduce<MEAN|OUTER, n> (the lazy-phase gradient mean and the unfused
    outer step) for every group count, bitwise vs the left fold (+ outer step)."""
    from paper_2511_17849_b200._lib import lib
    from paper_2511_17849_b200.engine import bucket_layout

    num, bucket = 50_003, 512
    n_pad = P.padded_len(num, n)
    layout = bucket_layout(n_pad, n, bucket)
    rng = np.random.default_rng([22, n, outer])
    f32 = np.float32
    xs = []
    for _ in range(n):
        x = np.zeros(n_pad, f32)
        x[:num] = rng.standard_normal(num).astype(f32)
        xs.append(x)
    anchor = np.zeros(n_pad, f32)
    anchor[:num] = rng.standard_normal(num).astype(f32)
    mom = np.zeros(n_pad, f32)
    mom[:num] = (rng.standard_normal(num) * 0.1).astype(f32)
    B = [torch.from_numpy(x).cuda() for x in xs]
    AN = [torch.from_numpy(_shard(anchor, layout, q)).cuda() for q in range(n)]
    MO = [torch.from_numpy(_shard(mom, layout, q)).cuda() for q in range(n)]
    streams = [torch.cuda.Stream() for _ in range(n)]
    torch.cuda.synchronize()
    rc = lib.pier_p2p_virtual_f32(n, outer, _ptrs(B), _ptrs(AN), _ptrs(MO), n_pad, bucket, 0.9, 0.95,
                                  (C.c_void_p * n)(*[s.cuda_stream for s in streams]))
    assert rc == 0, P._lib.last_error()
    torch.cuda.synchronize()
    avg = O.mean_left_fold(xs)
    if outer:
        want, want_mo = O.outer_anchor_form(avg, anchor, mom, 0.9, 0.95)
        got_an = _full([a.cpu().numpy() for a in AN], layout, n_pad)
        got_mo = _full([a.cpu().numpy() for a in MO], layout, n_pad)
        assert np.array_equal(got_an.view(np.uint32), want.view(np.uint32))
        assert np.array_equal(got_mo.view(np.uint32), want_mo.view(np.uint32))
    else:
        want = avg
    for q in range(n):
        assert np.array_equal(B[q].cpu().numpy().view(np.uint32), want.view(np.uint32)), q
