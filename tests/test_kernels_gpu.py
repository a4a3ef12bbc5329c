"""GPU parity of every kernel against the reference (golden fixtures made by
the reference itself) and the pinned oracle.  Bar: BITWISE for every
elementwise fp32/fp64 path (one IEEE rounding per reference ufunc, same
order); the clip norm's BLAS dot order is implementation-defined, so the
norm is held to 2 ulp and everything downstream of the scale is bitwise
given the scale."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import pier_oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2511_17849_b200")
K = np.load(os.path.join(GOLDEN, "kernels.npz"))
TAGS = ("float32", "float64")
MU_LR = ((0.99, 0.205), (0.9, 1.1), (0.9, 0.9), (0.0, 1.0), (0.95, 0.5))


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.detach().cpu().numpy()


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.dtype == b.dtype and a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


# --------------------------------------------------------------------------- AdamW

@pytest.mark.parametrize("tag", TAGS)
@pytest.mark.parametrize("as_numpy", [False, True])
def test_adamw_chain_bitwise_vs_reference(tag, as_numpy):
    conv = (lambda a: a) if as_numpy else cu
    th = conv(K[f"adamw_{tag}_theta0"])
    st = P.AdamWState(m=conv(K[f"adamw_{tag}_m0"]), v=conv(K[f"adamw_{tag}_v0"]), step=10)
    cfg = P.AdamWConfig()
    th_before = K[f"adamw_{tag}_theta0"].copy()
    for k, lr in enumerate(K[f"adamw_{tag}_lrs"]):
        th, st = P.adamw_step(th, conv(K[f"adamw_{tag}_g{k}"]), st, float(lr), cfg)
        get = (lambda a: a) if as_numpy else host
        assert same(get(th), K[f"adamw_{tag}_theta{k + 1}"])
        assert same(get(st.m), K[f"adamw_{tag}_m{k + 1}"])
        assert same(get(st.v), K[f"adamw_{tag}_v{k + 1}"])
    assert st.step == int(K[f"adamw_{tag}_step_final"])
    assert same(K[f"adamw_{tag}_theta0"], th_before)  # purity


def test_adamw_hand_examples():
    # test_optim.py:30-50
    th, st = P.adamw_step(np.array([1.0]), np.array([1.0]), P.AdamWState(np.zeros(1), np.zeros(1)), 0.1,
                          P.AdamWConfig(weight_decay=0.0))
    assert st.step == 1 and st.m[0] == pytest.approx(0.1, rel=1e-12) and st.v[0] == pytest.approx(0.001, rel=1e-12)
    assert th[0] == pytest.approx(0.9, abs=1e-8)
    th, _ = P.adamw_step(np.array([1.0]), np.zeros(1), P.AdamWState(np.zeros(1), np.zeros(1)), 0.1,
                         P.AdamWConfig(weight_decay=0.1))
    assert th[0] == pytest.approx(0.99, rel=1e-15)


@pytest.mark.parametrize("tag", TAGS)
def test_clip_norm_and_scaled_copy(tag):
    g = K[f"clip_{tag}_long"]
    out, nrm = P.clip_global_norm(cu(g), 1.0)
    ref_n = float(K[f"clip_{tag}_long_norm"])
    assert abs(nrm - ref_n) <= 2 * np.spacing(np.dtype(tag).type(ref_n))
    # bitwise given the scale
    scale = np.dtype(tag).type(1.0 / nrm)
    assert same(host(out), g * scale)
    np.testing.assert_allclose(host(out), K[f"clip_{tag}_long_out"], rtol=4 * np.finfo(tag).eps)
    gs_t = cu(K[f"clip_{tag}_short"])
    o2, n2 = P.clip_global_norm(gs_t, 1.0)
    assert o2 is gs_t  # test_optim.py:117-121: no copy under the threshold
    assert n2 == pytest.approx(float(K[f"clip_{tag}_short_norm"]), rel=4 * np.finfo(tag).eps)
    # hand example test_optim.py:111-114
    o3, n3 = P.clip_global_norm(np.array([3.0, 4.0]), 1.0)
    assert n3 == 5.0 and np.allclose(o3, [0.6, 0.8], rtol=1e-15)


@pytest.mark.parametrize("tag", TAGS)
@pytest.mark.parametrize("n", [1, 3, 4, 4099, 1 << 20, (1 << 20) + 7])
def test_fused_clip_adamw_bitwise_given_scale(tag, n):
    rng = np.random.default_rng(n)
    dt = np.dtype(tag)
    th = (rng.standard_normal(n) * 0.02).astype(dt)
    g = (rng.standard_normal(n) * 0.05).astype(dt)
    m = (rng.standard_normal(n) * 1e-4).astype(dt)
    v = (m * m + dt.type(1e-12)).astype(dt)
    tt, gg, mm, vv = cu(th), cu(g), cu(m), cu(v)
    ws = P.norm_workspace()
    cfg = P.AdamWConfig()
    P.grad_sqnorm_(gg, cfg.clip_norm, ws)
    P.adamw_(tt, gg, mm, vv, 11, 2e-3, cfg, ws)
    rec = P.read_clip(ws)
    sq = float(np.dot(g.astype(np.float64), g.astype(np.float64)))
    assert rec.sqnorm == pytest.approx(sq, rel=1e-12)
    gc = g * dt.type(rec.scale) if rec.clipped else g
    want = O.adamw(th, gc, m, v, 10, 2e-3)
    assert same(host(tt), want[0]) and same(host(mm), want[1]) and same(host(vv), want[2])
    # the kernel's norm is the reference formula (dot rounded to the dtype, then a
    # dtype sqrt) on an fp64-accumulated dot: within 1 ulp of the exact norm ...
    exact = float(np.sqrt(np.dtype(tag).type(sq)))
    assert abs(rec.norm - exact) <= 4 * np.spacing(dt.type(exact))
    # ... and within the north_star fp32 tolerance (1e-5) of the reference's BLAS dot,
    # whose fp32 accumulation order is implementation-defined (optim.py:76)
    _, ref_norm = O.clip_global_norm(g, 1.0)
    assert abs(rec.norm - ref_norm) <= 1e-5 * ref_norm


def test_norm_deterministic_and_reusable_workspace():
    g = torch.randn(10_000_003, device="cuda")
    ws = P.norm_workspace()
    vals = []
    for _ in range(3):
        P.grad_sqnorm_(g, 1.0, ws)
        vals.append(P.read_clip(ws).sqnorm)
    assert vals[0] == vals[1] == vals[2]
    assert vals[0] == pytest.approx(float((g.double() ** 2).sum()), rel=1e-12)


def test_unaligned_views_take_scalar_path():
    n = 1001
    base = [torch.randn(n + 1, device="cuda", dtype=torch.float32) for _ in range(4)]
    th, g, m, v = (b[1:] for b in base)  # 4-byte offset: not 16-B aligned
    v.abs_()
    th0, g0, m0, v0 = (host(x).copy() for x in (th, g, m, v))
    P.adamw_(th, g, m, v, 3, 1e-3, P.AdamWConfig())
    want = O.adamw(th0, g0, m0, v0, 2, 1e-3)
    assert same(host(th), want[0]) and same(host(m), want[1]) and same(host(v), want[2])


def _at_offset(x: torch.Tensor, off: int) -> torch.Tensor:
    """A view of a copy of x starting `off` elements into a fresh allocation."""
    buf = torch.empty(x.numel() + off, dtype=x.dtype, device="cuda")
    view = buf[off:]
    view.copy_(x)
    return view


@pytest.mark.parametrize("off", [0, 4, 1], ids=["256bit", "128bit", "scalar"])
def test_vector_width_paths_bitwise(off):
    """The 256-bit body (32-B aligned), the 128-bit body (16-B aligned) and the
    scalar instantiation (unaligned) give the same bits as the reference."""
    n = 100_003
    rng = np.random.default_rng(11)
    th, g, m, an, mo = ((rng.standard_normal(n) * s).astype(np.float32) for s in (0.02, 1e-2, 1e-3, 0.02, 1e-3))
    v = (m * m + np.float32(1e-12)).astype(np.float32)
    T = [_at_offset(cu(x), off) for x in (th, g, m, v, an, mo)]
    ws = P.norm_workspace()
    P.grad_sqnorm_(T[1], 1.0, ws)
    rec = P.read_clip(ws)
    hp = P.AdamWConfig().hyper(3e-3, 7)
    import ctypes as C
    from paper_2511_17849_b200._lib import lib
    assert lib.pier_adamw_outer_f32(*(t.data_ptr() for t in T), n, C.byref(hp), ws.data_ptr(), 1.1, 0.9,
                                    torch.cuda.current_stream().cuda_stream) == 0
    gc = g * np.float32(rec.scale) if rec.clipped else g
    th2, m2, v2, _ = O.adamw(th, gc, m, v, 6, 3e-3)
    want_th, want_mo = O.outer_anchor_form(th2, an, mo, 1.1, 0.9)
    assert same(host(T[2]), m2) and same(host(T[3]), v2)
    assert same(host(T[0]), want_th) and same(host(T[4]), want_th) and same(host(T[5]), want_mo)


@pytest.mark.parametrize("offs", [(0, 0), (0, 1), (4, 0), (1, 3)], ids=["aligned", "bf16_off", "f32_16B", "both_off"])
def test_bf16_master_adamw(offs):
    n = 100_003
    rng = np.random.default_rng(3)
    master = (rng.standard_normal(n) * 0.02).astype(np.float32)
    g32 = (rng.standard_normal(n) * 1e-2).astype(np.float32)
    g16 = torch.from_numpy(g32).to(torch.bfloat16)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    fo, bo = offs
    tm, tmm, tvv = (_at_offset(cu(x), fo) for x in (master, m, v))
    tb = _at_offset(torch.zeros(n, dtype=torch.bfloat16, device="cuda"), bo)
    tg = _at_offset(g16.cuda(), bo)
    ws = P.norm_workspace()
    P.grad_sqnorm_bf16_(tg, 1.0, ws)
    P.adamw_bf16_(tm, tb, tg, tmm, tvv, 1, 3e-3, P.AdamWConfig(), ws)
    rec = P.read_clip(ws)
    gref = g16.float().numpy()
    gc = gref * np.float32(rec.scale) if rec.clipped else gref
    want = O.adamw(master, gc, m, v, 0, 3e-3)
    assert same(host(tm), want[0]) and same(host(tmm), want[1]) and same(host(tvv), want[2])
    assert torch.equal(tb.cpu(), torch.from_numpy(want[0]).to(torch.bfloat16))  # RNE cast
    # the master -> bf16 refresh kernel (after an outer step) on the same layout
    tb.zero_()
    from paper_2511_17849_b200._lib import lib
    assert lib.pier_cast_bf16(tm.data_ptr(), tb.data_ptr(), n, torch.cuda.current_stream().cuda_stream) == 0
    assert torch.equal(tb.cpu(), torch.from_numpy(want[0]).to(torch.bfloat16))


def _mt_against_oracle(params, steps, lr, threads=1):
    """MultiTensorAdamW on `params` for `steps` steps; every tensor checked bitwise
    against the oracle (optim.py:82-103) given the clip scale the kernel applied."""
    import os

    opt = P.MultiTensorAdamW(params)
    host = [(p.detach().cpu().numpy(), p.grad.cpu().numpy()) for p in params]
    ms = [np.zeros_like(h[0]) for h in host]
    vs = [np.zeros_like(h[0]) for h in host]
    ths = [h[0] for h in host]
    clipped = []
    for step in range(1, steps + 1):
        opt.step(lr)
        rec = P.read_clip(opt.ws)               # the scale this step applied (optim.py:76-78)
        clipped.append(bool(rec.clipped))
        for i, (th, (_, g)) in enumerate(zip(ths, host)):
            gc = g * g.dtype.type(rec.scale) if rec.clipped else g
            fn = lambda a, b, c, d: O.adamw(a, b, c, d, step - 1, lr)[:3]  # noqa: E731
            if threads > 1 and th.size > (1 << 22):
                ths[i], ms[i], vs[i] = O.chunked(fn, [th.reshape(-1), gc.reshape(-1), ms[i].reshape(-1),
                                                      vs[i].reshape(-1)], threads)
                ths[i], ms[i], vs[i] = (x.reshape(th.shape) for x in (ths[i], ms[i], vs[i]))
            else:
                ths[i], ms[i], vs[i] = fn(th, gc, ms[i], vs[i])
    bad = [i for i, p in enumerate(params)
           if not (same(p.detach().cpu().numpy(), ths[i]) and same(opt.m[i].cpu().numpy(), ms[i])
                   and same(opt.v[i].cpu().numpy(), vs[i]))]
    opt.close()
    return bad, clipped


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_multi_tensor_adamw_bitwise_vs_oracle(dtype):
    """Odd shapes: chunk tails that are not a multiple of the vector width, tensors
    shorter than one vector, and a clip that turns on at step 2."""
    shapes = [(50257 // 7, 64), (1024, 64), (64,), (64,), (64, 192), (192,), (3,), (5, 7), (1,), (8191,), (8193,)]
    torch.manual_seed(7)
    params = [torch.randn(s, dtype=dtype, device="cuda") * 0.02 for s in shapes]
    for p in params:
        p.grad = torch.randn_like(p) * 0.001
    bad, clipped = _mt_against_oracle(params, 1, 1e-3)
    assert not bad and clipped == [False]
    for p in params:
        p.grad.mul_(1000.0)                     # |g| ~ 25 > clip 1.0
    opt_bad, clipped = _mt_against_oracle(params, 2, 3e-3)
    assert not opt_bad and clipped == [True, True]


def test_multi_tensor_adamw_gpt2_xl_list_bitwise_vs_oracle():
    """The 580-tensor GPT-2 XL list (1.56e9 params, separate allocations), one
    clipped step, every tensor bitwise against the oracle given the scale."""
    import os
    avail = 0
    for line in open("/proc/meminfo"):
        if line.startswith("MemAvailable:"):
            avail = int(line.split()[1]) * 1024
    if avail < 96e9:
        pytest.skip("needs ~96 GB of host RAM for the oracle")
    d, V, L = 1600, 50257, 48
    shapes = [(V, d), (1024, d)]
    for _ in range(L):
        shapes += [(d,), (d,), (d, 3 * d), (3 * d,), (d, d), (d,), (d,), (d,), (d, 4 * d), (4 * d,), (4 * d, d), (d,)]
    shapes += [(d,), (d,)]
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    params = [torch.empty(s, device="cuda").normal_(0, 0.02, generator=gen) for s in shapes]
    for p in params:
        p.grad = torch.empty_like(p).normal_(0, 1e-4, generator=gen)   # |g| ~ 3.9 > 1: clipped
    assert len(params) == 580 and sum(p.numel() for p in params) == 1_557_611_200
    bad, clipped = _mt_against_oracle(params, 1, 3e-3, threads=len(os.sched_getaffinity(0)))
    assert not bad and clipped == [True], bad[:5]


# --------------------------------------------------------------------------- outer step

@pytest.mark.parametrize("tag", TAGS)
@pytest.mark.parametrize("mu,lr", MU_LR)
def test_outer_fold_pure_forms_bitwise(tag, mu, lr):
    anchor, mom = K[f"outer_{tag}_anchor"], K[f"outer_{tag}_mom"]
    ths = [K[f"outer_{tag}_theta{i}"] for i in range(8)]
    key = f"{mu}_{lr}"
    for n in (1, 2, 3, 4, 8):
        avg = P.allreduce_avg([cu(t) for t in ths[:n]])
        assert same(host(avg), K[f"mean_{tag}_n{n}"])
        delta = P.pseudograd(avg, cu(anchor))
        assert same(host(delta), K[f"mean_{tag}_n{n}"] - anchor)
        st = P.OuterState(momentum=cu(mom), snapshot=cu(anchor))
        th_new, st2 = P.outer_step(st, delta, lr, mu, anchor=avg)
        assert same(host(th_new), K[f"outer_{tag}_{key}_n{n}_theta"])
        assert same(host(st2.momentum), K[f"outer_{tag}_{key}_n{n}_mom"])
        assert st2.mu == mu and st2.snapshot is st.snapshot
        # fused K3 on the SUM (division inside the kernel, topology.py:121)
        acc = ths[0].copy()
        for t in ths[1:n]:
            acc += t
        s_, a_, m_ = cu(acc), cu(anchor), cu(mom)
        P.outer_update_(s_, a_, m_, lr, mu, divisor=n)
        assert same(host(s_), K[f"outer_{tag}_{key}_n{n}_theta"])
        assert same(host(a_), K[f"outer_{tag}_{key}_n{n}_theta"])
        assert same(host(m_), K[f"outer_{tag}_{key}_n{n}_mom"])
    th_s, st_s = P.outer_step(P.OuterState(momentum=mom, snapshot=anchor), ths[0] - anchor, lr, mu)
    assert same(th_s, K[f"outer_{tag}_{key}_snapform_theta"])
    assert same(st_s.momentum, K[f"outer_{tag}_{key}_snapform_mom"])
    assert same(host(P.fold_momentum(cu(mom), cu(ths[0] - anchor), mu)), K[f"fold_{tag}_{key}"])
    a_, m_ = cu(anchor), cu(mom)
    P.warmup_fold_(cu(ths[0]), a_, m_, mu)
    assert same(host(m_), K[f"fold_{tag}_{key}"]) and same(host(a_), ths[0])


def test_edge_cases_empty_zero_and_max_participants():
    # empty buffers: every entry point is a no-op, not an error
    e = np.zeros(0, np.float32)
    th, st = P.adamw_step(e, e, P.AdamWState(e, e), 1e-3, P.AdamWConfig())
    assert th.shape == (0,) and st.step == 1
    assert P.fold_momentum(e, e, 0.9).shape == (0,)
    assert P.allreduce_avg([e, e]).shape == (0,)
    # zero gradient: norm 0 <= max_norm -> returned unscaled, same object (optim.py:77-79)
    z = torch.zeros(1000, device="cuda")
    out, nrm = P.clip_global_norm(z, 1.0)
    assert out is z and nrm == 0.0
    # 64 participants is the K6 limit; more is rejected like a malformed collective
    parts = [torch.full((37,), float(i), device="cuda") for i in range(64)]
    want = O.mean_left_fold([host(p) for p in parts])
    assert same(host(P.allreduce_avg(parts)), want)
    with pytest.raises(ValueError):
        P.allreduce_avg(parts + [parts[0]])
    # non-finite gradients are reported by the norm record (NumericError in the engine)
    g = torch.ones(10, device="cuda")
    g[3] = float("nan")
    ws = P.norm_workspace()
    P.grad_sqnorm_(g, 1.0, ws)
    assert P.read_clip(ws).nonfinite == 1


def test_full_size_xl_fused_round_properties():
    """N = 1,557,611,200 (GPT-2 XL, the bench size): K5 on the whole buffer equals
    the oracle on a strided sample bitwise; mu=0, lr=1 makes the outer part land
    bitwise on the AdamW result (the degenerate step, test_optim.py:236-246)."""
    n = 1_557_611_200
    gen = torch.Generator(device="cuda").manual_seed(9)
    f = dict(device="cuda", dtype=torch.float32)
    th = torch.empty(n, **f).normal_(0, 0.02, generator=gen)
    g = torch.empty(n, **f).normal_(0, 1e-4, generator=gen)
    m = torch.empty(n, **f).normal_(0, 1e-4, generator=gen)
    v = (m * m).add_(1e-12)
    an = th + torch.empty(n, **f).normal_(0, 1e-3, generator=gen)
    mo = torch.empty(n, **f).normal_(0, 1e-3, generator=gen)
    idx = torch.arange(5, n, 104_729, device="cuda")
    s = [host(x[idx]) for x in (th, g, m, v, an, mo)]
    ws = P.norm_workspace()
    P.grad_sqnorm_(g, 1.0, ws)
    from paper_2511_17849_b200._lib import lib
    import ctypes as C
    hp = P.AdamWConfig().hyper(2e-3, 11)
    rc = lib.pier_adamw_outer_f32(th.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), an.data_ptr(),
                                  mo.data_ptr(), n, C.byref(hp), ws.data_ptr(), 1.1, 0.9,
                                  torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    rec = P.read_clip(ws)
    assert rec.clipped == 1   # |g| ~ 3.9 > 1 at XL: the clip path is active
    gc = s[1] * np.float32(rec.scale)
    t1, m1, v1, _ = O.adamw(s[0], gc, s[2], s[3], 10, 2e-3)
    t2, mo2 = O.outer_anchor_form(t1, s[4], s[5], 1.1, 0.9)
    assert same(host(th[idx]), t2) and same(host(mo[idx]), mo2) and same(host(an[idx]), t2)
    assert same(host(m[idx]), m1) and same(host(v[idx]), v1)


def test_7b_scale_bf16_path_int64_indexing():
    """N = 6,658,596,864 (BASELINE config 5, the synthetic 7B: > 2^32 elements,
    107 GB of state on one GPU): bf16 norm + bf16-master AdamW + the master ->
    bf16 refresh equal the oracle bitwise on samples that straddle the 2^31 and
    2^32 element boundaries and the tail."""
    n = 6_658_596_864
    torch.cuda.empty_cache()   # earlier XL tests leave ~40 GB cached
    gen = torch.Generator(device="cuda").manual_seed(7)
    f = dict(device="cuda", dtype=torch.float32)
    master = torch.empty(n, **f).normal_(0, 0.02, generator=gen)
    g16 = torch.empty(n, device="cuda", dtype=torch.bfloat16).normal_(0, 1e-4, generator=gen)
    m = torch.empty(n, **f).normal_(0, 1e-4, generator=gen)
    v = (m * m).add_(1e-12)
    th16 = torch.zeros(n, device="cuda", dtype=torch.bfloat16)
    edges = [0, 1, (1 << 31) - 3, 1 << 31, (1 << 32) - 5, 1 << 32, n - 9]
    idx = torch.cat([torch.arange(3, n, 1_048_573, device="cuda")] +
                    [torch.arange(e, min(e + 9, n), device="cuda") for e in edges])
    s_master, s_m, s_v = (host(x[idx]) for x in (master, m, v))
    s_g = g16[idx].float().cpu().numpy()
    ws = P.norm_workspace()
    P.grad_sqnorm_bf16_(g16, 1.0, ws)
    P.adamw_bf16_(master, th16, g16, m, v, 5, 1e-3, P.AdamWConfig(), ws)
    rec = P.read_clip(ws)
    assert rec.clipped == 1   # |g| ~ 8.2 at 6.7e9 params
    gc = s_g * np.float32(rec.scale)
    want = O.adamw(s_master, gc, s_m, s_v, 4, 1e-3)
    assert same(host(master[idx]), want[0]) and same(host(m[idx]), want[1]) and same(host(v[idx]), want[2])
    want16 = torch.from_numpy(want[0]).to(torch.bfloat16)
    assert torch.equal(th16[idx].cpu(), want16)
    th16.zero_()
    from paper_2511_17849_b200._lib import lib
    assert lib.pier_cast_bf16(master.data_ptr(), th16.data_ptr(), n, torch.cuda.current_stream().cuda_stream) == 0
    assert torch.equal(th16[idx].cpu(), want16)


def test_fold_and_mean_hand_examples():
    assert np.array_equal(P.fold_momentum(np.array([1.0, 2.0]), np.array([0.5, 0.5]), 0.9), [1.4, 2.3])
    assert np.array_equal(P.allreduce_avg([np.array([1.0, 3.0]), np.array([3.0, 5.0])]), [2.0, 4.0])
    x = np.random.default_rng(0).normal(size=50)
    out = P.allreduce_avg([x])
    assert np.array_equal(out, x) and out is not x
    d = np.random.default_rng(2).normal(size=10)
    assert np.all(P.outer_delta_sync([d, -d, d, -d]) == 0.0)
    with pytest.raises(ValueError):
        P.allreduce_avg([np.zeros(3), np.zeros(4)])
    with pytest.raises(ValueError):
        P.allreduce_avg([])


def test_empty_and_tiny_sizes():
    for n in (0, 1, 2, 3, 5):
        a = torch.randn(n, device="cuda")
        b = torch.randn(n, device="cuda")
        m = torch.randn(n, device="cuda")
        want = O.outer_anchor_form(host(a), host(b), host(m), 0.9, 0.99)
        P.outer_update_(a, b, m, 0.9, 0.99)
        assert same(host(a), want[0]) and same(host(m), want[1])


def test_full_size_gpt2_small_properties():
    """N = 124,439,808 (GPT-2 small): degenerate step lands bitwise on the
    average; a strided sample equals the oracle bitwise (elementwise ops are
    position-independent)."""
    n = 124_439_808
    gen = torch.Generator(device="cuda").manual_seed(0)
    anchor = torch.randn(n, device="cuda", generator=gen) * 0.02
    avg = anchor + torch.randn(n, device="cuda", generator=gen) * 1e-3
    mom = torch.randn(n, device="cuda", generator=gen) * 1e-3
    idx = torch.arange(0, n, 9973, device="cuda")
    a0, an0, m0 = host(avg[idx]), host(anchor[idx]), host(mom[idx])
    th = avg.clone()
    P.outer_update_(th, anchor.clone(), mom.clone(), 1.0, 0.0)
    assert torch.equal(th, avg)  # test_optim.py:236-246 at full size
    an, mm = anchor.clone(), mom.clone()
    th = avg.clone()
    P.outer_update_(th, an, mm, 0.205, 0.99)
    want = O.outer_anchor_form(a0, an0, m0, 0.205, 0.99)
    assert same(host(th[idx]), want[0]) and same(host(mm[idx]), want[1]) and torch.equal(an, th)


# --------------------------------------------------------------------------- open loop / engine

@pytest.mark.parametrize("T,g", [(200, 1), (200, 2), (200, 3), (200, 4), (200, 8), (1000, 2), (1000, 8)])
def test_open_loop_virtual_groups_bitwise_vs_reference_engine(T, g):
    """K6 (left-fold mean of g virtual groups on one GPU) + K3b/K3 driven through
    the whole schedule equals the reference ENGINE's final anchor/momentum."""
    f = np.load(os.path.join(GOLDEN, f"open_loop_T{T}_r10_g{g}.npz"))
    sched = P.ScheduleConfig(total_iters=T, lazy_fraction=0.1, sync_interval=10)
    from paper_2511_17849_b200.engine import PierSchedule
    plan = PierSchedule(sched, "pier")
    anchor = cu(f["theta0"])
    mom = torch.zeros_like(anchor)
    k = 0
    for t in range(1, T + 1):
        ev = plan.event(t)
        if ev is None:
            continue
        a_h = host(anchor)
        thetas = [cu(O.open_loop_inputs(0, k, gi, a_h)) for gi in range(g)]
        if ev.kind == "fold":
            P.warmup_fold_(thetas[0], anchor, mom, ev.mu)
        else:
            avg = P.allreduce_avg(thetas)
            P.outer_update_(avg, anchor, mom, ev.outer_lr, ev.mu)
        k += 1
    assert same(host(anchor), f["anchor"])
    assert same(host(mom), f["momentum"])


def test_engine_single_group_open_loop_and_offload():
    """PierEngine (n=1) boundary stage through the T=200 schedule, params
    overwritten open-loop before each boundary: bitwise equal to the reference
    engine; with offload the results are identical and the counters follow
    the reference's HostStore accounting (driver.py:133-150)."""
    f = np.load(os.path.join(GOLDEN, "open_loop_T200_r10_g1.npz"))
    n = f["theta0"].shape[0]
    outs = []
    for offload in (False, True):
        sched = P.ScheduleConfig(total_iters=200, lazy_fraction=0.1, sync_interval=10)
        eng = P.PierEngine(n, sched, offload=offload, theta0=cu(f["theta0"]), bucket_elems=64)
        k = 0
        for t in range(1, 201):
            if eng.is_boundary(t):
                anc = host(eng.snapshot())
                eng.theta[:n].copy_(cu(O.open_loop_inputs(0, k, 0, anc)))
                k += 1
                eng.boundary(t)
        outs.append((host(eng.params()), host(eng.outer_momentum()), eng.host.counters(), eng.warmup_folds))
        assert [r.kind for r in eng.records].count("fold") == 2
    for got in outs:
        assert same(got[0], f["anchor"]) and same(got[1], f["momentum"])
        assert got[3] == int(f["folds"])
    c = outs[1][2]
    boundaries = 20
    assert c["to_host_bytes"] == (boundaries + 1) * 2 * n * 4
    assert c["store_events"] == (boundaries + 1) * 2 and c["load_events"] == boundaries * 2
    assert c["resident_bytes"] == 2 * n * 4
    assert outs[0][2]["to_host_bytes"] == 0.0


def test_engine_trace_and_inner_steps_match_oracle():
    """Engine with real inner steps (random grads): records equal the
    reference driver's schedule; params equal a pure-oracle replay bitwise."""
    n = 4099
    T, r = 60, 10
    sched = P.ScheduleConfig(total_iters=T, lazy_fraction=0.5, sync_interval=r)
    rng = np.random.default_rng(11)
    theta0 = (rng.standard_normal(n) * 0.02).astype(np.float32)
    eng = P.PierEngine(n, sched, theta0=cu(theta0), bucket_elems=1024)
    th, m, v = theta0.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)
    anchor, mom = theta0.copy(), np.zeros(n, np.float32)
    osch = O.Sched(total_iters=T, lazy_fraction=0.5, sync_interval=r)
    evs = {e.t: e for e in O.boundary_events(osch, "pier")}
    for t in range(1, T + 1):
        g = (rng.standard_normal(n) * 0.1).astype(np.float32)
        eng.grad[:n].copy_(cu(g))
        eng.step(t)
        clip = eng.last_clip()
        gc = g * np.float32(clip.scale) if clip.clipped else g
        th, m, v, _ = O.adamw(th, gc, m, v, t - 1, O.inner_lr(t, osch))
        e = evs.get(t)
        if e is not None and e.kind == "fold":
            mom, anchor = O.warmup_fold(th, anchor, mom, e.mu)
        elif e is not None:
            th, mom = O.outer_anchor_form(th, anchor, mom, e.lr, e.mu)
            anchor = th.copy()
        assert same(host(eng.params()), th), t
    assert same(host(eng.outer_momentum()), mom)
    assert [(x.iteration, x.kind, x.mu, x.outer_lr) for x in eng.records] == \
        [(e.t, e.kind, e.mu, e.lr) for e in evs.values()]


@pytest.mark.parametrize("offload", [False, True])
def test_fused_boundary_round_equals_unfused(offload):
    """K5 (AdamW + outer step in one pass) == K4b then K3, bitwise, with clipping."""
    n = 300_007
    T = 100
    sched = P.ScheduleConfig(total_iters=T, lazy_fraction=0.1, sync_interval=10)
    rng = np.random.default_rng(5)
    theta0 = cu((rng.standard_normal(n) * 0.02).astype(np.float32))
    outs = []
    for fuse in (True, False):
        eng = P.PierEngine(n, sched, theta0=theta0, offload=offload, bucket_elems=4096)
        g = torch.Generator(device="cuda").manual_seed(1)
        for t in range(1, T + 1):
            eng.grad[:n].normal_(0.0, 0.01, generator=g)   # |g| ~ 5.5 > 1: clip path active
            eng.step(t, fuse=fuse)
        outs.append((host(eng.params()), host(eng.outer_momentum()), host(eng.m[:n]), host(eng.v[:n])))
    for a, b in zip(*outs):
        assert same(a, b)


def test_step_host_equals_device_step():
    """The host-buffer call (e2e path: H2D, round, D2H every step; chunked
    pipeline at outer boundaries) gives bitwise the device-resident result."""
    n = 200_003
    T = 60
    sched = P.ScheduleConfig(total_iters=T, lazy_fraction=0.5, sync_interval=10)
    rng = np.random.default_rng(6)
    theta0 = (rng.standard_normal(n) * 0.02).astype(np.float32)
    dev_eng = P.PierEngine(n, sched, theta0=cu(theta0))
    host_eng = P.PierEngine(n, sched, theta0=cu(theta0))
    host_eng.host_chunk = 4096 * 3
    pin = dict(dtype=torch.float32, pin_memory=True)
    hs = {"theta": torch.from_numpy(theta0.copy()).pin_memory(), "grad": torch.empty(n, **pin),
          "m": torch.zeros(n, **pin), "v": torch.zeros(n, **pin),
          "anchor": torch.from_numpy(theta0.copy()).pin_memory(), "mom": torch.zeros(n, **pin)}
    for t in range(1, T + 1):
        g = (rng.standard_normal(n) * 0.01).astype(np.float32)
        dev_eng.grad[:n].copy_(cu(g))
        dev_eng.step(t)
        hs["grad"].copy_(torch.from_numpy(g))
        host_eng.step_host(t, hs)
    assert same(hs["theta"].numpy(), host(dev_eng.params()))
    assert same(hs["mom"].numpy(), host(dev_eng.outer_momentum()))
    assert same(hs["m"].numpy(), host(dev_eng.m[:n])) and same(hs["v"].numpy(), host(dev_eng.v[:n]))
    assert [r.kind for r in host_eng.records] == [r.kind for r in dev_eng.records]


@pytest.mark.parametrize("mode", ["pier", "diloco_baseline"])
@pytest.mark.parametrize("fuse", [True, False])
def test_degenerate_settings_reduce_to_adamw_baseline(mode, fuse):
    """test_driver.py:203-227 (acceptance criterion 1) on the GPU engine: one
    group, lazy_fraction 0, outer lr fixed 1, mu fixed 0 -> every outer step
    lands bitwise on the AdamW result, so the run equals the synchronous AdamW
    baseline bitwise (fused K5 boundary and the unfused K4b + K3 path)."""
    n = 50_021
    T, r = 60, 10
    rng = np.random.default_rng(21)
    theta0 = cu((rng.standard_normal(n) * 0.02).astype(np.float32))
    grads = [cu((rng.standard_normal(n) * 0.05).astype(np.float32)) for _ in range(T)]   # |g| ~ 11: clipped
    runs = []
    for kw in (dict(mode=mode, outer_lr_fixed=1.0, outer_mu_fixed=0.0), dict(mode="adamw_baseline")):
        eng = P.PierEngine(n, P.ScheduleConfig(total_iters=T, lazy_fraction=0.0, sync_interval=r), theta0=theta0,
                           bucket_elems=1024, **kw)
        for t in range(1, T + 1):
            eng.grad[:n].copy_(grads[t - 1])
            eng.step(t, fuse=fuse)
        runs.append((host(eng.params()), eng.opt_step, [x.kind for x in eng.records]))
    (pier_th, pier_steps, kinds), (base_th, base_steps, base_kinds) = runs
    assert same(pier_th, base_th)
    assert pier_steps == base_steps == T
    assert kinds == ["outer"] * (T // r) and base_kinds == []


def test_step_is_graph_capturable():
    """No host synchronisation on the hot path: one inner step (K4a norm + K4b)
    and one fused boundary step (K4a + K5) captured into CUDA graphs replay to
    the eager engine's results bitwise (the clip scale stays on the device)."""
    n = 100_003
    T, r = 100, 10
    sched = P.ScheduleConfig(total_iters=T, lazy_fraction=0.1, sync_interval=r)
    rng = np.random.default_rng(31)
    theta0 = cu((rng.standard_normal(n) * 0.02).astype(np.float32))
    grads = [cu((rng.standard_normal(n) * 0.05).astype(np.float32)) for _ in range(2)]   # clipped
    eager = P.PierEngine(n, sched, theta0=theta0, bucket_elems=1024)
    graphed = P.PierEngine(n, sched, theta0=theta0, bucket_elems=1024)
    t_inner, t_outer = 29, 30          # lazy_end = 10: t = 30 is an outer step
    for eng in (eager, graphed):
        eng.opt_step = t_inner - 1
    for t, gr in ((t_inner, grads[0]), (t_outer, grads[1])):
        eager.grad[:n].copy_(gr)
        eager.step(t)
        graphed.grad[:n].copy_(gr)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            graphed.step(t)
        g.replay()
        torch.cuda.synchronize()
        assert same(host(graphed.params()), host(eager.params())), t
    assert same(host(graphed.outer_momentum()), host(eager.outer_momentum()))
    assert same(host(graphed.m[:n]), host(eager.m[:n])) and same(host(graphed.v[:n]), host(eager.v[:n]))


def test_snapshot_frozen_between_boundaries_and_inner_step_count():
    """test_driver.py:261-282: the anchor (snapshot) changes exactly at boundary
    iterations -- folds and outer steps -- and never in between; the inner
    step count equals total_iters for any sync interval."""
    n = 20_011
    T = 60
    rng = np.random.default_rng(41)
    theta0 = cu((rng.standard_normal(n) * 0.02).astype(np.float32))
    for r in (5, 10, 30):
        sched = P.ScheduleConfig(total_iters=T, lazy_fraction=0.5, sync_interval=r)
        eng = P.PierEngine(n, sched, theta0=theta0, bucket_elems=1024)
        prev = host(eng.snapshot()).copy()
        for t in range(1, T + 1):
            eng.grad[:n].copy_(cu((rng.standard_normal(n) * 0.05).astype(np.float32)))
            eng.step(t)
            snap = host(eng.snapshot())
            changed = not same(snap, prev)
            assert changed == (t % r == 0), (r, t)
            prev = snap.copy()
        assert eng.opt_step == T
        assert [x.iteration for x in eng.records] == list(range(r, T + 1, r))
