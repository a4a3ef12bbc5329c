"""The C-ABI exactly as a reference maintainer would bind it:
raw ctypes, raw device pointers, the torch stream as a void*, int status codes."""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import pier_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_17849_b200 import _lib
    return C.CDLL(_lib.LIB_PATH)


class PierAdamW(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("weight_decay", C.c_double), ("step", C.c_int64)]


class PierClip(C.Structure):
    _fields_ = [("sqnorm", C.c_double), ("norm", C.c_double), ("scale", C.c_double),
                ("clipped", C.c_int32), ("nonfinite", C.c_int32)]


def vp(t):
    return C.c_void_p(t.data_ptr())


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def same(a, b):
    return np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))


def test_raw_abi_clip_adamw_outer_round(lib):
    n = 65_539
    rng = np.random.default_rng(21)
    th = (rng.standard_normal(n) * 0.02).astype(np.float32)
    g = (rng.standard_normal(n) * 0.02).astype(np.float32)
    anchor = (th + rng.standard_normal(n).astype(np.float32) * np.float32(1e-3)).astype(np.float32)
    mom = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    d = [torch.from_numpy(x.copy()).cuda() for x in (th, g, m, v, anchor, mom)]
    lib.pier_norm_ws_bytes.restype = C.c_size_t
    ws = torch.zeros(int(lib.pier_norm_ws_bytes()), dtype=torch.uint8, device="cuda")
    assert lib.pier_grad_sqnorm_f32(vp(d[1]), C.c_int64(n), C.c_double(1.0), vp(ws), stream()) == 0
    hp = PierAdamW(3e-3, 0.9, 0.999, 1e-8, 0.1, 1)
    assert lib.pier_adamw_f32(vp(d[0]), vp(d[1]), vp(d[2]), vp(d[3]), C.c_int64(n), C.byref(hp), vp(ws),
                              stream()) == 0
    rc = lib.pier_outer_update_f32(vp(d[0]), vp(d[4]), vp(d[5]), vp(d[0]), C.c_int64(n), C.c_double(1.1),
                                   C.c_double(0.9), C.c_int32(1), stream())
    assert rc == 0
    torch.cuda.synchronize()
    clip = PierClip.from_buffer_copy(ws[:C.sizeof(PierClip)].cpu().numpy().tobytes())
    assert clip.clipped == 1 and abs(clip.norm - float(np.linalg.norm(g.astype(np.float64)))) < 1e-5
    gc = g * np.float32(clip.scale)
    t1, m1, v1, _ = O.adamw(th, gc, m, v, 0, 3e-3)
    t2, mo2 = O.outer_anchor_form(t1, anchor, mom, 1.1, 0.9)
    assert same(d[0].cpu().numpy(), t2) and same(d[5].cpu().numpy(), mo2) and same(d[4].cpu().numpy(), t2)
    assert same(d[2].cpu().numpy(), m1) and same(d[3].cpu().numpy(), v1)


def test_raw_abi_error_codes_and_messages(lib):
    lib.pier_last_error.restype = C.c_char_p
    hp = PierAdamW(1e-3, 0.9, 0.999, 1e-8, 0.1, 0)   # step 0 is invalid (state.step + 1 >= 1)
    x = torch.zeros(8, device="cuda")
    rc = lib.pier_adamw_f32(vp(x), vp(x), vp(x), vp(x), C.c_int64(8), C.byref(hp), None, stream())
    assert rc == -1 and b"step" in lib.pier_last_error()
    assert lib.pier_outer_update_f32(vp(x), vp(x), vp(x), vp(x), C.c_int64(8), C.c_double(1.0),
                                     C.c_double(0.9), C.c_int32(0), stream()) == -1   # divisor 0
    # offload protocol (driver.py:136-146): double park / fetch before park -> PIER_EPROTOCOL (-4)
    off = C.c_void_p()
    assert lib.pier_offload_create(C.c_int32(1), C.c_size_t(32), C.byref(off)) == 0
    assert lib.pier_offload_fetch(off, C.c_int32(0), vp(x), C.c_size_t(32), stream()) == -4
    assert lib.pier_offload_park(off, C.c_int32(0), vp(x), C.c_size_t(32), stream()) == 0
    assert lib.pier_offload_park(off, C.c_int32(0), vp(x), C.c_size_t(32), stream()) == -4
    assert b"stored twice" in lib.pier_last_error()
    assert lib.pier_offload_fetch(off, C.c_int32(0), vp(x), C.c_size_t(32), stream()) == 0
    assert lib.pier_offload_sync(off) == 0
    assert lib.pier_offload_destroy(off) == 0


def test_launch_counter_counts_kernels(lib):
    lib.pier_launch_count.restype = C.c_ulonglong
    x = torch.zeros(1 << 20, device="cuda")
    before = lib.pier_launch_count()
    for _ in range(3):
        assert lib.pier_pseudograd_f32(vp(x), vp(x), vp(x), C.c_int64(x.numel()), stream()) == 0
    assert lib.pier_launch_count() - before == 3


def test_raw_abi_virtual_group_round(lib):
    """A C/C++ host's view of several groups on one device: pier_vgroup_create hands
    out one communicator per rank; each rank's host thread maps its buffers
    (pier_comm_alloc_shared, collective) and calls the persistent round
    (pier_round_fused_f32) -- one cooperative launch for both ranks -- with raw
    pointers; the result is the oracle's clip + AdamW + left-fold mean + outer step."""
    import threading

    P2 = 2
    n_pad, B = 8192, 1024
    comms = (C.c_void_p * P2)()
    assert lib.pier_vgroup_create(P2, comms) == 0
    lib.pier_comm_is_virtual.argtypes = [C.c_void_p]
    lib.pier_vgroup_abort.argtypes = [C.c_void_p]
    assert all(lib.pier_comm_is_virtual(comms[r]) == 1 for r in range(P2))
    rng = np.random.default_rng(5)
    anchor = (rng.standard_normal(n_pad) * 0.02).astype(np.float32)
    thetas = [anchor + (rng.standard_normal(n_pad) * 1e-3).astype(np.float32) for _ in range(P2)]
    grads = [(rng.standard_normal(n_pad) * 1e-4).astype(np.float32) for _ in range(P2)]
    mom = (rng.standard_normal(n_pad) * 1e-3).astype(np.float32)
    out = [None] * P2
    errors = []
    lib.pier_norm_ws_bytes.restype = C.c_size_t
    lib.pier_comm_alloc_shared.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p), C.POINTER(C.c_int32)]
    lib.pier_round_fused_f32.argtypes = [C.c_void_p, C.c_int32] + [C.c_void_p] * 5 + [
        C.c_int64, C.c_int64, C.POINTER(PierAdamW), C.c_void_p, C.c_double, C.c_double, C.c_void_p]

    def shard(x, r):   # rank r's slice of every span (layout of csrc/pier_comm.cu)
        return np.concatenate([x[off + r * B: off + (r + 1) * B] for off in range(0, n_pad, P2 * B)])

    def rank(r):
        try:
            torch.cuda.set_device(0)
            ptr, bid = C.c_void_p(), C.c_int32()
            assert lib.pier_comm_alloc_shared(comms[r], n_pad * 4, C.byref(ptr), C.byref(bid)) == 0
            # the raw device pointer of the mapped buffer, viewed through __cuda_array_interface__
            cai = type("B", (), {"__cuda_array_interface__": {"shape": (n_pad,), "typestr": "<f4",
                                                               "data": (ptr.value, False), "version": 3}})()
            theta = torch.as_tensor(cai, device="cuda")
            theta.copy_(torch.from_numpy(thetas[r]).cuda())
            g = torch.from_numpy(grads[r]).cuda()
            m, v = torch.zeros(n_pad, device="cuda"), torch.zeros(n_pad, device="cuda")
            an, mo = torch.from_numpy(shard(anchor, r)).cuda(), torch.from_numpy(shard(mom, r)).cuda()
            ws = torch.zeros(int(lib.pier_norm_ws_bytes()), dtype=torch.uint8, device="cuda")
            assert lib.pier_grad_sqnorm_f32(vp(g), C.c_int64(n_pad), C.c_double(1.0), vp(ws), stream()) == 0
            hp = PierAdamW(3e-3, 0.9, 0.999, 1e-8, 0.1, 1)
            assert lib.pier_round_fused_f32(comms[r], bid.value, vp(g), vp(m), vp(v), vp(an), vp(mo), n_pad, B,
                                            C.byref(hp), vp(ws), 1.1, 0.9, stream()) == 0
            torch.cuda.synchronize()
            out[r] = (theta.cpu().numpy(), an.cpu().numpy(), mo.cpu().numpy())
        except BaseException as exc:   # noqa: BLE001
            errors.append(exc)
            lib.pier_vgroup_abort(C.c_void_p(comms[r]))

    th = [threading.Thread(target=rank, args=(r,)) for r in range(P2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    new = [O.adamw(thetas[r], grads[r], np.zeros(n_pad, np.float32), np.zeros(n_pad, np.float32), 0, 3e-3)[0]
           for r in range(P2)]
    want, want_mo = O.outer_anchor_form(O.mean_left_fold(new), anchor, mom, 1.1, 0.9)
    for r in range(P2):
        assert same(out[r][0], want)
        assert same(out[r][1], shard(want, r)) and same(out[r][2], shard(want_mo, r))
    for r in range(P2):
        assert lib.pier_comm_destroy(C.c_void_p(comms[r])) == 0


def test_raw_abi_virtual_group_lazy_step(lib):
    """The sharded lazy-phase step through raw ctypes (driver.py:380-399): three
    virtual ranks, each with NVLink-mapped theta / grad / m / v buffers, call
    pier_lazy_step_p2p_f32 (reduce-scatter + norm of the mean, AdamW on the rank's
    third, all-gather of theta) and then pier_gather_p2p_f32 on m and v; every rank
    ends with the oracle's mean -> clip -> AdamW, bitwise, and the same clip record."""
    import threading

    P3 = 3
    n_pad = 3 * 4096 + 12          # a multiple of 4 * 3 but not of 8 * 3: the 128-bit path
    comms = (C.c_void_p * P3)()
    assert lib.pier_vgroup_create(P3, comms) == 0
    lib.pier_vgroup_abort.argtypes = [C.c_void_p]
    lib.pier_norm_ws_bytes.restype = C.c_size_t
    lib.pier_comm_alloc_shared.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p), C.POINTER(C.c_int32)]
    lib.pier_lazy_step_p2p_f32.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64,
                                           C.c_int64, C.POINTER(PierAdamW), C.c_double, C.c_void_p, C.c_void_p]
    lib.pier_gather_p2p_f32.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_void_p]
    B = 1024   # shard = slice of every span of 3 * 1024 elements; the last span 12 elements (4 per rank)
    rng = np.random.default_rng(8)
    theta0 = (rng.standard_normal(n_pad) * 0.02).astype(np.float32)
    m0 = (rng.standard_normal(n_pad) * 1e-4).astype(np.float32)
    v0 = (m0 * m0 + np.float32(1e-12)).astype(np.float32)
    grads = [rng.standard_normal(n_pad).astype(np.float32) for _ in range(P3)]   # |mean| >> 1: clipped
    out, errors = [None] * P3, []

    guard = 1024   # sentinel tail behind every buffer: the kernels must never touch it

    def mapped(comm):
        ptr, bid = C.c_void_p(), C.c_int32()
        assert lib.pier_comm_alloc_shared(comm, (n_pad + guard) * 4, C.byref(ptr), C.byref(bid)) == 0
        cai = type("B", (), {"__cuda_array_interface__": {"shape": (n_pad + guard,), "typestr": "<f4",
                                                           "data": (ptr.value, False), "version": 3}})()
        full = torch.as_tensor(cai, device="cuda")
        full[n_pad:].fill_(-7.25)
        return full[:n_pad], bid.value, full

    def rank(r):
        try:
            torch.cuda.set_device(0)
            (th, tid, thf), (g, gid, gf), (m, mid, mf), (v, vid, vf) = (mapped(comms[r]) for _ in range(4))
            for buf, src in ((th, theta0), (g, grads[r]), (m, m0), (v, v0)):
                buf.copy_(torch.from_numpy(src).cuda())
            ws = torch.zeros(int(lib.pier_norm_ws_bytes()), dtype=torch.uint8, device="cuda")
            hp = PierAdamW(3e-3, 0.9, 0.999, 1e-8, 0.1, 11)
            assert lib.pier_lazy_step_p2p_f32(comms[r], tid, gid, vp(m), vp(v), n_pad, B, C.byref(hp), 1.0,
                                              vp(ws), stream()) == 0
            assert lib.pier_gather_p2p_f32(comms[r], mid, n_pad, B, stream()) == 0
            assert lib.pier_gather_p2p_f32(comms[r], vid, n_pad, B, stream()) == 0
            torch.cuda.synchronize()
            rec = PierClip.from_buffer_copy(ws[:C.sizeof(PierClip)].cpu().numpy().tobytes())
            tails_intact = all(bool(torch.all(f[n_pad:] == -7.25)) for f in (thf, gf, mf, vf))
            out[r] = (th.cpu().numpy(), m.cpu().numpy(), v.cpu().numpy(), rec.clipped, rec.scale, rec.sqnorm,
                      tails_intact)
        except BaseException as exc:   # noqa: BLE001
            errors.append(exc)
            lib.pier_vgroup_abort(C.c_void_p(comms[r]))

    th = [threading.Thread(target=rank, args=(r,)) for r in range(P3)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    gm = O.mean_left_fold(grads)
    assert len({o[5] for o in out}) == 1 and all(o[3] == 1 for o in out)   # one clip record, clipped
    want = O.adamw(theta0, gm * np.float32(out[0][4]), m0, v0, 10, 3e-3)
    for r in range(P3):
        assert same(out[r][0], want[0]) and same(out[r][1], want[1]) and same(out[r][2], want[2])
        assert out[r][6], "a kernel wrote past n_padded"
    for r in range(P3):
        assert lib.pier_comm_destroy(C.c_void_p(comms[r])) == 0


def _bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (round to nearest even) -> fp32, exactly."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return (((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16).astype(np.uint32).view(np.float32)


def test_raw_abi_virtual_group_lazy_step_bf16(lib):
    """The 7B recipe's sharded lazy step through raw ctypes: bf16 gradients reduce-scattered
    (fp32 left fold, one RNE rounding), AdamW on each rank's third of the fp32 master, the
    RNE bf16 of the new master in every rank's live params; then the master / m / v
    gathered.  Bitwise vs the oracle; sentinel tails untouched."""
    import threading

    P3, guard = 3, 1024
    n_pad = 3 * 8 * 512
    comms = (C.c_void_p * P3)()
    assert lib.pier_vgroup_create(P3, comms) == 0
    lib.pier_vgroup_abort.argtypes = [C.c_void_p]
    lib.pier_norm_ws_bytes.restype = C.c_size_t
    lib.pier_comm_alloc_shared.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p), C.POINTER(C.c_int32)]
    lib.pier_lazy_step_p2p_bf16.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                            C.c_int64, C.c_int64, C.POINTER(PierAdamW), C.c_double, C.c_void_p,
                                            C.c_void_p]
    lib.pier_gather_p2p_f32.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_void_p]
    B = 0      # one span: the contiguous thirds
    rng = np.random.default_rng(21)
    master0 = (rng.standard_normal(n_pad) * 0.02).astype(np.float32)
    grads = [_bf16_round(rng.standard_normal(n_pad).astype(np.float32)) for _ in range(P3)]
    out, errors = [None] * P3, []

    def mapped(comm, n32, dtype):   # n32 fp32 words + a sentinel tail, viewed as dtype
        ptr, bid = C.c_void_p(), C.c_int32()
        assert lib.pier_comm_alloc_shared(comm, (n32 + guard) * 4, C.byref(ptr), C.byref(bid)) == 0
        cai = type("B", (), {"__cuda_array_interface__": {"shape": (n32 + guard,), "typestr": "<f4",
                                                           "data": (ptr.value, False), "version": 3}})()
        full = torch.as_tensor(cai, device="cuda")
        full[n32:].fill_(-7.25)
        return full[:n32].view(dtype), bid.value, full, n32

    def rank(r):
        try:
            torch.cuda.set_device(0)
            ma, mid, maf, _ = mapped(comms[r], n_pad, torch.float32)
            lv, lid, lvf, _ = mapped(comms[r], n_pad // 2, torch.bfloat16)
            g, gid, gf, _ = mapped(comms[r], n_pad // 2, torch.bfloat16)
            m, m_id, mf, _ = mapped(comms[r], n_pad, torch.float32)
            v, v_id, vf, _ = mapped(comms[r], n_pad, torch.float32)
            ma.copy_(torch.from_numpy(master0).cuda())
            g.copy_(torch.from_numpy(grads[r]).cuda().to(torch.bfloat16))
            m.zero_()
            v.zero_()
            ws = torch.zeros(int(lib.pier_norm_ws_bytes()), dtype=torch.uint8, device="cuda")
            hp = PierAdamW(3e-3, 0.9, 0.999, 1e-8, 0.1, 1)
            assert lib.pier_lazy_step_p2p_bf16(comms[r], mid, lid, gid, vp(m), vp(v), n_pad, B, C.byref(hp), 1.0,
                                               vp(ws), stream()) == 0
            for bid in (mid, m_id, v_id):
                assert lib.pier_gather_p2p_f32(comms[r], bid, n_pad, B, stream()) == 0
            torch.cuda.synchronize()
            rec = PierClip.from_buffer_copy(ws[:C.sizeof(PierClip)].cpu().numpy().tobytes())
            tails = [(maf, n_pad), (lvf, n_pad // 2), (gf, n_pad // 2), (mf, n_pad), (vf, n_pad)]
            out[r] = (ma.cpu().numpy(), lv.float().cpu().numpy(), m.cpu().numpy(), v.cpu().numpy(),
                      rec.clipped, rec.scale, all(bool(torch.all(f[k:] == -7.25)) for f, k in tails))
        except BaseException as exc:   # noqa: BLE001
            errors.append(exc)
            lib.pier_vgroup_abort(C.c_void_p(comms[r]))

    th = [threading.Thread(target=rank, args=(r,)) for r in range(P3)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    gm = _bf16_round(O.mean_left_fold(grads))          # fp32 left fold of the bf16 values, one RNE rounding
    assert all(o[4] == 1 for o in out) and len({o[5] for o in out}) == 1
    want = O.adamw(master0, gm * np.float32(out[0][5]), np.zeros(n_pad, np.float32), np.zeros(n_pad, np.float32),
                   0, 3e-3)
    for r in range(P3):
        assert same(out[r][0], want[0]) and same(out[r][1], _bf16_round(want[0]))
        assert same(out[r][2], want[1]) and same(out[r][3], want[2])
        assert out[r][6], "a kernel wrote past n_padded"
    for r in range(P3):
        assert lib.pier_comm_destroy(C.c_void_p(comms[r])) == 0
