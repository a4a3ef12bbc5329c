"""Open-loop K-round parity at the SURVEY §8(d) sizes: N = 306,176 (tiny) and
124,439,808 (GPT-2 small), n = 1, 2, 4, 8 groups (one per rank; n > 1 as a
VirtualGroup on one GPU, the same kernels as n GPUs), T = 1000, r = 10,
lazy_fraction 0.1 -> 10 warmup folds + 90 outer steps crossing the mu
boundaries 150/200 and the lr boundaries 200/800 (driver.py:404-443).

* N = 306,176: the reference protocol (group params at boundary k =
  anchor + N(0, 1e-3^2) from default_rng([seed, 300, k, g])) against
  ``oracle.open_loop_run`` (pinned to the reference ENGINE by the golden
  open-loop fixtures), full vectors, bitwise.
* N = 124,439,808: per-element counter-based inputs (``oracle.hash_inputs``),
  generated on the GPU for every element; the oracle replays a strided sample
  of 124,815 elements through all 100 boundaries (the update is elementwise,
  so each sampled element's trajectory is exact), bitwise.
"""

import numpy as np
import pytest
import torch

from group_checks import bits_equal, torch_hash_values
from oracle import pier_oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2511_17849_b200")

SEED = 4


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _sched():
    return (P.ScheduleConfig(total_iters=1000, lazy_fraction=0.1, sync_interval=10),
            O.Sched(total_iters=1000, lazy_fraction=0.1, sync_interval=10))


def _run_groups(n, fn):
    if n == 1:
        return [fn(None)]
    with P.VirtualGroup(n) as vg:
        return vg.run(fn)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_open_loop_tiny_reference_protocol(n):
    N = 306_176
    sched, osch = _sched()
    theta0 = (np.random.default_rng(SEED).standard_normal(N) * 0.02).astype(np.float32)
    want_an, want_mo, evs = O.open_loop_run(osch, theta0, n, SEED)
    assert sum(e.kind == "fold" for e in evs) == 10 and sum(e.kind == "outer" for e in evs) == 90

    def fn(comm):
        dev = torch.device("cuda", torch.cuda.current_device())
        rank = comm.rank if comm else 0
        eng = P.PierEngine(N, sched, comm=comm, theta0=torch.from_numpy(theta0).to(dev), bucket_elems=1 << 14)
        k = 0
        for t in range(1, 1001):
            if not eng.is_boundary(t):
                continue
            anchor = eng.params().cpu().numpy()      # == the anchor before every boundary
            g = 0 if t <= sched.lazy_end else rank
            eng.theta[:N].copy_(torch.from_numpy(O.open_loop_inputs(SEED, k, g, anchor)).to(dev))
            k += 1
            eng.boundary(t)
        out = (eng.params().cpu().numpy(), eng.outer_momentum().cpu().numpy(),
               [(r.iteration, r.kind, r.mu, r.outer_lr) for r in eng.records])
        eng.close()
        return out

    for th, mo, recs in _run_groups(n, fn):
        assert [(e.t, e.kind, e.mu, e.lr) for e in evs] == recs
        assert bits_equal(th, want_an) and bits_equal(mo, want_mo)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_open_loop_gpt2_small_full_size(n):
    N = 124_439_808
    sched, osch = _sched()
    idx = np.arange(0, N, 997, dtype=np.int64)
    idx = np.unique(np.concatenate([idx, [N - 1]]))
    theta0_s = O.hash_values(O.hash_key(SEED, -1, 0), idx, O.THETA0_SCALE)
    want_an, want_mo, evs = O.open_loop_run(
        osch, theta0_s, n, SEED, inputs=lambda seed, k, g, anchor: O.hash_inputs(seed, k, g, anchor, idx))

    def fn(comm):
        dev = torch.device("cuda", torch.cuda.current_device())
        rank = comm.rank if comm else 0
        theta0 = torch_hash_values(O.hash_key(SEED, -1, 0), N, O.THETA0_SCALE, dev)
        assert bits_equal(theta0[torch.from_numpy(idx).to(dev)].cpu().numpy(), theta0_s)
        eng = P.PierEngine(N, sched, comm=comm, theta0=theta0, bucket_elems=1 << 22)
        del theta0
        k = 0
        for t in range(1, 1001):
            if not eng.is_boundary(t):
                continue
            g = 0 if t <= sched.lazy_end else rank
            # the params equal the anchor before every boundary: anchor + noise, one rounding
            eng.theta[:N].add_(torch_hash_values(O.hash_key(SEED, k, g), N, O.NOISE_SCALE, dev))
            k += 1
            eng.boundary(t)
        sel = torch.from_numpy(idx).to(dev)
        out = (eng.params()[sel].cpu().numpy(), eng.outer_momentum()[sel].cpu().numpy(), len(eng.records))
        eng.close()
        return out

    for th, mo, nrec in _run_groups(n, fn):
        assert nrec == 100
        assert bits_equal(th, want_an) and bits_equal(mo, want_mo)
