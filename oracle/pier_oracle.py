"""NumPy restatement of the Pier optimizer hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker the CUDA path is compared against and the CPU
baseline ``bench.py --impl reference`` times.  It is never imported by the
product package.  Every function cites the reference line it restates
(paths relative to ``/root/reference/pkg/src/pier``).  Pinned against the
reference's own outputs by ``tests/test_oracle_golden.py`` (fixtures written by
``tests/golden/make_golden.py``, which imports the reference).

Rounding model (why this is bitwise-comparable with the CUDA kernels): every
elementwise operation below is one IEEE-754 correctly-rounded NumPy ufunc in
the array dtype; Python-float scalars are first rounded to that dtype (NumPy 2
"weak scalar" promotion, which the reference relies on, e.g. ``optim.py:97``
multiplies a float32 array by the Python float ``beta1``).  The CUDA kernels
use the same operation order with ``__f*_rn`` intrinsics and no FMA
contraction, so they agree bit for bit except where a reduction order is
implementation-defined (``np.dot`` in the clip norm, the all-reduce order of
NCCL).
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# constants (optim.py:25-31, config.py:28-29)
# ---------------------------------------------------------------------------

LR_PLATEAU = 1.1          # optim.py:25
LR_COOLDOWN = 0.9         # optim.py:26
MU_TABLE = (0.9, 0.99, 0.95, 0.9)  # optim.py:27
FRAC_RAMP_START = 0.1     # optim.py:28
FRAC_RAMP_END = 0.2       # optim.py:29
FRAC_MU_MID = 0.15        # optim.py:30
FRAC_LATE = 0.8           # optim.py:31
DILOCO_LR = 0.7           # config.py:28
DILOCO_MU = 0.9           # config.py:29


def floor_frac(frac: float, total: int) -> int:
    """``optim.py:162-163``: schedule boundaries are floored products."""
    return int(math.floor(frac * total))


# ---------------------------------------------------------------------------
# schedules (optim.py:148-219)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Sched:
    total_iters: int = 3000
    lazy_fraction: float = 0.1
    sync_interval: int = 20
    inner_warmup_fraction: float = 0.02
    inner_lr_peak: float = 3e-3
    inner_lr_min: float = 3e-4
    decay_iters: int | None = None

    @property
    def lazy_end(self) -> int:                      # optim.py:148-151
        return floor_frac(self.lazy_fraction, self.total_iters)

    @property
    def warmup_iters(self) -> int:                  # optim.py:153-155
        return floor_frac(self.inner_warmup_fraction, self.total_iters)

    @property
    def decay_horizon(self) -> int:                 # optim.py:157-159
        return self.total_iters if self.decay_iters is None else self.decay_iters


def inner_lr(t: int, s: Sched) -> float:
    """``optim.py:166-178``: linear warmup, cosine decay, clamp at the floor."""
    if t < 0:
        raise ValueError("negative iteration")
    w, hi, lo = s.warmup_iters, s.inner_lr_peak, s.inner_lr_min
    if w > 0 and t <= w:
        return hi * (t / w)
    h = s.decay_horizon
    if t >= h:
        return lo
    x = (t - w) / (h - w)
    return lo + 0.5 * (hi - lo) * (1.0 + math.cos(math.pi * x))


def outer_lr(t: int, s: Sched) -> float:
    """``optim.py:181-202``: 0->1 ramp on [0.1T, 0.2T), 1.1 plateau, 0.9 from 0.8T."""
    T = s.total_iters
    a, b, c = floor_frac(FRAC_RAMP_START, T), floor_frac(FRAC_RAMP_END, T), floor_frac(FRAC_LATE, T)
    if t < a or t > T:
        raise ValueError(f"outer_lr undefined at t={t}")
    if t < b:
        return (t - a) / (b - a)
    return LR_PLATEAU if t < c else LR_COOLDOWN


def momentum_mu(t: int, T: int) -> float:
    """``optim.py:205-219``: 0.9 | 0.99 | 0.95 | 0.9 split at 0.1T, 0.15T, 0.2T."""
    if t < 0:
        raise ValueError("negative iteration")
    for frac, mu in ((FRAC_RAMP_START, MU_TABLE[0]), (FRAC_MU_MID, MU_TABLE[1]),
                     (FRAC_RAMP_END, MU_TABLE[2])):
        if t < floor_frac(frac, T):
            return mu
    return MU_TABLE[3]


# ---------------------------------------------------------------------------
# inner step (optim.py:70-103)
# ---------------------------------------------------------------------------

def clip_global_norm(g: np.ndarray, max_norm: float):
    """``optim.py:70-79``.  The dot goes through BLAS (order implementation-defined)."""
    nrm = float(np.sqrt(np.dot(g, g)))
    if nrm > max_norm:
        return g * g.dtype.type(max_norm / nrm), nrm
    return g, nrm


def clip_scale(norm: float, max_norm: float, dtype) -> float:
    """Scale factor ``optim.py:77-78`` applies (1 when no clipping happens)."""
    return float(np.dtype(dtype).type(max_norm / norm)) if norm > max_norm else 1.0


def adamw(theta, g, m, v, step, lr, beta1=0.9, beta2=0.999, eps=1e-8, wd=0.1):
    """``optim.py:82-103`` on arrays; returns ``(theta', m', v', step+1)``.

    Op order (each op rounded in ``theta.dtype``): decay ``theta*c`` (:96);
    ``m = b1*m + c1*g`` (:97); ``v = b2*v + c2*(g*g)`` (:98); ``mh = m/bc1`` (:99);
    ``den = sqrt(v/bc2) + eps`` (:100-101); ``theta -= (lr*mh)/den`` (:102).
    """
    s = step + 1
    f = theta.dtype.type
    out = theta * f(1.0 - lr * wd)
    m2 = f(beta1) * m + f(1.0 - beta1) * g
    v2 = f(beta2) * v + f(1.0 - beta2) * (g * g)
    mh = m2 / f(1.0 - beta1 ** s)
    den = np.sqrt(v2 / f(1.0 - beta2 ** s))
    den += f(eps)
    out -= f(lr) * mh / den
    return out, m2, v2, s


# ---------------------------------------------------------------------------
# outer step (optim.py:226-276) and the driver's use of it (driver.py:404-443)
# ---------------------------------------------------------------------------

def fold(M: np.ndarray, d: np.ndarray, mu: float) -> np.ndarray:
    """``optim.py:243-245``: ``(mu*M) + d``, two roundings, fixed order."""
    return (M.dtype.type(mu) * M) + d


def outer_anchor_form(avg, anchor, M, lr, mu):
    """``driver.py:434-438`` + ``optim.py:269-276`` with ``anchor=avg``.

    Returns ``(theta_new, M_new)``; the caller re-anchors to ``theta_new``.
    """
    d = avg - anchor                               # driver.py:434
    M2 = fold(M, d, mu)                            # optim.py:270
    upd = d.dtype.type(lr) * fold(M2, d, mu)       # optim.py:271
    return avg + (upd - d), M2                     # optim.py:275


def outer_snapshot_form(snapshot, M, d, lr, mu):
    """``optim.py:272-273``: the ``anchor=None`` branch."""
    M2 = fold(M, d, mu)
    return snapshot + d.dtype.type(lr) * fold(M2, d, mu), M2


def warmup_fold(theta, anchor, M, mu):
    """``driver.py:412-420``: ``M = fold(M, theta-anchor, mu)``; anchor <- theta."""
    return fold(M, theta - anchor, mu), theta.copy()


# ---------------------------------------------------------------------------
# collectives and layout (topology.py:104-160)
# ---------------------------------------------------------------------------

def mean_left_fold(arrays) -> np.ndarray:
    """``topology.py:104-122``: ascending left fold, then divide by n."""
    if len(arrays) == 0:
        raise ValueError("need at least one participant")
    acc = np.array(arrays[0], copy=True)
    for a in arrays[1:]:
        if a.shape != acc.shape or a.dtype != acc.dtype:
            raise ValueError("participants disagree on shape/dtype")
        acc += a
    acc /= acc.dtype.type(len(arrays))
    return acc


def ring_bytes(payload: float, n: int) -> float:
    """``topology.py:135-139``."""
    return 0.0 if n <= 1 else 2.0 * payload * (n - 1) / n


def shard_ranges(n_params: int, k: int):
    """``topology.py:146-160``: near-equal contiguous ranges, remainder first."""
    q, r = divmod(n_params, k)
    out, lo = [], 0
    for i in range(k):
        hi = lo + q + (i < r)
        out.append((lo, hi))
        lo = hi
    return out


# ---------------------------------------------------------------------------
# boundary schedule of the engine (driver.py:333-348, 404-443)
# ---------------------------------------------------------------------------

@dataclass
class BoundaryEvent:
    t: int
    kind: str            # "fold" | "anchor" (diloco lazy re-anchor) | "outer"
    mu: float | None
    lr: float | None


def boundary_events(s: Sched, mode: str = "pier", lr_fixed=None, mu_fixed=None):
    """Every boundary of a run, as ``driver.py:404-443`` would visit them.

    ``mode`` in {"pier", "diloco_baseline", "adamw_baseline"}; DiLoCo defaults
    to the fixed coefficients ``config.py:123-132``.
    """
    if mode == "adamw_baseline":
        return []
    if mode == "diloco_baseline":
        lr_fixed = DILOCO_LR if lr_fixed is None else lr_fixed
        mu_fixed = DILOCO_MU if mu_fixed is None else mu_fixed
    ev = []
    for t in range(s.sync_interval, s.total_iters + 1, s.sync_interval):
        mu = mu_fixed if mu_fixed is not None else momentum_mu(t, s.total_iters)
        if t <= s.lazy_end:
            ev.append(BoundaryEvent(t, "fold" if mode == "pier" else "anchor",
                                    mu if mode == "pier" else None, None))
        else:
            lr = lr_fixed if lr_fixed is not None else outer_lr(t, s)
            ev.append(BoundaryEvent(t, "outer", mu, lr))
    return ev


def open_loop_inputs(seed: int, k: int, g: int, anchor: np.ndarray, sigma=1e-3):
    """Per-boundary group params ``anchor + N(0, sigma^2)`` from
    ``default_rng([seed, 300, k, g])`` (SURVEY.md §8d open-loop protocol)."""
    rng = np.random.default_rng([seed, 300, k, g])
    return anchor + anchor.dtype.type(sigma) * rng.standard_normal(anchor.shape[0], dtype=anchor.dtype)


# Counter-based per-element inputs for open-loop runs at full model size: the
# value at element i depends only on (seed, k, g, i), so the GPU test generates
# a whole group's params on the device while the oracle replays any subset of
# elements on the CPU, bit for bit (splitmix64 finalizer; a 24-bit integer
# scaled by one fp32 product, then added to the anchor with one rounding).
_SM_C1, _SM_C2, _SM_GOLD = 0xBF58476D1CE4E5B9, 0x94D049BB133111EB, 0x9E3779B97F4A7C15
NOISE_SCALE = np.float32(1e-3 * math.sqrt(3.0) / 2 ** 23)   # uniform, std 1e-3
THETA0_SCALE = np.float32(0.02 * math.sqrt(3.0) / 2 ** 23)  # uniform, std 0.02


def hash_key(seed: int, k: int, g: int) -> int:
    """Stream key of (seed, boundary k, group g); k = -1 is the initial params."""
    return ((seed * 1_000_003 + (k + 1)) * 64 + g + 1) & 0xFFFFFFFFFFFFFFFF


def hash_uniform24(key: int, idx: np.ndarray) -> np.ndarray:
    """splitmix64(key * GOLD + i) >> 40, as int64 in [0, 2^24)."""
    with np.errstate(over="ignore"):
        z = np.uint64((key * _SM_GOLD) & 0xFFFFFFFFFFFFFFFF) + idx.astype(np.uint64)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_SM_C1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_SM_C2)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(40)).astype(np.int64)


def hash_values(key: int, idx: np.ndarray, scale: np.float32) -> np.ndarray:
    """f32(u - 2^23) * scale: exact integer conversion, one rounding."""
    return (hash_uniform24(key, idx) - (1 << 23)).astype(np.float32) * scale


def hash_inputs(seed: int, k: int, g: int, anchor: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """``anchor + noise`` for the elements ``idx`` (anchor holds those elements)."""
    return anchor + hash_values(hash_key(seed, k, g), idx, NOISE_SCALE)


def open_loop_run(s: Sched, theta0: np.ndarray, groups: int, seed: int, mode="pier",
                  stop_after: int | None = None, dp: int = 1, inputs=None):
    """Drive only the boundary stage (no inner model) through a whole schedule.

    At every boundary k each group's params are replaced by
    :func:`open_loop_inputs` (or ``inputs(seed, k, g, anchor)``); folds use
    group 0 (replicas agree in the lazy phase, ``driver.py:412``), outer steps
    average all groups (``driver.py:428-440``).  Returns ``(anchor, M, events)``.
    The update is elementwise, so a run over a subset of elements (with
    per-element ``inputs``) equals those elements of the full run.
    """
    inputs = open_loop_inputs if inputs is None else inputs
    anchor = theta0.copy()
    M = np.zeros_like(theta0)
    evs = boundary_events(s, mode)
    done = []
    for k, e in enumerate(evs):
        if stop_after is not None and e.t > stop_after:
            break
        if e.kind == "fold":
            th = inputs(seed, k, 0, anchor)
            M, anchor = warmup_fold(th, anchor, M, e.mu)
        elif e.kind == "anchor":
            anchor = inputs(seed, k, 0, anchor)
        else:
            # every replica joins in ascending rank order; dp replicas of a group
            # hold identical params (driver.py:426-429)
            ths = [inputs(seed, k, gi, anchor) for gi in range(groups) for _ in range(dp)]
            avg = mean_left_fold(ths)
            anchor, M = outer_anchor_form(avg, anchor, M, e.lr, e.mu)
        done.append(e)
    return anchor, M, done


# ---------------------------------------------------------------------------
# host offload bookkeeping (driver.py:115-164, 318-329)
# ---------------------------------------------------------------------------

class ProtocolViolation(RuntimeError):
    pass


@dataclass
class HostLedger:
    """``driver.py:115-164`` semantics: copy in, surrender out, counters."""
    enabled: bool
    live: dict = field(default_factory=dict)
    to_host: float = 0.0
    from_host: float = 0.0
    stores: int = 0
    loads: int = 0

    def store(self, key, arr):
        if not self.enabled:
            return
        if key in self.live:
            raise ProtocolViolation(f"{key} stored twice")
        self.live[key] = np.array(arr, copy=True)
        self.to_host += arr.nbytes
        self.stores += 1

    def load(self, key):
        if not self.enabled:
            raise ProtocolViolation("offload disabled")
        if key not in self.live:
            raise ProtocolViolation(f"{key} not stored")
        a = self.live.pop(key)
        self.from_host += a.nbytes
        self.loads += 1
        return a


# ---------------------------------------------------------------------------
# chunked multi-threaded application (for the CPU baseline leg only)
# ---------------------------------------------------------------------------

def chunked(fn, arrays, threads: int, chunk: int = 1 << 22):
    """Apply an elementwise oracle ``fn(*slices) -> tuple`` over chunks on a
    thread pool (NumPy releases the GIL in ufunc loops).  Elementwise ops are
    position-independent, so results equal the unchunked call bit for bit."""
    n = arrays[0].shape[0]
    spans = [(a, min(a + chunk, n)) for a in range(0, n, chunk)]

    def one(span):
        a, b = span
        return span, fn(*[x[a:b] for x in arrays])

    outs = None
    with ThreadPoolExecutor(max_workers=threads) as ex:
        for (a, b), res in ex.map(one, spans):
            res = res if isinstance(res, tuple) else (res,)
            if outs is None:
                outs = [np.empty(n, dtype=r.dtype) for r in res]
            for o, r in zip(outs, res):
                o[a:b] = r
    return tuple(outs)
