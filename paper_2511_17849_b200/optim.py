"""Drop-in for ``pier.optim`` (optim.py:34-276) backed by sm_100a kernels.

Same names, arguments, defaults, validation errors and value semantics as the
reference: the pure functions never mutate their inputs and return new
arrays (``optim.py:9-11``).  Arrays are torch CUDA tensors or NumPy arrays
(NumPy in -> NumPy out, computed on the GPU).  For the hot loop, the
in-place variants with a trailing underscore operate on caller-owned CUDA
tensors with no allocation and no host synchronisation.

The schedules (``inner_lr``, ``outer_lr``, ``momentum_mu``) are scalar host
control logic and are restated here exactly (integer boundaries via
``floor(frac * T)``, ``optim.py:162-163``).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev
from ._lib import PierAdamW, PierClip, check, lib
from .errors import ConfigError

OUTER_LR_HIGH = 1.1                 # optim.py:25
OUTER_LR_LATE = 0.9                 # optim.py:26
MU_STAGES = (0.9, 0.99, 0.95, 0.9)  # optim.py:27
_RAMP_START_FRAC = 0.1
_RAMP_END_FRAC = 0.2
_MU_MID_FRAC = 0.15
_LATE_FRAC = 0.8


# ---------------------------------------------------------------------------
# configs and state (optim.py:34-67)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class AdamWConfig:
    """Inner AdamW hyper-parameters; validation as ``optim.py:44-54``."""

    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.1
    clip_norm: float = 1.0

    def __post_init__(self):
        for name in ("beta1", "beta2"):
            b = getattr(self, name)
            if not 0.0 <= b < 1.0:
                raise ConfigError(f"{name} must lie in [0, 1), got {b}")
        if self.eps <= 0.0:
            raise ConfigError(f"eps must be positive, got {self.eps}")
        if self.weight_decay < 0.0:
            raise ConfigError(f"weight_decay must be non-negative, got {self.weight_decay}")
        if self.clip_norm <= 0.0:
            raise ConfigError(f"clip_norm must be positive, got {self.clip_norm}")

    def hyper(self, lr: float, step: int) -> PierAdamW:
        return PierAdamW(lr=float(lr), beta1=self.beta1, beta2=self.beta2, eps=self.eps,
                         weight_decay=self.weight_decay, step=int(step))


def _np_or_torch_dtype(dtype):
    if isinstance(dtype, torch.dtype):
        return dtype
    return {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}[np.dtype(dtype)]


@dataclass
class AdamWState:
    """First/second moments plus the completed step count (``optim.py:57-67``)."""

    m: object
    v: object
    step: int = 0

    @classmethod
    def initial(cls, num_params: int, dtype=np.float64, device=None) -> "AdamWState":
        dev = device if device is not None else _dev.require_cuda()
        dt = _np_or_torch_dtype(dtype)
        return cls(m=torch.zeros(num_params, dtype=dt, device=dev),
                   v=torch.zeros(num_params, dtype=dt, device=dev))


@dataclass(frozen=True)
class ScheduleConfig:
    """Run-length bookkeeping; fields, defaults and checks of ``optim.py:110-159``."""

    total_iters: int = 3000
    lazy_fraction: float = 0.1
    sync_interval: int = 20
    inner_warmup_fraction: float = 0.02
    inner_lr_peak: float = 3e-3
    inner_lr_min: float = 3e-4
    decay_iters: int | None = None

    def __post_init__(self):
        if self.total_iters < 1:
            raise ConfigError(f"total_iters must be positive, got {self.total_iters}")
        if not 0.0 <= self.lazy_fraction < 1.0:
            raise ConfigError(f"lazy_fraction must lie in [0, 1), got {self.lazy_fraction}")
        if self.sync_interval < 1:
            raise ConfigError(f"sync_interval must be a positive integer, got {self.sync_interval}")
        if self.sync_interval >= self.total_iters:
            raise ConfigError(f"sync_interval ({self.sync_interval}) must be smaller than "
                              f"total_iters ({self.total_iters})")
        if not 0.0 <= self.inner_warmup_fraction < 1.0:
            raise ConfigError(f"inner_warmup_fraction must lie in [0, 1), got {self.inner_warmup_fraction}")
        if self.inner_lr_peak <= 0.0 or self.inner_lr_min < 0.0:
            raise ConfigError(f"inner_lr_peak/inner_lr_min must be positive, got "
                              f"{self.inner_lr_peak}/{self.inner_lr_min}")
        if self.inner_lr_min > self.inner_lr_peak:
            raise ConfigError(f"inner_lr_min ({self.inner_lr_min}) must not exceed "
                              f"inner_lr_peak ({self.inner_lr_peak})")
        if self.decay_iters is not None and self.decay_iters < 1:
            raise ConfigError(f"decay_iters must be positive, got {self.decay_iters}")

    @property
    def lazy_end(self) -> int:
        return _boundary(self.lazy_fraction, self.total_iters)

    @property
    def warmup_iters(self) -> int:
        return _boundary(self.inner_warmup_fraction, self.total_iters)

    @property
    def decay_horizon(self) -> int:
        return self.total_iters if self.decay_iters is None else self.decay_iters


def _boundary(frac: float, total: int) -> int:
    return int(math.floor(frac * total))


# ---------------------------------------------------------------------------
# schedules (optim.py:166-219) -- exact host restatement
# ---------------------------------------------------------------------------

def inner_lr(t: int, sched: ScheduleConfig) -> float:
    """Linear warmup to the peak, cosine decay to the floor (``optim.py:166-178``)."""
    if t < 0:
        raise ValueError(f"iteration must be non-negative, got {t}")
    w = sched.warmup_iters
    if w > 0 and t <= w:
        return sched.inner_lr_peak * (t / w)
    h = sched.decay_horizon
    if t >= h:
        return sched.inner_lr_min
    frac = (t - w) / (h - w)
    lo, hi = sched.inner_lr_min, sched.inner_lr_peak
    return lo + 0.5 * (hi - lo) * (1.0 + math.cos(math.pi * frac))


def outer_lr(t: int, sched: ScheduleConfig) -> float:
    """0 -> 1 ramp over [0.1T, 0.2T), 1.1 plateau, 0.9 from 0.8T (``optim.py:181-202``)."""
    total = sched.total_iters
    start, end, late = (_boundary(f, total) for f in (_RAMP_START_FRAC, _RAMP_END_FRAC, _LATE_FRAC))
    if t < start:
        raise ValueError(f"outer_lr is undefined before iteration {start} (got t={t}); "
                         "the synchronous phase has no outer updates")
    if t > total:
        raise ValueError(f"outer_lr is undefined past total_iters={total} (got t={t})")
    if t < end:
        return (t - start) / (end - start)
    return OUTER_LR_HIGH if t < late else OUTER_LR_LATE


def momentum_mu(t: int, total_iters: int) -> float:
    """0.9 -> 0.99 -> 0.95 -> 0.9 at 0.1T, 0.15T, 0.2T (``optim.py:205-219``)."""
    if t < 0:
        raise ValueError(f"iteration must be non-negative, got {t}")
    if t < _boundary(_RAMP_START_FRAC, total_iters):
        return MU_STAGES[0]
    if t < _boundary(_MU_MID_FRAC, total_iters):
        return MU_STAGES[1]
    if t < _boundary(_RAMP_END_FRAC, total_iters):
        return MU_STAGES[2]
    return MU_STAGES[3]


# ---------------------------------------------------------------------------
# gradient norm / clip (optim.py:70-79)
# ---------------------------------------------------------------------------

_WS_BYTES = int(lib.pier_norm_ws_bytes())


def norm_workspace(device=None) -> torch.Tensor:
    """Zeroed device workspace for the norm kernel (reusable across launches)."""
    dev = device if device is not None else _dev.require_cuda()
    return torch.zeros(_WS_BYTES, dtype=torch.uint8, device=dev)


def read_clip(ws: torch.Tensor) -> PierClip:
    """Host copy of the PierClip record (synchronises the current stream)."""
    host = ws[: C.sizeof(PierClip)].cpu().numpy().tobytes()
    return PierClip.from_buffer_copy(host)


def grad_sqnorm_(grad: torch.Tensor, max_norm: float, ws: torch.Tensor) -> None:
    """Launch K4a: global norm + clip scale into ``ws`` (no host sync)."""
    fn = getattr(lib, f"pier_grad_sqnorm_{_dev.suffix(grad)}")
    check(fn(grad.data_ptr(), grad.numel(), float(max_norm), ws.data_ptr(), _dev.stream_ptr()),
          "grad_sqnorm")


def clip_global_norm(grad, max_norm: float):
    """``optim.py:70-79``: returns ``(clipped, norm)``; ``grad`` itself when within bounds."""
    g, is_np = _dev.to_device(grad)
    ws = norm_workspace(g.device)
    grad_sqnorm_(g, max_norm, ws)
    rec = read_clip(ws)
    if not rec.clipped:
        return grad, float(rec.norm)
    out = torch.empty_like(g)
    # grad * dtype(max_norm / norm): one rounding, scale read on the device (K4c)
    fn = getattr(lib, f"pier_apply_clip_{_dev.suffix(g)}")
    check(fn(g.data_ptr(), out.data_ptr(), g.numel(), ws.data_ptr(), _dev.stream_ptr()), "apply_clip")
    return _dev.back(out, is_np, np.shape(grad) if is_np else grad.shape), float(rec.norm)


# ---------------------------------------------------------------------------
# AdamW (optim.py:82-103)
# ---------------------------------------------------------------------------

def adamw_(theta: torch.Tensor, grad: torch.Tensor, m: torch.Tensor, v: torch.Tensor, step: int,
           lr: float, cfg: AdamWConfig, clip_ws: torch.Tensor | None = None) -> None:
    """In-place fused AdamW on CUDA tensors; ``step`` is the NEW count.

    With ``clip_ws`` (written by :func:`grad_sqnorm_` on the same stream) the
    reference's clip (``optim.py:77-78``) is applied to ``grad`` in flight.
    """
    n = _dev.same_shape(theta, grad, m, v)
    hp = cfg.hyper(lr, step)
    fn = getattr(lib, f"pier_adamw_{_dev.suffix(theta)}")
    check(fn(theta.data_ptr(), grad.data_ptr(), m.data_ptr(), v.data_ptr(), n, C.byref(hp),
             None if clip_ws is None else clip_ws.data_ptr(), _dev.stream_ptr()), "adamw")


def adamw_step(theta, grad, state: AdamWState, lr: float, cfg: AdamWConfig):
    """One AdamW update; returns ``(new_theta, new_state)`` (``optim.py:82-103``)."""
    th, is_np = _dev.to_device(theta)
    g, _ = _dev.to_device(grad, th.dtype)
    m, _ = _dev.to_device(state.m, th.dtype)
    v, _ = _dev.to_device(state.v, th.dtype)
    th, m, v = th.clone(), m.clone(), v.clone()
    step = state.step + 1
    adamw_(th, g, m, v, step, lr, cfg)
    shape = np.shape(theta) if is_np else theta.shape
    return _dev.back(th, is_np, shape), AdamWState(m=_dev.back(m, is_np), v=_dev.back(v, is_np), step=step)


def adamw_bf16_(master: torch.Tensor, theta_bf16: torch.Tensor, grad_bf16: torch.Tensor,
                m: torch.Tensor, v: torch.Tensor, step: int, lr: float, cfg: AdamWConfig,
                clip_ws: torch.Tensor | None = None) -> None:
    """bf16 live params / bf16 grads with fp32 master, m, v (7B config): the
    fp32 update of :func:`adamw_` plus the RNE bf16 refresh, one pass."""
    n = _dev.same_shape(master, m, v)
    if theta_bf16.numel() != n or grad_bf16.numel() != n or theta_bf16.dtype != torch.bfloat16 \
            or grad_bf16.dtype != torch.bfloat16 or master.dtype != torch.float32:
        raise ConfigError("adamw_bf16_: bf16 params/grads and fp32 master/m/v of one length")
    hp = cfg.hyper(lr, step)
    check(lib.pier_adamw_bf16_f32(master.data_ptr(), theta_bf16.data_ptr(), grad_bf16.data_ptr(),
                                  m.data_ptr(), v.data_ptr(), n, C.byref(hp),
                                  None if clip_ws is None else clip_ws.data_ptr(), _dev.stream_ptr()),
          "adamw_bf16")


def grad_sqnorm_bf16_(grad: torch.Tensor, max_norm: float, ws: torch.Tensor) -> None:
    check(lib.pier_grad_sqnorm_bf16(grad.data_ptr(), grad.numel(), float(max_norm), ws.data_ptr(),
                                    _dev.stream_ptr()), "grad_sqnorm_bf16")


class MultiTensorAdamW:
    """Fused multi-tensor AdamW over a list of torch params (one launch for the
    norm, one for the update), e.g. 580 GPT-2 XL tensors.  The chunk table is
    uploaded once at construction; grads are read from ``p.grad``."""

    def __init__(self, params, cfg: AdamWConfig | None = None):
        self.params = [p for p in params]
        if not self.params:
            raise ConfigError("MultiTensorAdamW needs at least one parameter")
        self.cfg = cfg or AdamWConfig()
        dt = self.params[0].dtype
        if dt not in (torch.float32, torch.float64) or any(p.dtype != dt for p in self.params):
            raise ConfigError("MultiTensorAdamW: all params float32 or all float64")
        for p in self.params:
            if not p.is_cuda or not p.is_contiguous():
                raise ConfigError("MultiTensorAdamW: params must be contiguous CUDA tensors")
        self.m = [torch.zeros_like(p) for p in self.params]
        self.v = [torch.zeros_like(p) for p in self.params]
        self.step_count = 0
        self.ws = norm_workspace(self.params[0].device)
        self._list = None
        self._grad_ptrs = None
        self._dtype_code = 0 if dt == torch.float32 else 1

    def _build(self):
        grads = [p.grad for p in self.params]
        if any(g is None or not g.is_contiguous() or g.shape != p.shape for g, p in zip(grads, self.params)):
            raise ConfigError("MultiTensorAdamW: every param needs a contiguous .grad")
        ptrs = tuple(g.data_ptr() for g in grads)
        if self._list is not None and ptrs == self._grad_ptrs:
            return
        self.close()
        descs = (type(_DESC_PROTO) * len(self.params))()
        for i, (p, g, m, v) in enumerate(zip(self.params, grads, self.m, self.v)):
            descs[i].param, descs[i].grad = p.data_ptr(), g.data_ptr()
            descs[i].exp_avg, descs[i].exp_avg_sq, descs[i].numel = m.data_ptr(), v.data_ptr(), p.numel()
        h = C.c_void_p()
        check(lib.pier_tensor_list_create(descs, len(self.params), self._dtype_code, C.byref(h)),
              "tensor_list_create")
        self._list, self._grad_ptrs = h, ptrs

    def step(self, lr: float, clip: bool = True) -> None:
        self._build()
        self.step_count += 1
        s = _dev.stream_ptr()
        if clip:
            check(lib.pier_grad_sqnorm_mt(self._list, float(self.cfg.clip_norm), self.ws.data_ptr(), s),
                  "grad_sqnorm_mt")
        hp = self.cfg.hyper(lr, self.step_count)
        check(lib.pier_adamw_mt(self._list, C.byref(hp), self.ws.data_ptr() if clip else None, s),
              "adamw_mt")

    def close(self):
        if self._list is not None:
            lib.pier_tensor_list_destroy(self._list)
            self._list = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


from ._lib import PierTensorDesc as _PTD  # noqa: E402

_DESC_PROTO = _PTD()


# ---------------------------------------------------------------------------
# outer (cross-group) momentum step (optim.py:226-276)
# ---------------------------------------------------------------------------

@dataclass
class OuterState:
    """Outer momentum buffer + window-start snapshot (``optim.py:226-240``)."""

    momentum: object
    snapshot: object
    mu: float = MU_STAGES[0]

    @classmethod
    def initial(cls, theta) -> "OuterState":
        if isinstance(theta, np.ndarray):
            return cls(momentum=np.zeros_like(theta), snapshot=theta)
        return cls(momentum=torch.zeros_like(theta), snapshot=theta)


def fold_momentum(momentum, delta, mu: float):
    """``(mu * momentum) + delta``, fixed order (``optim.py:243-245``)."""
    m, is_np = _dev.to_device(momentum)
    d, _ = _dev.to_device(delta, m.dtype)
    n = _dev.same_shape(m, d)
    out = torch.empty_like(m)
    fn = getattr(lib, f"pier_fold_momentum_{_dev.suffix(m)}")
    check(fn(m.data_ptr(), d.data_ptr(), out.data_ptr(), n, float(mu), _dev.stream_ptr()), "fold_momentum")
    return _dev.back(out, is_np, np.shape(momentum) if is_np else momentum.shape)


def outer_step(state: OuterState, delta, lr: float, mu: float, *, anchor=None):
    """Nesterov step on the averaged delta (``optim.py:248-276``); returns
    ``(theta_new, OuterState(new_momentum, state.snapshot, mu))``."""
    d, is_np = _dev.to_device(delta)
    m, _ = _dev.to_device(state.momentum, d.dtype)
    s, _ = _dev.to_device(state.snapshot, d.dtype)
    a = None if anchor is None else _dev.to_device(anchor, d.dtype)[0]
    n = _dev.same_shape(d, m, s, *(() if a is None else (a,)))
    th = torch.empty_like(d)
    mo = torch.empty_like(d)
    fn = getattr(lib, f"pier_outer_step_{_dev.suffix(d)}")
    check(fn(m.data_ptr(), s.data_ptr(), d.data_ptr(), _dev.ptr(a), th.data_ptr(), mo.data_ptr(), n,
             float(lr), float(mu), _dev.stream_ptr()), "outer_step")
    shape = np.shape(delta) if is_np else delta.shape
    return _dev.back(th, is_np, shape), OuterState(momentum=_dev.back(mo, is_np, shape),
                                                   snapshot=state.snapshot, mu=mu)


# ---------------------------------------------------------------------------
# in-place fused boundary kernels (engine hot path)
# ---------------------------------------------------------------------------

def pseudograd(theta: torch.Tensor, anchor: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """K1: ``theta - anchor`` (``driver.py:415``, ``:434``)."""
    n = _dev.same_shape(theta, anchor)
    out = torch.empty_like(theta) if out is None else out
    fn = getattr(lib, f"pier_pseudograd_{_dev.suffix(theta)}")
    check(fn(theta.data_ptr(), anchor.data_ptr(), out.data_ptr(), n, _dev.stream_ptr()), "pseudograd")
    return out


def outer_update_(avg: torch.Tensor, anchor: torch.Tensor, momentum: torch.Tensor, lr: float, mu: float,
                  theta_out: torch.Tensor | None = None, divisor: int = 1) -> torch.Tensor:
    """K3: the whole outer step after the mean (``driver.py:434-440``) in one
    HBM pass; ``anchor``/``momentum`` updated in place, new params written to
    ``theta_out`` (default: in place into ``avg``)."""
    theta_out = avg if theta_out is None else theta_out
    n = _dev.same_shape(avg, anchor, momentum, theta_out)
    fn = getattr(lib, f"pier_outer_update_{_dev.suffix(avg)}")
    check(fn(avg.data_ptr(), anchor.data_ptr(), momentum.data_ptr(), theta_out.data_ptr(), n, float(lr),
             float(mu), int(divisor), _dev.stream_ptr()), "outer_update")
    return theta_out


def warmup_fold_(theta: torch.Tensor, anchor: torch.Tensor, momentum: torch.Tensor, mu: float) -> None:
    """K3b: ``M = mu*M + (theta - anchor); anchor = theta`` (``driver.py:412-420``)."""
    n = _dev.same_shape(theta, anchor, momentum)
    fn = getattr(lib, f"pier_warmup_fold_{_dev.suffix(theta)}")
    check(fn(theta.data_ptr(), anchor.data_ptr(), momentum.data_ptr(), n, float(mu), _dev.stream_ptr()),
          "warmup_fold")
