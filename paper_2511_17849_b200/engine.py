"""Per-GPU Pier optimizer engine: the inner AdamW stage and the boundary stage
of the reference's ``_Engine`` (driver.py:372-443), one replica per GPU.

Where the reference keeps one in-process worker per replica, here each
process owns ONE replica (or one tensor shard of it) on its GPU, laid out as
the reference's Topology: rank = (group * dp_per_group + dp) * tp_size + tp.

* ``theta``/``grad``/``m``/``v``: flat fp32 buffers (param tensors are views),
  padded to ``team*64`` elements; zero padding is inert.
* outer state: this rank's 1/n share of the anchor ("snapshot") and outer
  momentum among the n replicas of its tensor shard (the outer team), in the
  span/slice layout of csrc/pier_comm.cu, optionally parked in pinned host
  memory between boundaries (HostStore, driver.py:307-329).

Per iteration ``t`` (driver.py:465-474):
  reduce  -- lazy phase / adamw_baseline: left-fold mean of the gradients over
             all replicas; afterwards within each group when dp_per_group > 1
             (driver.py:372-393)
  apply   -- K4a global-norm clip (global over a replica's tp shards) + K4b
             fused AdamW with inner_lr(t) (driver.py:395-399)
  boundary (t % r == 0, driver.py:404-443):
      t <= lazy_end: pier -> K3b warmup fold with mu(t); anchor <- theta
                     diloco -> anchor <- theta only
      t >  lazy_end: mean over the outer team, Nesterov update, re-anchor and
                     broadcast -- fused with the AdamW pass (K5 for one replica,
                     the persistent round kernel over NVLink for several)
The schedule (which t fold, which outer, every (mu, lr)) is the reference's
exactly; ``records`` logs it for the trace-parity tests.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import torch

from . import _dev
from ._lib import check, lib
from ._lib import last_error as _lib_error
from .errors import ConfigError, NumericError
from .offload import HostStore
from .optim import (AdamWConfig, ScheduleConfig, adamw_, adamw_bf16_, grad_sqnorm_, grad_sqnorm_bf16_,
                    inner_lr, momentum_mu, norm_workspace, outer_lr, read_clip)
from .topology import GroupComm, Topology, padded_len, ring_allreduce_bytes, valid_shard_prefix

MODES = ("pier", "adamw_baseline", "diloco_baseline")  # config.py:24
DILOCO_OUTER_LR = 0.7                                  # config.py:28
DILOCO_OUTER_MU = 0.9                                  # config.py:29


@dataclass
class BoundaryRecord:
    iteration: int
    kind: str              # "fold" | "anchor" | "outer"
    phase: str
    mu: float | None
    outer_lr: float | None


@dataclass
class CommStats:
    """``driver.py:103-112``: algorithmic (ring-formula) bytes and event counts."""

    inner_bytes: float = 0.0
    outer_bytes: float = 0.0
    inner_events: int = 0
    outer_events: int = 0

    @property
    def total_bytes(self) -> float:
        return self.inner_bytes + self.outer_bytes


def bucket_layout(n_padded: int, nranks: int, bucket_elems: int):
    """Python mirror of csrc/pier_comm.cu ``layout()``: [(span_off, slice, shard_off)]."""
    out, off, sh = [], 0, 0
    span = bucket_elems * nranks
    while off < n_padded:
        ln = min(n_padded - off, span)
        out.append((off, ln // nranks, sh))
        off += ln
        sh += ln // nranks
    return out


def validate_run(sched: ScheduleConfig, mode: str, outer_lr_fixed, outer_mu_fixed) -> None:
    """The hot-path subset of ``RunConfig.validate`` (config.py:136-185)."""
    if mode not in MODES:
        raise ConfigError(f"mode must be one of {MODES}, got {mode!r}")
    if sched.lazy_end % sched.sync_interval != 0:
        raise ConfigError(
            f"lazy_fraction * total_iters ({sched.lazy_end}) must be a multiple of "
            f"sync_interval ({sched.sync_interval}) so the phase switch lands on a boundary")
    for name, value in (("outer_lr_fixed", outer_lr_fixed), ("outer_mu_fixed", outer_mu_fixed)):
        if value is not None and value < 0.0:
            raise ConfigError(f"{name} must be non-negative, got {value}")
    lr_fixed = outer_lr_fixed if outer_lr_fixed is not None else (
        DILOCO_OUTER_LR if mode == "diloco_baseline" else None)
    if mode != "adamw_baseline" and lr_fixed is None and sched.lazy_end < math.floor(0.1 * sched.total_iters):
        raise ConfigError("lazy_fraction below 0.1 leaves early outer steps outside the outer LR "
                          "schedule domain; raise lazy_fraction or set outer_lr_fixed")


class PierSchedule:
    """Host-side phase logic of the engine (driver.py:301-348, 404-443): which
    iterations fold, re-anchor or take an outer step, with which (mu, lr).
    Pure integer/float control logic -- no device work, testable on CPU."""

    def __init__(self, sched: ScheduleConfig, mode: str = "pier", outer_lr_fixed: float | None = None,
                 outer_mu_fixed: float | None = None):
        validate_run(sched, mode, outer_lr_fixed, outer_mu_fixed)
        self.sched, self.mode = sched, mode
        self.lr_fixed = outer_lr_fixed if outer_lr_fixed is not None else (
            DILOCO_OUTER_LR if mode == "diloco_baseline" else None)     # config.py:123-127
        self.mu_fixed = outer_mu_fixed if outer_mu_fixed is not None else (
            DILOCO_OUTER_MU if mode == "diloco_baseline" else None)     # config.py:129-132
        self.synchronous = mode == "adamw_baseline"                     # driver.py:301
        self.warmup_accumulation = mode == "pier"                       # driver.py:305

    def mu(self, t: int) -> float:                                      # driver.py:333-336
        return self.mu_fixed if self.mu_fixed is not None else momentum_mu(t, self.sched.total_iters)

    def outer_lr(self, t: int) -> float:                                # driver.py:338-341
        return self.lr_fixed if self.lr_fixed is not None else outer_lr(t, self.sched)

    def phase(self, t: int) -> str:                                     # driver.py:343-348
        if self.synchronous:
            return "sync"
        if t <= self.sched.lazy_end:
            return "lazy_start"
        return "pier" if self.mode == "pier" else "diloco"

    def is_boundary(self, t: int) -> bool:                              # driver.py:408
        return (not self.synchronous) and t % self.sched.sync_interval == 0

    def syncs_gradients(self, t: int) -> bool:                          # driver.py:372-374
        return self.synchronous or t <= self.sched.lazy_end

    def event(self, t: int) -> BoundaryRecord | None:
        """What the boundary stage does at ``t`` (driver.py:409-443), or None."""
        if not self.is_boundary(t):
            return None
        if t <= self.sched.lazy_end:
            if self.warmup_accumulation:
                return BoundaryRecord(t, "fold", self.phase(t), self.mu(t), None)
            return BoundaryRecord(t, "anchor", self.phase(t), None, None)
        return BoundaryRecord(t, "outer", self.phase(t), self.mu(t), self.outer_lr(t))



class SpanTracker:
    """Which spans of ``span`` elements (the shard layout of a sharded step) hold a final
    gradient, from disjoint ranges reported by the backward (``PierEngine.grad_ready``).
    Padding past ``num_params`` is final from the start; a span is returned once, by the
    ``report`` that completes it (spans completed by one report in ascending order), and
    ``rest()`` returns the spans never returned, in descending (backward) order."""

    def __init__(self, num_params: int, n_pad: int, span: int):
        self.span = span
        self.left = [max(0, min(num_params, off + span) - off) for off in range(0, n_pad, span)]
        self.done = [False] * len(self.left)

    def report(self, lo: int, hi: int) -> list:
        out = []
        for k in range(lo // self.span, min(len(self.left), -(-hi // self.span))):
            self.left[k] -= max(0, min(hi, (k + 1) * self.span) - max(lo, k * self.span))
            if self.left[k] < 0:
                raise ConfigError(f"grad_ready: overlapping ranges reported for span {k}")
            if self.left[k] == 0 and not self.done[k]:
                self.done[k] = True
                out.append(k)
        return out

    def rest(self) -> list:
        out = [k for k in reversed(range(len(self.done))) if not self.done[k]]
        for k in out:
            self.done[k] = True
        return out

class PierEngine:
    """One Pier group on this GPU; see the module docstring."""

    def __init__(self, num_params: int, sched: ScheduleConfig, adamw: AdamWConfig | None = None, *,
                 mode: str = "pier", comm: GroupComm | None = None, offload: bool = False,
                 bucket_elems: int = 1 << 24, outer_lr_fixed: float | None = None,
                 outer_mu_fixed: float | None = None, theta0: torch.Tensor | None = None,
                 bf16_params: bool = False, check_finite: bool = False, reduce: str = "p2p",
                 topology: Topology | None = None, model_params: int | None = None, lazy_shard: bool = True):
        if reduce not in ("p2p", "nvls", "nccl"):
            raise ConfigError(f"reduce must be 'p2p' (fused NVLink kernel, bitwise), 'nvls' (in-switch "
                              f"reduction) or 'nccl' (bucketed RS/AG), got {reduce!r}")
        self.plan = PierSchedule(sched, mode, outer_lr_fixed, outer_mu_fixed)
        world = comm.world_size if comm else 1
        if reduce != "p2p" and world > 2:
            # the ring / in-switch sums are not the reference's ascending left fold
            # (topology.py:113-121): after K open-loop rounds the outer momentum drifts
            # past the 1e-5 bound at n > 2 (7e-5 max-rel measured at n = 4)
            raise ConfigError(f"reduce={reduce!r} is bitwise only at 2 groups; with {world} use reduce='p2p' "
                              "(ascending left fold, bitwise at every group count)")
        if reduce != "p2p" and getattr(comm, "virtual", False):
            raise ConfigError("a VirtualGroup has no NCCL communicator: use reduce='p2p'")
        self.dev = _dev.require_cuda()
        self.sched, self.cfg, self.mode = sched, adamw or AdamWConfig(), mode
        self.comm = comm
        self.rank = comm.rank if comm else 0
        # groups x dp x tp layout (topology.py:31-92); default: one group per rank
        self.topo = topology if topology is not None else Topology(groups=world)
        if self.topo.world_size != world:
            raise ConfigError(f"topology {self.topo} needs {self.topo.world_size} ranks, communicator has {world}")
        g, _, tp = self.topo.coords(self.rank)
        # outer participants of this rank's tensor shard (outer_participant_ranks) and
        # the dp replicas of its group (_sync_groups, driver.py:372-378), ascending
        self.outer_team = self.topo.outer_participant_ranks(tp)
        self.group_team = [self.topo.rank(g, d, tp) for d in range(self.topo.dp_per_group)]
        self.nranks = len(self.outer_team)              # ranks sharing this buffer's outer state
        self.trank = self.outer_team.index(self.rank)   # this rank's position among them
        self._teams_trivial = len(self.outer_team) == world
        self.num_params = int(num_params)
        self.bucket = int(bucket_elems)
        if self.bucket % 64:
            raise ConfigError("bucket_elems must be a multiple of 64")
        self.n_pad = padded_len(self.num_params, self.nranks)
        self.shard_len = self.n_pad // self.nranks
        self.layout = bucket_layout(self.n_pad, self.nranks, self.bucket)
        self.synchronous = self.plan.synchronous
        self.check_finite = check_finite

        f32 = dict(dtype=torch.float32, device=self.dev)
        self.bf16 = bool(bf16_params)
        # p2p / nvls: theta (and fp32 grads) live in NVLink-mapped buffers so the
        # fused kernels load/store every rank's copy directly (p2p: CUDA IPC peer
        # pointers; nvls: NCCL symmetric window with a multicast mapping)
        self.reduce = reduce if world > 1 else "none"
        self.p2p = self.reduce in ("p2p", "nvls")
        if not self._teams_trivial or self.topo.dp_per_group > 1:
            if self.reduce != "p2p" or self.bf16:
                raise ConfigError("dp_per_group > 1 / tp_size > 1 layouts run on the fp32 p2p exchange")
        self._outer_team_c = self._team_c(self.outer_team)
        self._group_team_c = self._team_c(self.group_team)
        # the tp shards of this rank's replica: their clip norm is global (optim.py:76)
        self.replica_team = list(self.topo.replica_ranks(g, self.topo.coords(self.rank)[1]))
        self._replica_team_c = self._team_c(self.replica_team)
        alloc = None if not self.p2p else (comm.alloc_shared if self.reduce == "p2p" else comm.alloc_window)
        # lazy phase sharded over the ranks (pier_lazy_step_p2p_f32 / _bf16): every replica holds
        # the same params/m/v there, so rank r runs AdamW on its shard (its bucket-slice of every
        # span, 1/n of the buffer) and broadcasts the params; m, v (and with bf16 params the fp32
        # master) then live in NVLink-mapped buffers, current on this rank's shard until gathered
        # back (once the groups diverge, or on read)
        self.lazy_sharded = lazy_shard and self.reduce == "p2p" and self.nranks > 1
        self._master_sharded = False                      # bf16 recipe: master current on our slice only
        # opt-in with grad_ready: the sharded step leaves the all-gather of the params to the copy
        # engines behind the next forward (params_ready(lo, hi) before reading a range)
        self.defer_allgather = False
        self._ag_events = []
        self._theta_id = self._grad_id = self._live_id = None
        if self.p2p:
            self.theta, self._theta_id = alloc(self.n_pad)
        else:
            self.theta = torch.zeros(self.n_pad, **f32)      # fp32 (master) params
        if theta0 is not None:
            self.theta[: self.num_params].copy_(theta0.reshape(-1))
        if self.bf16:
            if self.lazy_sharded:   # the sharded lazy step pushes the live params into every rank
                l32, self._live_id = alloc(self.n_pad // 2)
                self.theta_bf16 = l32.view(torch.bfloat16)
            else:
                self.theta_bf16 = torch.empty(self.n_pad, dtype=torch.bfloat16, device=self.dev)
            check(lib.pier_cast_bf16(self.theta.data_ptr(), self.theta_bf16.data_ptr(), self.n_pad,
                                     _dev.stream_ptr()), "cast_bf16")
            if self.reduce == "p2p":
                # NVLink-mapped like theta: the lazy-phase mean folds every rank's copy
                g32, self._grad_id = alloc(self.n_pad // 2)
                self.grad = g32.view(torch.bfloat16)
            else:
                self.grad = torch.zeros(self.n_pad, dtype=torch.bfloat16, device=self.dev)
        elif self.p2p:
            self.grad, self._grad_id = alloc(self.n_pad)
        else:
            self.grad = torch.zeros(self.n_pad, **f32)
        self._m_id = self._v_id = None
        if self.lazy_sharded:
            self._m, self._m_id = alloc(self.n_pad)
            self._v, self._v_id = alloc(self.n_pad)
        else:
            self._m = torch.zeros(self.n_pad, **f32)
            self._v = torch.zeros(self.n_pad, **f32)
        self._moments_sharded = False                     # m/v current on this rank's slice only ...
        self._moments_team = None                         # ... of this team (None: all ranks)
        self.opt_step = 0
        self.ws = norm_workspace(self.dev)

        self.host = HostStore(offload and not self.synchronous)
        self.anchor = self.mom = None
        if not self.synchronous:
            self.anchor = torch.empty(self.shard_len, **f32)
            self._gather_own(self.anchor)                # OuterState.initial: snapshot = theta0
            self.mom = torch.zeros(self.shard_len, **f32)
            if self.host.enabled:
                self._park()                              # driver.py:308-309
        # reference accounting (driver.py:262): the whole model's bytes per collective
        self.payload_bytes = float((model_params if model_params is not None else self.num_params) * 4)
        self.commstats = CommStats()
        self.records: list[BoundaryRecord] = []
        self.warmup_folds = 0

    # ------------------------------------------------------------------ views
    def params_ready(self, lo: int, hi: int) -> None:
        """Make the current stream wait until params ``[lo, hi)`` hold the last step's values --
        only needed with ``defer_allgather`` (call it in the forward, per range, before reading
        the params' views); every engine call waits for the whole all-gather itself."""
        if self._ag_events:
            for k in range(lo // self._ag_span, min(len(self._ag_events), -(-hi // self._ag_span))):
                if self._ag_events[k] is not None:
                    torch.cuda.current_stream().wait_event(self._ag_events[k])
                    self._ag_events[k] = None

    def _wait_params(self) -> None:
        if self._ag_events:
            self.params_ready(0, self.n_pad)
            self._ag_events = []

    @property
    def theta(self) -> torch.Tensor:
        """fp32 (master) params, full replica.  With bf16 params the sharded lazy steps keep
        only this rank's slice of the master current (the live bf16 params are always
        full), so a read inside the lazy phase gathers the slices first -- collective."""
        self._wait_params()
        self._gather_master()
        return self._theta

    @theta.setter
    def theta(self, value) -> None:
        self._theta = value

    def gather_state(self) -> None:
        """Full replicas of every sharded optimizer array (m, v and, with bf16 params, the
        fp32 master) -- what reading ``theta`` / ``m`` / ``v`` does implicitly.  Collective:
        call it on every rank before a rank-local read (a checkpoint on rank 0 only)."""
        self._wait_params()
        self.gather_moments()
        self._gather_master()

    def _gather_master(self) -> None:
        if self._master_sharded:
            self.comm.gather_p2p_(self._theta_id, self.n_pad, self.bucket)
            self._master_sharded = False

    @property
    def m(self) -> torch.Tensor:
        """AdamW first moment (full replica).  Inside the lazy phase the sharded steps
        keep only this rank's slice current, so a read there gathers every rank's slice
        first -- collective then, like every engine step (the last lazy iteration
        gathers on its own: outside the lazy phase the read is local)."""
        self.gather_moments()
        return self._m

    @property
    def v(self) -> torch.Tensor:
        """AdamW second moment (full replica); see ``m``."""
        self.gather_moments()
        return self._v

    def gather_moments(self) -> None:
        """Restore full m / v replicas after sharded steps (each rank's slice into every
        rank of the team it was sharded over: 2 * (n-1)/n * 4N bytes per direction).
        Collective."""
        if self._moments_sharded:
            self.comm.gather_p2p_(self._m_id, self.n_pad, self.bucket, self._moments_team)
            self.comm.gather_p2p_(self._v_id, self.n_pad, self.bucket, self._moments_team)
            self._moments_sharded = False
            self._moments_team = None

    # ------------------------------------------- sharded step overlapped with backward
    def _sync_team(self, t: int):
        """The team whose sharded step iteration ``t`` runs (None: every rank), its size,
        or (False, 0) when the iteration averages no gradients."""
        if self.nranks > 1 and self.plan.syncs_gradients(t):            # driver.py:373-374
            return (None if self._teams_trivial else self._outer_team_c), self.nranks
        if self.topo.dp_per_group > 1 and not self.synchronous:          # driver.py:375-378
            return self._group_team_c, self.topo.dp_per_group
        return False, 0

    def grad_ready(self, t: int, lo: int, hi: int) -> None:
        """Gradient elements ``[lo, hi)`` of iteration ``t`` are final -- call it from the
        backward pass (e.g. per parameter tensor, in backward order).  In an iteration that
        averages gradients (the lazy phase; with dp > 1 every iteration) the sharded step's
        reduce-scatter then runs behind the backward: as soon as a whole span (team size x
        ``bucket_elems`` elements, the shard layout) is final here, the ranks meet on it and
        the copy engines pull this rank's slice of every team member's gradient into a local
        staging buffer on a side stream -- no SMs are taken from the backward; ``step(t)`` /
        ``inner_step(t)`` then folds the staged copies, finalises the clip record and runs
        AdamW on this rank's shard + the all-gather (pier_lazy_pull_span_p2p_f32 /
        pier_lazy_finish_staged_p2p_f32).  Every rank must report the same ranges in the
        same order (the backward of a replicated model does); ranges are disjoint.  A no-op
        in iterations without a gradient exchange.  With bf16 params (7B recipe) the pulls and
        the fold run on the bf16 gradients."""
        if not self.lazy_sharded:
            raise ConfigError("grad_ready: the overlapped sharded step needs the p2p exchange with several "
                              "replicas")
        if self.bf16 and self.defer_allgather:
            raise ConfigError("grad_ready: defer_allgather is for fp32 params (the 7B recipe all-gathers "
                              "its 2-byte live params in the step)")
        team, n = self._sync_team(t)
        if team is False:
            return
        if not 0 <= lo <= hi <= self.num_params:
            raise ConfigError(f"grad_ready: range [{lo}, {hi}) outside [0, {self.num_params})")
        if getattr(self, "_rs_t", None) != t:       # first report of iteration t
            if self._moments_sharded and self._moments_team is not team:
                self.gather_moments()                 # sharded over another team: replicas first,
                                                      # before any of this iteration's pulls
            self._rs_t, self._rs_team = t, team
            self._rs_spans = SpanTracker(self.num_params, self.n_pad, self.bucket * n)
            if not hasattr(self, "_rs_stream"):   # high priority: its few kernels go first
                self._rs_stream = torch.cuda.Stream(self.dev, priority=-1)
                self._staging = torch.empty(self.n_pad, dtype=torch.bfloat16 if self.bf16 else torch.float32,
                                            device=self.dev)
        for k in self._rs_spans.report(lo, hi):
            self._issue_pull(k)

    def _issue_pull(self, k: int) -> None:
        ev = torch.cuda.Event()
        ev.record()                                   # span k's gradient is written on this stream
        self._rs_stream.wait_event(ev)
        with torch.cuda.stream(self._rs_stream):
            if self.bf16:
                self.comm.lazy_pull_span_bf16_(self._grad_id, self._staging, self.n_pad, self.bucket, k)
            else:
                self.comm.lazy_pull_span_(self._grad_id, self._staging, self.n_pad, self.bucket, k, self._rs_team)

    def _step_or_finish(self, t: int, lr: float, team, mark) -> None:
        """The sharded step of iteration ``t`` over ``team``: the overlapped finish when its
        spans were reported (grad_ready), else the one-call step."""
        pending = getattr(self, "_rs_t", None)
        if pending is not None and pending != t:
            raise ConfigError(f"grad_ready reported iteration {pending} but the step is for iteration {t}")
        if pending is None:
            self._sharded_step(t, lr, team, mark)
            return
        for k in self._rs_spans.rest():               # backward order; the same on every rank
            self._issue_pull(k)
        torch.cuda.current_stream().wait_stream(self._rs_stream)
        self._rs_t = None
        self.opt_step += 1
        if mark is not None:
            mark()
        hp = self.cfg.hyper(lr, self.opt_step)
        if self.bf16:   # 7B recipe: bf16 fold, AdamW on our shard of the master, live params out
            self.comm.lazy_finish_staged_bf16_(self._theta_id, self._live_id, self._grad_id, self._staging, self._m,
                                               self._v, self.n_pad, self.bucket, hp, self.cfg.clip_norm, self.ws)
            self._master_sharded = True
            self._moments_sharded, self._moments_team = True, team
            return
        push = not self.defer_allgather
        self.comm.lazy_finish_staged_(self._theta_id, self._grad_id, self._staging, self._m, self._v, self.n_pad,
                                      self.bucket, hp, self.cfg.clip_norm, self.ws,
                                      team, self._replica_team_c if self.topo.tp_size > 1 else None, push)
        self._moments_sharded, self._moments_team = True, team
        if not push:   # every shard is final (the finish's closing barrier): pull the spans in forward order
            ev = torch.cuda.Event()
            ev.record()
            self._rs_stream.wait_event(ev)
            nteam = self.nranks if team is None else len(team)
            self._ag_span = self.bucket * nteam
            self._ag_events = []
            with torch.cuda.stream(self._rs_stream):
                for k in range(-(-self.n_pad // self._ag_span)):
                    self.comm.allgather_span_(self._theta_id, self.n_pad, self.bucket, k, team)
                    e = torch.cuda.Event()
                    e.record(self._rs_stream)
                    self._ag_events.append(e)

    def _sharded_step(self, t: int, lr: float, team, mark) -> None:
        """Sharded inner step over ``team`` (None: all ranks) -- every member holds the same
        theta/m/v and gets the same averaged gradient, so each updates its shard and the
        params are all-gathered (pier_lazy_step_p2p_team_f32)."""
        if self._moments_sharded and self._moments_team is not team:
            self.gather_moments()                         # sharded over another team before
        self.opt_step += 1
        if mark is not None:
            mark()
        hp = self.cfg.hyper(lr, self.opt_step)
        if self.bf16:   # 7B recipe: bf16 mean of the grads, AdamW on our shard of the master, live params out
            self.comm.lazy_step_p2p_bf16_(self._theta_id, self._live_id, self._grad_id, self._m, self._v, self.n_pad,
                                          self.bucket, hp, self.cfg.clip_norm, self.ws)
            self._master_sharded = True
        else:
            self.comm.lazy_step_p2p_(self._theta_id, self._grad_id, self._m, self._v, self.n_pad, self.bucket, hp,
                                     self.cfg.clip_norm, self.ws, team,
                                     self._replica_team_c if self.topo.tp_size > 1 else None)
        self._moments_sharded, self._moments_team = True, team

    def param_views(self, shapes):
        """Tensors viewing consecutive ranges of the flat params (GPT-2 layout etc.)."""
        src = self.theta_bf16 if self.bf16 else self.theta
        return self._views(src, shapes)

    def grad_views(self, shapes):
        return self._views(self.grad, shapes)

    @staticmethod
    def _views(buf, shapes):
        out, off = [], 0
        for shp in shapes:
            n = math.prod(shp)
            out.append(buf[off: off + n].view(shp))
            off += n
        return out

    # --------------------------------------------------------------- schedule
    def phase(self, t: int) -> str:
        return self.plan.phase(t)

    def is_boundary(self, t: int) -> bool:
        return self.plan.is_boundary(t)

    # ---------------------------------------------------------------- offload
    def _valid_shard(self) -> int:
        """Length of the real-parameter prefix of this rank's shard: the zero
        padding sits at the end of the flat buffer, inside the last span."""
        return valid_shard_prefix(self.layout, self.trank, self.num_params)

    def _park(self):
        # only real parameters travel, so the byte counters equal the
        # reference's (driver.py:139, :148); padding is re-zeroed on fetch
        v = self._valid_shard()
        self.host.store(("snapshot", self.rank), self.anchor[:v])
        self.host.store(("momentum", self.rank), self.mom[:v])
        self.anchor = self.mom = None                    # device memory back to the pool

    def prefetch_outer_state(self) -> None:
        """Start the H2D of the parked outer state (call during the last inner step)."""
        if self.host.enabled and self.anchor is None and getattr(self, "_dst", None) is None:
            v = self._valid_shard()
            self._dst = (torch.empty(self.shard_len, dtype=torch.float32, device=self.dev),
                         torch.empty(self.shard_len, dtype=torch.float32, device=self.dev))
            for buf in self._dst:
                buf[v:].zero_()
            self.host.prefetch(("snapshot", self.rank), self._dst[0][:v])
            self.host.prefetch(("momentum", self.rank), self._dst[1][:v])

    def _fetch(self):
        self.prefetch_outer_state()
        self.host.load(("snapshot", self.rank))
        self.host.load(("momentum", self.rank))
        (self.anchor, self.mom), self._dst = self._dst, None

    # ----------------------------------------------------------------- stages
    def inner_step(self, t: int, lr: float | None = None, mark=None) -> None:
        """Reduce + apply of iteration ``t`` on ``self.grad`` (driver.py:380-399).

        ``mark`` (optional callable) runs between the norm and the AdamW
        launches -- bench.py records a CUDA event there."""
        lr = inner_lr(t, self.sched) if lr is None else lr
        self._wait_params()
        if self.host.enabled and (self.plan.is_boundary(t) or self.plan.is_boundary(t + 1)):
            # start the H2D one iteration ahead: it overlaps this AdamW pass and
            # the next forward/backward instead of stalling the boundary
            self.prefetch_outer_state()
        normed = False
        if self.nranks > 1 and self.plan.syncs_gradients(t):
            # all replicas of this shard (driver.py:373-374)
            if self.lazy_sharded:
                # reduce-scatter + norm of the mean, AdamW on this rank's slice, all-gather of theta
                self.commstats.inner_bytes += ring_allreduce_bytes(self.payload_bytes, self.topo.num_replicas)
                self.commstats.inner_events += 1
                self._step_or_finish(t, lr, None if self._teams_trivial else self._outer_team_c, mark)
                if not self.plan.syncs_gradients(t + 1):
                    # the groups diverge from the next iteration on: full replicas again now,
                    # so no later read of eng.m / eng.v / eng.theta needs a collective
                    self.gather_state()
                return
            if self.reduce == "p2p" and self._teams_trivial and self.topo.tp_size == 1:
                # the mean and K4a in one pass over the gradient (the norm of the mean, optim.py:76)
                if self.bf16:
                    self.comm.allreduce_mean_norm_p2p_bf16_(self._grad_id, self.n_pad, self.cfg.clip_norm, self.ws)
                else:
                    self.comm.allreduce_mean_norm_p2p_(self._grad_id, self.n_pad, self.cfg.clip_norm, self.ws)
                normed = True
            else:
                self._grad_mean(self._outer_team_c, len(self.outer_team))
            self.commstats.inner_bytes += ring_allreduce_bytes(self.payload_bytes, self.topo.num_replicas)
            self.commstats.inner_events += 1
        elif self.topo.dp_per_group > 1 and not self.synchronous:
            # after lazy start: within each group only (driver.py:375-378)
            self.commstats.inner_bytes += self.topo.groups * ring_allreduce_bytes(self.payload_bytes,
                                                                                   self.topo.dp_per_group)
            self.commstats.inner_events += 1
            if self.lazy_sharded:
                # the group's dp replicas are identical too: shard the step over them (m/v
                # stay sharded within the group; eng.m / eng.v gather on read)
                self._step_or_finish(t, lr, self._group_team_c, mark)
                return
            self._grad_mean(self._group_team_c, len(self.group_team))
        self.opt_step += 1
        if self.bf16:
            if not normed:
                self._norm()
            if mark is not None:
                mark()
            adamw_bf16_(self.theta, self.theta_bf16, self.grad, self.m, self.v, self.opt_step, lr, self.cfg,
                        self.ws)
        else:
            if not normed:
                self._norm()
            if mark is not None:
                mark()
            adamw_(self.theta, self.grad, self.m, self.v, self.opt_step, lr, self.cfg, self.ws)

    def boundary(self, t: int) -> BoundaryRecord | None:
        """Boundary stage of iteration ``t`` (driver.py:404-443)."""
        rec = self.plan.event(t)
        if rec is None:
            return None
        self._wait_params()
        if self.check_finite and read_clip(self.ws).nonfinite:
            raise NumericError(f"non-finite gradient norm at iteration {t} on group {self.rank}", iteration=t)
        if self.host.enabled:
            self._fetch()                                 # driver.py:410-411, :424-425
        s = _dev.stream_ptr()
        if rec.kind == "fold":                            # driver.py:413-419
            if self._teams_trivial:
                check(lib.pier_warmup_fold_sharded_f32(self._comm_h(), self.theta.data_ptr(),
                                                       self.anchor.data_ptr(), self.mom.data_ptr(), self.n_pad,
                                                       self.bucket, rec.mu, s), "warmup_fold")
            else:                                         # this rank's slices within its outer team
                for off, sl, sh in self.layout:
                    lo = off + self.trank * sl
                    check(lib.pier_warmup_fold_f32(self.theta[lo:].data_ptr(), self.anchor[sh:].data_ptr(),
                                                   self.mom[sh:].data_ptr(), sl, rec.mu, s), "warmup_fold")
            self.warmup_folds += 1
        elif rec.kind == "anchor":                        # driver.py:420 (diloco: no accumulation)
            self._gather_own(self.anchor)
        elif self.p2p:                                    # driver.py:428-440, one fused NVLink kernel
            self._outer_exchange(rec.outer_lr, rec.mu)
            if self.bf16:
                check(lib.pier_cast_bf16(self.theta.data_ptr(), self.theta_bf16.data_ptr(), self.n_pad, s),
                      "cast_bf16")
            self.commstats.outer_bytes += ring_allreduce_bytes(self.payload_bytes, self.nranks)
            self.commstats.outer_events += 1
        else:                                             # driver.py:428-440, bucketed NCCL RS/K3/AG
            check(lib.pier_outer_step_sharded_f32(self._comm_h(), self.theta.data_ptr(), self.anchor.data_ptr(),
                                                  self.mom.data_ptr(), self.n_pad, self.bucket, rec.outer_lr,
                                                  rec.mu, s), "outer_step_sharded")
            if self.bf16:
                check(lib.pier_cast_bf16(self.theta.data_ptr(), self.theta_bf16.data_ptr(), self.n_pad, s),
                      "cast_bf16")
            self.commstats.outer_bytes += ring_allreduce_bytes(self.payload_bytes, self.nranks)
            self.commstats.outer_events += 1
        if self.host.enabled:
            self._park()                                  # driver.py:421-422, :441-442
        self.records.append(rec)
        return rec

    def step_host(self, t: int, host: dict) -> BoundaryRecord | None:
        """One Pier iteration whose state lives in HOST memory, as a caller of
        the reference holds it (NumPy arrays between calls): per call the
        inputs go host->device, the iteration runs on the GPU, the outputs go
        device->host, all asynchronous on two copy streams so the copies of
        later arrays overlap the kernels of earlier ones (PCIe is duplex).

        ``host``: pinned CPU tensors ``theta, grad, m, v`` ([num_params]) and
        ``anchor, mom`` (the real-parameter prefix of this rank's outer-state
        shard, ``valid_shard_prefix`` elements; all N at one group); updated
        in place.  Returns the boundary record; synchronises before returning.
        """
        if self.host.enabled or self.bf16 or not self._teams_trivial or self.topo.dp_per_group > 1:
            raise ConfigError("step_host drives the resident fp32 engine, one group per rank "
                              "(no offload / bf16 / dp / tp)")
        if not hasattr(self, "_h2d"):
            self._h2d, self._d2h = torch.cuda.Stream(), torch.cuda.Stream()
        self._wait_params()
        self.gather_moments()                             # on the caller's stream, before the copy streams fork
        ev = self.plan.event(t)
        if self.nranks == 1 and ev is not None and ev.kind == "outer":
            return self._step_host_chunked(t, host, ev)
        if self.nranks > 1 and self.reduce == "p2p" and ev is not None and ev.kind == "outer":
            return self._step_host_chunked_groups(t, host, ev)
        n, cur = self.num_params, torch.cuda.current_stream()
        ev_g, ev_w, ev_o = (torch.cuda.Event() for _ in range(3))
        ev_inner, ev_done = torch.cuda.Event(), torch.cuda.Event()
        self._h2d.wait_stream(cur)
        with torch.cuda.stream(self._h2d):
            self.grad[:n].copy_(host["grad"], non_blocking=True)
            ev_g.record()
            for name, dst in (("theta", self.theta), ("m", self.m), ("v", self.v)):
                dst[:n].copy_(host[name], non_blocking=True)
            ev_w.record()
            if self.anchor is not None:
                vs = self._valid_shard()
                self.anchor[:vs].copy_(host["anchor"], non_blocking=True)
                self.mom[:vs].copy_(host["mom"], non_blocking=True)
            ev_o.record()
        cur.wait_event(ev_g)
        cur.wait_event(ev_w)
        self.inner_step(t)
        ev_inner.record(cur)
        cur.wait_event(ev_o)
        rec = self.boundary(t)
        ev_done.record(cur)
        with torch.cuda.stream(self._d2h):
            self._d2h.wait_event(ev_inner)       # m, v are final after the AdamW pass
            host["m"].copy_(self.m[:n], non_blocking=True)
            host["v"].copy_(self.v[:n], non_blocking=True)
            self._d2h.wait_event(ev_done)
            host["theta"].copy_(self.theta[:n], non_blocking=True)
            if self.anchor is not None:
                vs = self._valid_shard()
                host["anchor"].copy_(self.anchor[:vs], non_blocking=True)
                host["mom"].copy_(self.mom[:vs], non_blocking=True)
        self._d2h.synchronize()
        return rec

    def _step_host_chunked(self, t: int, host: dict, ev: BoundaryRecord):
        """Single group at an outer-step boundary, host-resident state: the
        gradient goes up first (the clip needs the global norm), then per
        chunk the five state arrays go up, K5 (AdamW + outer step) runs on the
        chunk and its five results go down -- H2D of chunk c+1, compute of
        chunk c and D2H of chunk c-1 overlap, so the call runs at PCIe speed."""
        n, cur = self.num_params, torch.cuda.current_stream()
        chunk = getattr(self, "host_chunk", 1 << 25)
        lr = inner_lr(t, self.sched)
        self._h2d.wait_stream(cur)
        ev_g = torch.cuda.Event()
        with torch.cuda.stream(self._h2d):
            self.grad[:n].copy_(host["grad"], non_blocking=True)
            ev_g.record()
        cur.wait_event(ev_g)
        self.opt_step += 1
        grad_sqnorm_(self.grad[:n], self.cfg.clip_norm, self.ws)
        hp = self.cfg.hyper(lr, self.opt_step)
        names = (("theta", self.theta), ("m", self.m), ("v", self.v), ("anchor", self.anchor), ("mom", self.mom))
        s = _dev.stream_ptr()
        for a in range(0, n, chunk):
            b = min(n, a + chunk)
            up, done = torch.cuda.Event(), torch.cuda.Event()
            with torch.cuda.stream(self._h2d):
                for name, dst in names:
                    dst[a:b].copy_(host[name][a:b], non_blocking=True)
                up.record()
            cur.wait_event(up)
            check(lib.pier_adamw_outer_f32(self.theta[a:].data_ptr(), self.grad[a:].data_ptr(),
                                           self.m[a:].data_ptr(), self.v[a:].data_ptr(), self.anchor[a:].data_ptr(),
                                           self.mom[a:].data_ptr(), b - a, C.byref(hp), self.ws.data_ptr(),
                                           ev.outer_lr, ev.mu, s), "adamw_outer")
            done.record(cur)
            with torch.cuda.stream(self._d2h):
                self._d2h.wait_event(done)
                for name, src in names:
                    host[name][a:b].copy_(src[a:b], non_blocking=True)
        self._d2h.synchronize()
        self.commstats.outer_events += 1
        self.records.append(ev)
        return ev

    def _step_host_chunked_groups(self, t: int, host: dict, ev: BoundaryRecord):
        """Several groups at an outer boundary, host-resident state: gradient up
        (the clip needs the global norm), then chunk by chunk (whole spans) the
        params/moments and the matching outer-state shard slices go up, AdamW
        and the NVLink exchange of that region run, and its results go down --
        H2D of chunk c+1, compute of chunk c and D2H of chunk c-1 overlap."""
        n, cur, nr = self.num_params, torch.cuda.current_stream(), self.nranks
        span = self.bucket * nr
        chunk = max(span, (getattr(self, "host_chunk", 1 << 25) // span) * span)
        lr = inner_lr(t, self.sched)
        vs = self._valid_shard()
        self._h2d.wait_stream(cur)
        ev_g = torch.cuda.Event()
        with torch.cuda.stream(self._h2d):
            self.grad[:n].copy_(host["grad"], non_blocking=True)
            ev_g.record()
        cur.wait_event(ev_g)
        self.opt_step += 1
        grad_sqnorm_(self.grad, self.cfg.clip_norm, self.ws)
        s = _dev.stream_ptr()
        for a in range(0, self.n_pad, chunk):
            b = min(self.n_pad, a + chunk)
            ha, hb = min(a, n), min(b, n)               # real parameters of the chunk
            sa, sb = a // nr, b // nr                   # its slices in this rank's shard
            qa, qb = min(sa, vs), min(sb, vs)           # ... that hold real parameters
            up, adam_done, xdone = torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event()
            with torch.cuda.stream(self._h2d):
                for name, dst in (("theta", self.theta), ("m", self.m), ("v", self.v)):
                    if hb > ha:
                        dst[ha:hb].copy_(host[name][ha:hb], non_blocking=True)
                if qb > qa:
                    self.anchor[qa:qb].copy_(host["anchor"][qa:qb], non_blocking=True)
                    self.mom[qa:qb].copy_(host["mom"][qa:qb], non_blocking=True)
                up.record()
            cur.wait_event(up)
            adamw_(self.theta[a:b], self.grad[a:b], self.m[a:b], self.v[a:b], self.opt_step, lr, self.cfg, self.ws)
            adam_done.record(cur)
            check(lib.pier_outer_step_p2p_region_f32(self.comm.handle, self._theta_id, a, b - a,
                                                     self.anchor[sa:].data_ptr(), self.mom[sa:].data_ptr(),
                                                     self.bucket, float(ev.outer_lr), float(ev.mu), s),
                  "outer_step_p2p_region")
            xdone.record(cur)
            with torch.cuda.stream(self._d2h):
                self._d2h.wait_event(adam_done)
                if hb > ha:
                    host["m"][ha:hb].copy_(self.m[ha:hb], non_blocking=True)
                    host["v"][ha:hb].copy_(self.v[ha:hb], non_blocking=True)
                self._d2h.wait_event(xdone)
                if hb > ha:
                    host["theta"][ha:hb].copy_(self.theta[ha:hb], non_blocking=True)
                if qb > qa:
                    host["anchor"][qa:qb].copy_(self.anchor[qa:qb], non_blocking=True)
                    host["mom"][qa:qb].copy_(self.mom[qa:qb], non_blocking=True)
        self._d2h.synchronize()
        self.commstats.outer_bytes += ring_allreduce_bytes(self.payload_bytes, self.nranks)
        self.commstats.outer_events += 1
        self.records.append(ev)
        return ev

    def step(self, t: int, mark=None, fuse: bool = True) -> BoundaryRecord | None:
        """Iteration ``t``: inner step then boundary stage (driver.py:466-474).

        At an outer-step boundary the two stages are fused (bitwise identical
        results): one group -> K5 ``pier_adamw_outer`` (one HBM pass for both);
        several groups over NVLink -> ``pier_round_p2p`` (AdamW span by span,
        each span's pull-fold-update-push overlapping the next span's AdamW).
        """
        self._wait_params()
        ev = self.plan.event(t)
        # bf16 params (7B recipe): fused only as the persistent p2p round (no K5 / NVLS variant)
        bf16_unfused = self.bf16 and (self.nranks == 1 or self.reduce != "p2p"
                                      or getattr(self, "round_impl", "persistent") != "persistent")
        # dp > 1 with sharded steps: the boundary is the sharded group step followed by the
        # P2P outer exchange (the fused round would first need the m/v replicas back)
        dp_sharded = self.lazy_sharded and self.topo.dp_per_group > 1
        if (not fuse or ev is None or ev.kind != "outer" or bf16_unfused or dp_sharded
                or (self.nranks > 1 and not self.p2p)):
            self.inner_step(t, mark=mark)
            return self.boundary(t)
        lr = inner_lr(t, self.sched)
        if self.host.enabled:
            self.prefetch_outer_state()
        if self.topo.dp_per_group > 1:   # outer steps follow the lazy phase: group-local mean (driver.py:375-378)
            self._grad_mean(self._group_team_c, len(self.group_team))
            self.commstats.inner_bytes += self.topo.groups * ring_allreduce_bytes(self.payload_bytes,
                                                                                   self.topo.dp_per_group)
            self.commstats.inner_events += 1
        self.opt_step += 1
        self._norm()
        if mark is not None:
            mark()
        if self.check_finite and read_clip(self.ws).nonfinite:
            raise NumericError(f"non-finite gradient norm at iteration {t} on group {self.rank}", iteration=t)
        if self.host.enabled:
            self._fetch()
        hp = self.cfg.hyper(lr, self.opt_step)
        s = _dev.stream_ptr()
        if self.nranks == 1:
            check(lib.pier_adamw_outer_f32(self.theta.data_ptr(), self.grad.data_ptr(), self.m.data_ptr(),
                                           self.v.data_ptr(), self.anchor.data_ptr(), self.mom.data_ptr(),
                                           self.n_pad, C.byref(hp), self.ws.data_ptr(), ev.outer_lr, ev.mu, s),
                  "adamw_outer")
        else:
            if self.reduce == "nvls":
                rnd = lib.pier_round_nvls_f32
            elif self.bf16:
                rnd = lib.pier_round_fused_bf16_f32  # bf16 grads, exchange on the fp32 master
            elif not self._teams_trivial:
                rnd = self._round_team              # one cooperative kernel over the outer team
            elif getattr(self, "round_impl", "persistent") == "persistent":
                rnd = lib.pier_round_fused_f32      # one cooperative kernel: AdamW || exchange
            else:
                rnd = lib.pier_round_p2p_f32        # two streams, NCCL barriers per span
            args = (self.comm.handle, self._theta_id, self.grad.data_ptr(), self.m.data_ptr(), self.v.data_ptr(),
                    self.anchor.data_ptr(), self.mom.data_ptr(), self.n_pad, self.bucket, C.byref(hp),
                    self.ws.data_ptr(), ev.outer_lr, ev.mu, s)
            rc = rnd(*args)
            if rc != 0 and rnd is lib.pier_round_fused_f32:
                # the cooperative grid could not be placed (same on every rank, so all
                # ranks take this branch): run the two-stream pipelined round instead
                import warnings
                warnings.warn(f"persistent round kernel unavailable ({_lib_error()}); using the "
                              "two-stream round", RuntimeWarning)
                self.round_impl = "streams"
                rc = lib.pier_round_p2p_f32(*args)
            check(rc, "round")
            if self.bf16:   # live bf16 params from the new master (the round leaves them stale)
                check(lib.pier_cast_bf16(self.theta.data_ptr(), self.theta_bf16.data_ptr(), self.n_pad, s),
                      "cast_bf16")
            self.commstats.outer_bytes += ring_allreduce_bytes(self.payload_bytes, self.nranks)
        self.commstats.outer_events += 1
        if self.host.enabled:
            self._park()
        self.records.append(ev)
        return ev

    # ------------------------------------------------------------- reporting
    def _comm_h(self):
        # NULL communicator = one group: the C layer runs the fused update over the whole buffer
        return self.comm.handle if self.comm is not None else None

    def _norm(self) -> None:
        """K4a: global gradient norm + clip scale into ``self.ws`` (optim.py:76-78).
        With tensor parallelism the norm stays global over the replica: the
        partial square sums of its tp shards are summed, then re-finalised."""
        if self.bf16:
            grad_sqnorm_bf16_(self.grad, self.cfg.clip_norm, self.ws)
        else:
            grad_sqnorm_(self.grad, self.cfg.clip_norm, self.ws)
        if self.topo.tp_size > 1:
            check(lib.pier_norm_allreduce_team(self.comm.handle, self._replica_team_c, len(self.replica_team),
                                               self.ws.data_ptr(), float(self.cfg.clip_norm), _dev.stream_ptr()),
                  "norm_allreduce_team")

    @staticmethod
    def _team_c(team):
        return (C.c_int32 * len(team))(*team)

    def _grad_mean(self, team_c, nteam: int) -> None:
        """Left-fold mean of ``self.grad`` over ``team`` (inner_gradient_sync, topology.py:125-127)."""
        if self.bf16 and self.reduce == "p2p":   # bf16 grads (7B recipe): fp32 left fold, one RNE rounding
            self.comm.allreduce_mean_p2p_bf16_(self._grad_id, self.n_pad)
        elif self.bf16:            # NVLS engine at <= 2 groups: NCCL bf16 average
            check(lib.pier_allreduce_mean_bf16(self.comm.handle, self.grad.data_ptr(), self.n_pad, self.bucket,
                                               _dev.stream_ptr()), "allreduce_mean_bf16")
        elif self.reduce == "p2p" and (not self._teams_trivial or nteam != len(self.outer_team)):
            check(lib.pier_allreduce_mean_p2p_team_f32(self.comm.handle, self._grad_id, team_c, nteam, self.n_pad,
                                                       _dev.stream_ptr()), "allreduce_mean_p2p_team")
        elif self.reduce == "p2p":   # bitwise = the reference's left fold
            self.comm.allreduce_mean_p2p_(self._grad_id, self.n_pad)
        elif self.reduce == "nvls":
            self.comm.allreduce_mean_nvls_(self._grad_id, self.n_pad)
        else:
            self.comm.allreduce_mean_(self.grad, self.bucket)

    def _outer_exchange(self, lr: float, mu: float) -> None:
        """Mean over the outer team + fused update + broadcast (driver.py:428-440)."""
        if self.reduce == "nvls":
            self.comm.outer_step_nvls_(self._theta_id, self.anchor, self.mom, self.n_pad, self.bucket, lr, mu)
        elif self.topo.dp_per_group > 1:
            # the dp replicas of a group hold identical params: pull one per group, the copy
            # with this rank's dp index, and fold it in for each of the group's ranks (bitwise)
            reps = self.topo.stand_in_ranks(self.rank)
            team = None if self._teams_trivial else self._outer_team_c
            check(lib.pier_outer_step_p2p_reps_f32(self.comm.handle, self._theta_id, team,
                                                   0 if team is None else len(self.outer_team),
                                                   self._team_c(reps), self.anchor.data_ptr(), self.mom.data_ptr(),
                                                   self.n_pad, self.bucket, float(lr), float(mu),
                                                   _dev.stream_ptr()), "outer_step_p2p_reps")
        elif self._teams_trivial:
            self.comm.outer_step_p2p_(self._theta_id, self.anchor, self.mom, self.n_pad, self.bucket, lr, mu)
        else:
            check(lib.pier_outer_step_p2p_team_f32(self.comm.handle, self._theta_id, self._outer_team_c,
                                                   len(self.outer_team), self.anchor.data_ptr(),
                                                   self.mom.data_ptr(), self.n_pad, self.bucket, float(lr),
                                                   float(mu), _dev.stream_ptr()), "outer_step_p2p_team")

    def _round_team(self, h, tid, g, m, v, an, mo, n_pad, bucket, hp, ws, lr, mu, s):
        return lib.pier_round_fused_team_f32(h, tid, self._outer_team_c, len(self.outer_team), g, m, v, an, mo,
                                             n_pad, bucket, hp, ws, lr, mu, s)

    def _gather_own(self, dst: torch.Tensor) -> None:
        """dst[shard] <- this rank's slices of theta (setup / DiLoCo re-anchor)."""
        for off, sl, sh in self.layout:
            lo = off + self.trank * sl
            dst[sh: sh + sl].copy_(self.theta[lo: lo + sl])

    def _full(self, shard: torch.Tensor) -> torch.Tensor:
        if self.nranks == 1:
            return shard[: self.num_params].clone()
        if not self._teams_trivial and getattr(self.comm, "virtual", False):
            # reporting only: the team's shards are tensors on this device
            allp = self.comm.allgather_object(shard)
            full = torch.empty(self.n_pad, dtype=torch.float32, device=self.dev)
            for q, member in enumerate(self.outer_team):
                for off, sl, sh in self.layout:
                    full[off + q * sl: off + (q + 1) * sl].copy_(allp[member][sh: sh + sl])
            self.comm.allgather_object(None)       # every rank copied before anyone moves on
            return full[: self.num_params]
        if not self._teams_trivial:
            # reporting only: all-gather the outer team's shards over a torch.distributed
            # subgroup, then place every member's slices (same span layout)
            import torch.distributed as dist
            if not hasattr(self, "_team_pg"):
                self._team_pg = None
                for tp in range(self.topo.tp_size):      # collective: every rank creates every team group
                    grp = dist.new_group(self.topo.outer_participant_ranks(tp))
                    if tp == self.topo.coords(self.rank)[2]:
                        self._team_pg = grp
            parts = [torch.empty_like(shard) for _ in self.outer_team]
            dist.all_gather(parts, shard.contiguous(), group=self._team_pg)
            full = torch.empty(self.n_pad, dtype=torch.float32, device=self.dev)
            for q, part in enumerate(parts):
                for off, sl, sh in self.layout:
                    full[off + q * sl: off + (q + 1) * sl].copy_(part[sh: sh + sl])
            return full[: self.num_params]
        full = torch.empty(self.n_pad, dtype=torch.float32, device=self.dev)
        check(lib.pier_shard_allgather_f32(self.comm.handle, shard.data_ptr(), full.data_ptr(), self.n_pad,
                                           self.bucket, _dev.stream_ptr()), "shard_allgather")
        return full[: self.num_params]

    def _resident(self, name: str) -> torch.Tensor:
        t = self.anchor if name == "snapshot" else self.mom
        if t is not None:
            return t
        parked = self.host.peek((name, self.rank))
        full = torch.zeros(self.shard_len, dtype=torch.float32, device=self.dev)
        full[: parked.numel()].copy_(parked)
        return full

    def outer_momentum(self) -> torch.Tensor:
        """Full outer momentum in the reference layout (collective when n > 1)."""
        return self._full(self._resident("momentum"))

    def snapshot(self) -> torch.Tensor:
        return self._full(self._resident("snapshot"))

    def params(self) -> torch.Tensor:
        return self.theta[: self.num_params]   # (the property waits for a deferred all-gather)

    def last_clip(self):
        return read_clip(self.ws)

    def close(self) -> None:
        """Release the NVLink-mapped theta / gradient buffers.  Collective: every
        rank of the communicator closes its engine at the same point (a peer may
        still read this rank's buffers until then)."""
        if self.comm is None or getattr(self, "_closed", False):
            return
        self._closed = True
        torch.cuda.synchronize(self.dev)
        self.comm.allgather_object(None)            # every rank's kernels on these buffers are done
        for bid in (self._theta_id, self._grad_id, self._m_id, self._v_id, self._live_id):
            if bid is not None and self.reduce == "p2p":
                self.comm.free_shared(bid)
        self._master_sharded = self._moments_sharded = False
        self.theta = self.grad = self._m = self._v = None
        if self.bf16:
            self.theta_bf16 = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
