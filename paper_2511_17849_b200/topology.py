"""Drop-in for ``pier.topology`` (topology.py:31-170) plus the real NCCL group
communicator that replaces the simulated collectives on an 8xB200 box.

* ``Topology`` / ``build_topology`` / ``shard_offsets`` / ``ring_allreduce_bytes``:
  integer layout logic, restated exactly.
* ``allreduce_avg`` / ``outer_delta_sync`` / ``inner_gradient_sync``: the
  reference's in-process mean over a list of replicas, computed on the GPU by
  the left-fold kernel K6 (bitwise equal to ``topology.py:113-122``).
* ``GroupComm``: one process per GPU (one Pier group per GPU) -- or n ranks on
  one GPU (``VirtualGroup``) -- whose exchanges are the C layer's kernels on
  NVLink peer memory (csrc/pier_p2p.cu, pier_round.cu), with NCCL for setup and
  the ordering barriers (and the bucketed RS -> K3 -> AG variant, pier_comm.cu).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _dev
from ._lib import check, lib
from .errors import ConfigError


@dataclass(frozen=True)
class Topology:
    """groups x data-parallel replicas x tensor shards (``topology.py:31-92``);
    ``rank = (group * dp_per_group + dp) * tp_size + tp``."""

    groups: int = 4
    dp_per_group: int = 1
    tp_size: int = 1

    def __post_init__(self):
        for name in ("groups", "dp_per_group", "tp_size"):
            if getattr(self, name) < 1:
                raise ConfigError(f"{name} must be a positive integer, got {getattr(self, name)}")

    @property
    def replicas_per_group(self) -> int:
        return self.dp_per_group

    @property
    def num_replicas(self) -> int:
        return self.groups * self.dp_per_group

    @property
    def world_size(self) -> int:
        return self.num_replicas * self.tp_size

    def rank(self, group: int, dp: int, tp: int) -> int:
        if not (0 <= group < self.groups and 0 <= dp < self.dp_per_group and 0 <= tp < self.tp_size):
            raise ValueError(f"coordinates ({group}, {dp}, {tp}) outside topology {self}")
        return (group * self.dp_per_group + dp) * self.tp_size + tp

    def coords(self, rank: int) -> tuple[int, int, int]:
        if not 0 <= rank < self.world_size:
            raise ValueError(f"rank {rank} outside world of size {self.world_size}")
        replica, tp = divmod(rank, self.tp_size)
        group, dp = divmod(replica, self.dp_per_group)
        return group, dp, tp

    def replica_index(self, group: int, dp: int) -> int:
        return group * self.dp_per_group + dp

    def replica_ranks(self, group: int, dp: int) -> range:
        first = self.rank(group, dp, 0)
        return range(first, first + self.tp_size)

    def group_replica_indices(self, group: int) -> list[int]:
        return [self.replica_index(group, d) for d in range(self.dp_per_group)]

    def outer_participant_ranks(self, tp: int) -> list[int]:
        return [self.rank(g, d, tp) for g in range(self.groups) for d in range(self.dp_per_group)]

    def stand_in_ranks(self, rank: int) -> list[int]:
        """For each outer participant of ``rank``'s tensor shard (ascending), the rank whose
        copy ``rank`` folds in for it: the replica of the participant's group with ``rank``'s
        own dp index -- the dp replicas of a group hold identical params at an outer boundary
        (driver.py:426-429), so one pull per group serves the group's every term of the fold
        (pier_outer_step_p2p_reps_f32).  An extension of the reference's Topology."""
        _, d, tp = self.coords(rank)
        return [self.rank(self.coords(q)[0], d, tp) for q in self.outer_participant_ranks(tp)]


def build_topology(groups: int, dp_per_group: int, tp_size: int) -> Topology:
    return Topology(groups=groups, dp_per_group=dp_per_group, tp_size=tp_size)


# ---------------------------------------------------------------------------
# in-process collectives on the GPU (K6)
# ---------------------------------------------------------------------------

def allreduce_avg(arrays: Sequence):
    """Ascending left-fold mean (``topology.py:104-122``), on the GPU.

    Accepts CUDA tensors or NumPy arrays; always returns a fresh array (a
    bitwise copy for one participant), never an alias of an input.
    """
    if len(arrays) == 0:
        raise ValueError("allreduce_avg needs at least one participant")
    if len(arrays) > 64:
        raise ValueError("allreduce_avg: at most 64 participants per launch")
    first = arrays[0]
    for a in arrays[1:]:
        if tuple(np.shape(a)) != tuple(np.shape(first)) or _dtype_name(a) != _dtype_name(first):
            raise ValueError(f"collective participants disagree on shape/dtype: {tuple(np.shape(a))}/"
                             f"{_dtype_name(a)} vs {tuple(np.shape(first))}/{_dtype_name(first)}")
    devs = []
    is_np = False
    for a in arrays:
        t, was_np = _dev.to_device(a)
        devs.append(t)
        is_np = is_np or was_np
    out = torch.empty_like(devs[0])
    fn = getattr(lib, f"pier_mean_left_fold_{_dev.suffix(devs[0])}")
    check(fn(_dev.ptr_array(devs), len(devs), out.data_ptr(), out.numel(), _dev.stream_ptr()), "allreduce_avg")
    shape = np.shape(first)
    return _dev.back(out, is_np, shape)


def _dtype_name(a) -> str:
    return str(a.dtype).replace("torch.", "")


def inner_gradient_sync(grads: Sequence):
    """Mean of one group's gradients (``topology.py:125-127``)."""
    return allreduce_avg(grads)


def outer_delta_sync(deltas: Sequence):
    """Mean across replicas at a boundary (``topology.py:130-132``)."""
    return allreduce_avg(deltas)


def ring_allreduce_bytes(payload_bytes: float, participants: int) -> float:
    """``2 * payload * (n-1) / n`` (``topology.py:135-139``)."""
    if participants <= 1:
        return 0.0
    return 2.0 * payload_bytes * (participants - 1) / participants


def shard_offsets(num_params: int, tp_size: int) -> list[tuple[int, int]]:
    """Near-equal contiguous ranges, remainder to the first shards (``topology.py:146-160``)."""
    if tp_size < 1:
        raise ConfigError(f"tp_size must be a positive integer, got {tp_size}")
    q, r = divmod(num_params, tp_size)
    bounds = [0]
    for i in range(tp_size):
        bounds.append(bounds[-1] + q + (1 if i < r else 0))
    return list(zip(bounds[:-1], bounds[1:]))


def shard_views(theta, tp_size: int):
    return [theta[a:b] for a, b in shard_offsets(int(theta.shape[0]), tp_size)]


def concat_shards(shards):
    if isinstance(shards[0], np.ndarray):
        return np.concatenate(shards)
    return torch.cat(list(shards))


# ---------------------------------------------------------------------------
# real multi-GPU communicator (one Pier group per GPU)
# ---------------------------------------------------------------------------

ALIGN = 64  # elements: every bucket slice starts on a 256-byte boundary


class _DeviceBuffer:
    """__cuda_array_interface__ view of a buffer the C layer allocated."""

    def __init__(self, ptr: int, numel: int, comm, bid: int):
        self.ptr, self.numel, self.comm, self.bid = ptr, numel, comm, bid

    @property
    def __cuda_array_interface__(self):
        return {"shape": (self.numel,), "typestr": "<f4", "data": (self.ptr, False), "version": 3,
                "strides": None, "stream": None}


def padded_len(num_params: int, nranks: int) -> int:
    """Flat length padded so every rank slice is 256-byte aligned; the zero
    padding is inert under AdamW and the outer step."""
    q = nranks * ALIGN
    return ((num_params + q - 1) // q) * q


def broadcast_unique_id(rank: int, world_size: int, pg=None):
    """Rank 0 creates the NCCL unique id; torch.distributed (any backend)
    carries its bytes to every rank.  Returns a ctypes char buffer."""
    import torch.distributed as dist

    nbytes = lib.pier_nccl_unique_id_bytes()
    uid = (C.c_char * nbytes)()
    if world_size > 1:
        payload = [None]
        if rank == 0:
            check(lib.pier_nccl_get_unique_id(uid), "nccl_get_unique_id")
            payload = [bytes(uid)]
        dist.broadcast_object_list(payload, src=0, group=pg)
        C.memmove(uid, payload[0], nbytes)
    else:
        check(lib.pier_nccl_get_unique_id(uid), "nccl_get_unique_id")
    return uid


def valid_shard_prefix(layout, rank: int, num_params: int) -> int:
    """Length of the real-parameter prefix of ``rank``'s shard for a
    ``bucket_layout``: the zero padding sits at the end of the flat buffer,
    inside the last span, so real parameters always form a prefix."""
    off, sl, sh = layout[-1]
    lo = off + rank * sl
    return sh + min(sl, max(0, num_params - lo))


def owned_ranges(layout, rank: int):
    """[(start, stop)] of the flat buffer owned by ``rank`` (one per span)."""
    return [(off + rank * sl, off + (rank + 1) * sl) for off, sl, _ in layout]


class GroupComm:
    """NCCL communicator over all groups (one group per GPU / process).

    Built from a ``torch.distributed`` process group (any backend) that is
    used only to broadcast the NCCL unique id; all data movement goes through
    the C++ layer's own NCCL communicator on its own stream.
    """

    virtual = False

    def __init__(self, rank: int, world_size: int, pg=None, *, _virtual=None):
        self.rank, self.world_size = int(rank), int(world_size)
        self._shared = []
        if _virtual is not None:                  # one rank of a VirtualGroup (no NCCL)
            self._h, self._vg = _virtual
            self.virtual = True
            return
        self._pg = pg
        uid = broadcast_unique_id(self.rank, self.world_size, pg)
        h = C.c_void_p()
        check(lib.pier_comm_init(uid, self.rank, self.world_size, C.byref(h)), "comm_init")
        self._h = h

    @property
    def handle(self):
        return self._h

    def allgather_object(self, obj) -> list:
        """Every rank's ``obj`` in rank order (host-side; setup and reporting only)."""
        if self.virtual:
            return self._vg._allgather(self.rank, obj)
        import torch.distributed as dist
        out = [None] * self.world_size
        dist.all_gather_object(out, obj, group=self._pg)
        return out

    def set_timeout(self, seconds: float) -> None:
        """Spin limit of the persistent round kernel's waits (pier_comm_set_timeout)."""
        check(lib.pier_comm_set_timeout(self._h, float(seconds)), "comm_set_timeout")

    def diag(self) -> list[int]:
        """The round kernel's timeout record {flag, rank, span, observed, target, kind, peer}."""
        out = (C.c_uint32 * 7)()
        check(lib.pier_comm_diag(self._h, out), "comm_diag")
        return list(out)

    def free_shared(self, bid: int) -> None:
        """Release a buffer from ``alloc_shared`` (collective in spirit: every rank frees its copy)."""
        check(lib.pier_comm_free_shared(self._h, int(bid)), "free_shared")
        self._shared = [h for h in self._shared if h.bid != bid]

    def layout(self, num_params: int, bucket_elems: int):
        """(n_padded, shard_len) of the sharded outer state for ``num_params``."""
        n_pad = padded_len(num_params, self.world_size)
        return n_pad, n_pad // self.world_size

    def alloc_shared(self, numel: int) -> tuple[torch.Tensor, int]:
        """Collective: a zeroed fp32 buffer every rank can load/store over
        NVLink (CUDA IPC), wrapped as a torch tensor.  Returns (tensor, id)."""
        ptr, bid = C.c_void_p(), C.c_int32()
        check(lib.pier_comm_alloc_shared(self._h, int(numel) * 4, C.byref(ptr), C.byref(bid)), "alloc_shared")
        holder = _DeviceBuffer(ptr.value, int(numel), self, bid.value)
        t = torch.as_tensor(holder, device=torch.device("cuda", torch.cuda.current_device()))
        self._shared.append(holder)  # the tensor does not own the memory: keep it alive with the comm
        return t, bid.value

    def alloc_window(self, numel: int) -> tuple[torch.Tensor, int]:
        """Collective: a zeroed fp32 NCCL symmetric window with an NVLS
        multicast mapping (for the in-switch reduction path)."""
        ptr, wid = C.c_void_p(), C.c_int32()
        check(lib.pier_comm_alloc_window(self._h, int(numel) * 4, C.byref(ptr), C.byref(wid)), "alloc_window")
        holder = _DeviceBuffer(ptr.value, int(numel), self, wid.value)
        t = torch.as_tensor(holder, device=torch.device("cuda", torch.cuda.current_device()))
        self._shared.append(holder)
        return t, wid.value

    def outer_step_nvls_(self, win_id: int, anchor_shard: torch.Tensor, mom_shard: torch.Tensor,
                         n_padded: int, bucket_elems: int, lr: float, mu: float) -> None:
        check(lib.pier_outer_step_nvls_f32(self._h, win_id, anchor_shard.data_ptr(), mom_shard.data_ptr(),
                                           n_padded, bucket_elems, float(lr), float(mu), _dev.stream_ptr()),
              "outer_step_nvls")

    def allreduce_mean_nvls_(self, win_id: int, n_padded: int) -> None:
        check(lib.pier_allreduce_mean_nvls_f32(self._h, win_id, n_padded, _dev.stream_ptr()), "allreduce_mean_nvls")

    def outer_step_p2p_(self, theta_id: int, anchor_shard: torch.Tensor, mom_shard: torch.Tensor,
                        n_padded: int, bucket_elems: int, lr: float, mu: float) -> None:
        check(lib.pier_outer_step_p2p_f32(self._h, theta_id, anchor_shard.data_ptr(), mom_shard.data_ptr(),
                                          n_padded, bucket_elems, float(lr), float(mu), _dev.stream_ptr()),
              "outer_step_p2p")

    def allreduce_mean_p2p_(self, buf_id: int, n_padded: int) -> None:
        check(lib.pier_allreduce_mean_p2p_f32(self._h, buf_id, n_padded, _dev.stream_ptr()), "allreduce_mean_p2p")

    def allreduce_mean_norm_p2p_(self, buf_id: int, n_padded: int, max_norm: float, ws: torch.Tensor) -> None:
        """The mean plus the clip record of the averaged gradient in ``ws`` (one pass)."""
        check(lib.pier_allreduce_mean_norm_p2p_f32(self._h, buf_id, n_padded, float(max_norm), ws.data_ptr(),
                                                   _dev.stream_ptr()), "allreduce_mean_norm_p2p")

    def lazy_step_p2p_(self, theta_id: int, grad_id: int, m: torch.Tensor, v: torch.Tensor, n_padded: int,
                       bucket: int, hp, max_norm: float, ws: torch.Tensor, team=None, norm_team=None) -> None:
        """Sharded inner step: mean of this rank's shard of the gradient (its ``bucket``-slice
        of every span; + the clip record of the whole mean in ``ws``), AdamW on the shard,
        new params to every rank -- of the team (ascending ranks, a ctypes int32 array) or
        of the whole communicator; ``norm_team``: the ranks of this replica's other tensor
        shards (global clip norm)."""
        nteam = 0 if team is None else len(team)
        nnorm = 0 if norm_team is None else len(norm_team)
        check(lib.pier_lazy_step_p2p_team_f32(self._h, theta_id, grad_id, team, nteam, norm_team, nnorm,
                                              m.data_ptr(), v.data_ptr(), n_padded, bucket, C.byref(hp),
                                              float(max_norm), ws.data_ptr(), _dev.stream_ptr()), "lazy_step_p2p")

    def lazy_pull_span_(self, grad_id: int, staging: torch.Tensor, n_padded: int, bucket: int, span: int,
                        team=None) -> None:
        """Overlapped sharded step: the ranks meet on ``span``; the copy engines bring this rank's
        slice of every team member's gradient into ``staging``."""
        nteam = 0 if team is None else len(team)
        check(lib.pier_lazy_pull_span_p2p_f32(self._h, grad_id, team, nteam, staging.data_ptr(), n_padded, bucket,
                                              span, _dev.stream_ptr()), "lazy_pull_span_p2p")

    def lazy_finish_staged_(self, theta_id: int, grad_id: int, staging: torch.Tensor, m: torch.Tensor,
                            v: torch.Tensor, n_padded: int, bucket: int, hp, max_norm: float, ws: torch.Tensor,
                            team=None, norm_team=None, push: bool = True) -> None:
        """Overlapped sharded step: fold the staged copies (+ clip record), AdamW on the shard,
        all-gather (``push=False``: deferred to ``allgather_span_``)."""
        nteam = 0 if team is None else len(team)
        nnorm = 0 if norm_team is None else len(norm_team)
        check(lib.pier_lazy_finish_staged_p2p_f32(self._h, theta_id, grad_id, team, nteam, norm_team, nnorm,
                                                  staging.data_ptr(), m.data_ptr(), v.data_ptr(), n_padded, bucket,
                                                  C.byref(hp), float(max_norm), ws.data_ptr(), int(push),
                                                  _dev.stream_ptr()), "lazy_finish_staged_p2p")

    def lazy_pull_span_bf16_(self, grad_id: int, staging: torch.Tensor, n_padded: int, bucket: int,
                             span: int) -> None:
        """The 7B recipe's overlapped step: the ranks meet on ``span``; copy-engine pulls of bf16 slices."""
        check(lib.pier_lazy_pull_span_p2p_bf16(self._h, grad_id, staging.data_ptr(), n_padded, bucket, span,
                                               _dev.stream_ptr()), "lazy_pull_span_p2p_bf16")

    def lazy_finish_staged_bf16_(self, master_id: int, live_id: int, grad_id: int, staging: torch.Tensor,
                                 m: torch.Tensor, v: torch.Tensor, n_padded: int, bucket: int, hp, max_norm: float,
                                 ws: torch.Tensor) -> None:
        """The 7B recipe's overlapped step: staged bf16 fold (+ clip record), AdamW on the master
        shard, live params pushed to every rank."""
        check(lib.pier_lazy_finish_staged_p2p_bf16(self._h, master_id, live_id, grad_id, staging.data_ptr(),
                                                   m.data_ptr(), v.data_ptr(), n_padded, bucket, C.byref(hp),
                                                   float(max_norm), ws.data_ptr(), _dev.stream_ptr()),
              "lazy_finish_staged_p2p_bf16")

    def allgather_span_(self, buf_id: int, n_padded: int, bucket: int, span: int, team=None) -> None:
        """Copy-engine pulls of every team member's slice of ``span`` into this rank's buffer."""
        nteam = 0 if team is None else len(team)
        check(lib.pier_allgather_span_p2p_f32(self._h, buf_id, team, nteam, n_padded, bucket, span,
                                              _dev.stream_ptr()), "allgather_span_p2p")

    def lazy_step_p2p_bf16_(self, master_id: int, live_id: int, grad_id: int, m: torch.Tensor, v: torch.Tensor,
                            n_padded: int, bucket: int, hp, max_norm: float, ws: torch.Tensor) -> None:
        """Sharded lazy step of the 7B recipe: bf16 gradient mean of this rank's shard (+ the
        clip record), AdamW on its shard of the fp32 master, RNE bf16 params to every rank."""
        check(lib.pier_lazy_step_p2p_bf16(self._h, master_id, live_id, grad_id, m.data_ptr(), v.data_ptr(),
                                          n_padded, bucket, C.byref(hp), float(max_norm), ws.data_ptr(),
                                          _dev.stream_ptr()), "lazy_step_p2p_bf16")

    def gather_p2p_(self, buf_id: int, n_padded: int, bucket: int = 0, team=None) -> None:
        """Every member's shard (its ``bucket``-slice of every span; 0: its 1/n) of a shared
        buffer into every member's copy."""
        nteam = 0 if team is None else len(team)
        check(lib.pier_gather_p2p_team_f32(self._h, buf_id, team, nteam, n_padded, bucket, _dev.stream_ptr()),
              "gather_p2p")

    def allreduce_mean_(self, buf: torch.Tensor, bucket_elems: int = 1 << 25) -> None:
        """In-place mean over all groups (lazy-phase gradient sync, ``driver.py:380-393``)."""
        if buf.dtype != torch.float32:
            raise ConfigError("allreduce_mean_: float32 buffers")
        check(lib.pier_allreduce_mean_f32(self._h, buf.data_ptr(), buf.numel(), int(bucket_elems),
                                          _dev.stream_ptr()), "allreduce_mean")

    def allreduce_mean_p2p_bf16_(self, buf_id: int, n_padded: int) -> None:
        """Left-fold mean of a shared bf16 buffer (fp32 accumulation, one RNE rounding)."""
        check(lib.pier_allreduce_mean_p2p_bf16(self._h, buf_id, n_padded, _dev.stream_ptr()),
              "allreduce_mean_p2p_bf16")

    def allreduce_mean_norm_p2p_bf16_(self, buf_id: int, n_padded: int, max_norm: float, ws: torch.Tensor) -> None:
        """The bf16 mean plus the clip record of the averaged gradient in ``ws`` (one pass)."""
        check(lib.pier_allreduce_mean_norm_p2p_bf16(self._h, buf_id, n_padded, float(max_norm), ws.data_ptr(),
                                                    _dev.stream_ptr()), "allreduce_mean_norm_p2p_bf16")

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.pier_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class VirtualGroup:
    """``n`` Pier ranks on ONE GPU, one host thread per rank (``pier_vgroup_create``).

    The reference runs its groups inside one process and orders every
    reduction with barriers (``driver.py:476-529``); a virtual group does the
    same on one B200: each rank owns its buffers on the device and drives them
    through the ordinary ``PierEngine`` / ``GroupComm`` calls from its own
    thread.  The communicator's collectives rendezvous on the host (stream
    order by CUDA events) instead of NCCL; the P2P exchanges and the
    persistent round are the same kernels as on n GPUs (the round is ONE
    cooperative launch for all ranks).  Every multi-rank kernel is therefore
    testable on one GPU, bitwise against the oracle.

    ``run(fn, *args)`` calls ``fn(comm, *args)`` on every rank's thread and
    returns the per-rank results; the first rank to raise aborts the group
    (the others' collectives raise ``GroupAborted``) and its exception is
    re-raised (``driver.py:494-501``).
    """

    def __init__(self, n: int):
        import threading

        self.n = int(n)
        self.device = torch.cuda.current_device()
        arr = (C.c_void_p * self.n)()
        check(lib.pier_vgroup_create(self.n, arr), "vgroup_create")
        self._objs = [None] * self.n
        self._bar = threading.Barrier(self.n)
        self.comms = [GroupComm(r, self.n, _virtual=(C.c_void_p(arr[r]), self)) for r in range(self.n)]

    def _allgather(self, rank: int, obj) -> list:
        self._bar.wait()                 # the previous round's readers are done
        self._objs[rank] = obj
        self._bar.wait()
        return list(self._objs)

    def abort(self) -> None:
        lib.pier_vgroup_abort(self.comms[0].handle)
        self._bar.abort()

    def run(self, fn, *args):
        import threading

        from ._lib import GroupAborted

        results = [None] * self.n
        failures = []
        lock = threading.Lock()

        def work(r):
            torch.cuda.set_device(self.device)
            try:
                results[r] = fn(self.comms[r], *args)
            except BaseException as exc:   # noqa: BLE001 -- surfaced in the calling thread
                with lock:
                    failures.append(exc)
                self.abort()

        threads = [threading.Thread(target=work, args=(r,), name=f"pier-vrank-{r}") for r in range(self.n)]
        for th in threads:
            th.start()
        for th in threads:
            th.join()
        torch.cuda.synchronize(self.device)
        if failures:
            primary = [e for e in failures if not isinstance(e, (GroupAborted, threading.BrokenBarrierError))]
            raise (primary or failures)[0]
        return results

    def close(self) -> None:
        for c in self.comms:
            c.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
