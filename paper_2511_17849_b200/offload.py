"""Drop-in for the reference's ``HostStore`` (driver.py:115-164): outer state
parked in pinned host memory between boundaries, moved with cudaMemcpyAsync on
a side stream (csrc/pier_offload.cpp).

Same protocol and counters as the reference: ``store`` copies in (the stored
copy is isolated from later writes to the source), ``load`` surrenders the
entry; storing a live key twice or loading a missing key raises
``ProtocolError``; a disabled store ignores ``store`` and rejects ``load``.
Unlike the reference, ``store`` is asynchronous and ``prefetch`` lets the
host->device copy overlap the inner loop before the boundary needs it.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _dev
from ._lib import check, lib
from .errors import ProtocolError


class _Slot:
    __slots__ = ("h", "nbytes", "shape", "dtype", "live", "pending")

    def __init__(self, nbytes: int):
        h = C.c_void_p()
        check(lib.pier_offload_create(1, nbytes, C.byref(h)), "offload_create")
        self.h, self.nbytes = h, nbytes
        self.shape, self.dtype, self.live, self.pending = None, None, False, None

    def close(self):
        if self.h is not None and self.h.value:
            lib.pier_offload_destroy(self.h)
            self.h = None


class HostStore:
    """Host parking for outer state keyed by ``(name, rank)`` (``driver.py:115-164``)."""

    def __init__(self, enabled: bool):
        self.enabled = bool(enabled)
        self._slots: dict[object, _Slot] = {}

    # -- protocol -----------------------------------------------------------
    def store(self, key, array: torch.Tensor) -> None:
        """Park a copy of ``array`` (a CUDA tensor) in pinned host memory."""
        if not self.enabled:
            return
        slot = self._slots.get(key)
        if slot is not None and (slot.live or slot.pending is not None):
            raise ProtocolError(f"offload key {key} stored twice without a reload")
        t, _ = _dev.to_device(array)
        nbytes = t.numel() * t.element_size()
        if slot is None or slot.nbytes < nbytes:
            if slot is not None:
                slot.close()
            slot = self._slots[key] = _Slot(nbytes)
        check(lib.pier_offload_park(slot.h, 0, t.data_ptr(), nbytes, _dev.stream_ptr()), "offload_park")
        # the D2H reads `t` on the side stream: keep the allocator from reusing it early
        t.record_stream(torch.cuda.ExternalStream(lib.pier_offload_stream(slot.h)))
        slot.shape, slot.dtype, slot.live = tuple(array.shape), t.dtype, True

    def prefetch(self, key, out: torch.Tensor | None = None) -> None:
        """Start the host->device copy of ``key`` now; :meth:`load` returns it."""
        if not self.enabled:
            raise ProtocolError("offload disabled: nothing to load")
        slot = self._slots.get(key)
        if slot is None or not slot.live:
            raise ProtocolError(f"offload key {key} loaded before being stored")
        dev = _dev.require_cuda()
        t = out if out is not None else torch.empty(slot.shape, dtype=slot.dtype, device=dev)
        nbytes = t.numel() * t.element_size()
        check(lib.pier_offload_prefetch(slot.h, 0, t.data_ptr(), nbytes, _dev.stream_ptr()), "offload_fetch")
        t.record_stream(torch.cuda.ExternalStream(lib.pier_offload_stream_h2d(slot.h)))
        slot.live, slot.pending = False, t

    def load(self, key, out: torch.Tensor | None = None) -> torch.Tensor:
        """Surrender ``key`` as a device tensor (the current stream waits for it)."""
        if not self.enabled:
            raise ProtocolError("offload disabled: nothing to load")
        slot = self._slots.get(key)
        if slot is None or (not slot.live and slot.pending is None):
            raise ProtocolError(f"offload key {key} loaded before being stored")
        if slot.pending is None:
            self.prefetch(key, out)
        t, slot.pending = slot.pending, None
        check(lib.pier_offload_wait(slot.h, 0, _dev.stream_ptr()), "offload_wait")
        return t

    def peek(self, key) -> torch.Tensor:
        """Device copy of a parked entry WITHOUT surrendering it (reporting only)."""
        slot = self._slots.get(key)
        if slot is None or not slot.live:
            raise ProtocolError(f"offload key {key} is not parked")
        check(lib.pier_offload_sync(slot.h), "offload_sync")
        nbytes = 1
        for d in slot.shape:
            nbytes *= d
        host = torch.empty(slot.shape, dtype=slot.dtype, pin_memory=True)
        C.memmove(host.data_ptr(), lib.pier_offload_host_ptr(slot.h, 0), host.numel() * host.element_size())
        return host.to(_dev.require_cuda())

    def synchronize(self) -> None:
        for s in self._slots.values():
            check(lib.pier_offload_sync(s.h), "offload_sync")

    # -- counters (driver.py:152-164) ---------------------------------------
    def _sum(self):
        tot = [0.0] * 5
        buf = (C.c_double * 5)()
        for s in self._slots.values():
            check(lib.pier_offload_counters(s.h, buf), "offload_counters")
            for i in range(5):
                tot[i] += buf[i]
        return tot

    @property
    def to_host_bytes(self) -> float:
        return self._sum()[0]

    @property
    def from_host_bytes(self) -> float:
        return self._sum()[1]

    @property
    def store_events(self) -> int:
        return int(self._sum()[2])

    @property
    def load_events(self) -> int:
        return int(self._sum()[3])

    @property
    def resident_bytes(self) -> float:
        return self._sum()[4]

    def counters(self) -> dict:
        th, fh, se, le, rb = self._sum()
        return {"enabled": self.enabled, "to_host_bytes": th, "from_host_bytes": fh,
                "store_events": int(se), "load_events": int(le), "resident_bytes": rb}

    def close(self) -> None:
        for s in self._slots.values():
            s.close()
        self._slots.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
