"""GPU-resident expert registry: on-demand loading of MESW deltas under an HBM byte budget.

Mirrors SPEC registry: `register` validates an artifact (container +
base digest) and records its size (`compressed_size_bytes`, no bytes resident);
`acquire` makes it resident -- evicting least-recently-used UNPINNED experts (logical
ticks) until it fits, else `BudgetExceededError` with the state unchanged -- and pins
it; `release` unpins; `stats` is a consistent snapshot with a monotone peak.

Loading is whole-artifact and synchronous for the caller, but the bytes
move the B200 way: file read outside the lock into a pinned host buffer, copied to HBM
on a dedicated copy stream and repacked there by the K1 kernels, so loads overlap the
decode stream.  One mutex guards the residency state; the byte reservation is taken
under it before the (unlocked) load, so `current_bytes <= budget_bytes` holds at every
observable point even with concurrent acquires.
"""

from __future__ import annotations

import json
import os
import threading
from dataclasses import dataclass, field

from . import compress
from .errors import (BaseDigestMismatchError, BudgetExceededError, DuplicateExpertError, UnknownExpertError)

__all__ = ["RegistryEntry", "ResidencyState", "ExpertRegistry", "GpuHandle", "GpuExpert", "gpu_loader"]


@dataclass(frozen=True)
class RegistryEntry:
    expert_id: str
    domain: str
    size_bytes: int
    source: object  # path or bytes


@dataclass(frozen=True)
class ResidencyState:
    resident: dict           # id -> (bytes, last_use_tick, pin_count)
    current_bytes: int
    peak_bytes: int
    load_count: int
    evict_count: int


@dataclass
class _Slot:
    nbytes: int
    tick: int
    pins: int
    handle: object = None
    ready: threading.Event = field(default_factory=threading.Event)
    error: BaseException | None = None


class GpuHandle:
    """Residency handle with a consumer fence.  `fence(stream)` (called by `release`)
    records an event on the stream whose kernels read the expert's buffers; eviction
    calls `wait_idle()` before the buffers are dropped, so a kernel still queued on a
    decode stream never reads freed (and possibly re-allocated) memory."""

    _events: list

    def fence(self, stream=None) -> None:
        import torch
        ev = torch.cuda.Event()
        ev.record(stream if stream is not None else torch.cuda.current_stream())
        self._events = [ev]  # stream order: the latest event covers the earlier ones

    def wait_idle(self) -> None:
        for ev in getattr(self, "_events", []):
            ev.synchronize()
        self._events = []


class GpuExpert(GpuHandle):
    """An expert's deltas resident in HBM: one DeviceDelta per MESW layer block, uploaded
    from pinned host buffers on a dedicated copy stream (K1 repack runs there too)."""

    def __init__(self, artifact, device="cuda"):
        import torch
        from .device import DeviceDelta
        self.manifest = artifact.manifest
        self.stream = torch.cuda.Stream(device=device)  # copy + repack off the decode stream
        staging: list = []
        self.layers = [DeviceDelta.from_blocks([blk], device=device, stream=self.stream, staging=staging)
                       for blk in artifact.layers]
        self.stream.synchronize()  # the pinned staging buffers are free after this
        del staging
        self.device_bytes = sum(d.nbytes for d in self.layers)

    @staticmethod
    def planned_bytes(artifact) -> int:
        from .device import DeviceDelta
        return sum(DeviceDelta.device_nbytes([blk]) for blk in artifact.layers)


def gpu_loader(expert_id, artifact):
    return GpuExpert(artifact)


def _read(source) -> bytes:
    if isinstance(source, (bytes, bytearray, memoryview)):
        return bytes(source)
    with open(source, "rb") as f:
        return f.read()


class ExpertRegistry:
    """`size_fn(artifact) -> bytes` sets what the budget counts: the SPEC's artifact bytes
    (`compressed_size_bytes`, the default) or the HBM bytes the loader will allocate
    (`GpuExpert.planned_bytes`, or the serving engine's `MistralMultiExpert.expert_device_bytes`)."""

    def __init__(self, budget_bytes: int, base_digest: str, loader=gpu_loader, unloader=None, size_fn=None):
        if budget_bytes <= 0:
            raise ValueError("budget_bytes must be positive")
        self.budget = int(budget_bytes)
        self.base_digest = base_digest
        self._loader = loader
        self._unloader = unloader
        self._size_fn = size_fn
        self._lock = threading.Lock()
        self._entries: dict = {}
        self._slots: dict = {}
        self._tick = 0
        self._current = 0
        self._peak = 0
        self._loads = 0
        self._evicts = 0

    # ------------------------------------------------------------------ SPEC ops
    def register(self, expert_id: str, source) -> RegistryEntry:
        """validate (container, base digest), record size; nothing resident."""
        blob = _read(source)
        art = compress.deserialize_artifact(blob)  # raises the ArtifactError family
        if art.manifest.base_digest != self.base_digest:
            raise BaseDigestMismatchError(
                f"expert {expert_id!r} was compressed against base {art.manifest.base_digest[:12]}…, "
                f"registry base is {self.base_digest[:12]}…")
        size = int(self._size_fn(art)) if self._size_fn is not None else compress.compressed_size_bytes(art).total
        entry = RegistryEntry(expert_id, art.manifest.domain, size, source)
        with self._lock:
            if expert_id in self._entries:
                raise DuplicateExpertError(f"expert {expert_id!r} already registered")
            if size > self.budget:
                raise BudgetExceededError(f"expert {expert_id!r} ({size} B) exceeds the budget ({self.budget} B)")
            self._entries[expert_id] = entry
        return entry

    def acquire(self, expert_id: str):
        """resident + pinned handle (loads / evicts as needed)."""
        victims = []
        with self._lock:
            entry = self._entries.get(expert_id)
            if entry is None:
                raise UnknownExpertError(f"expert {expert_id!r} is not registered")
            self._tick += 1
            slot = self._slots.get(expert_id)
            if slot is not None:
                slot.tick = self._tick
                slot.pins += 1
                loading = not slot.ready.is_set()
            else:
                free = self.budget - self._current
                cands = sorted((s.tick, k) for k, s in self._slots.items() if s.pins == 0 and s.ready.is_set())
                for _, k in cands:
                    if free >= entry.size_bytes:
                        break
                    victims.append(k)
                    free += self._slots[k].nbytes
                if free < entry.size_bytes:
                    self._tick -= 1
                    raise BudgetExceededError(
                        f"expert {expert_id!r} ({entry.size_bytes} B) does not fit: "
                        f"{self._current} B resident, all evictable experts would free only {free - (self.budget - self._current)} B")
                evicted = [(k, self._slots.pop(k)) for k in victims]
                for k, s in evicted:
                    self._current -= s.nbytes
                    self._evicts += 1
                slot = _Slot(entry.size_bytes, self._tick, 1)
                self._slots[expert_id] = slot
                self._current += entry.size_bytes  # reserved before the (unlocked) load
                self._peak = max(self._peak, self._current)
                self._loads += 1
                loading = None
        if loading is None:  # we own the load: evict, read and upload outside the lock
            for k, s in evicted:
                if hasattr(s.handle, "wait_idle"):
                    s.handle.wait_idle()  # kernels queued before its last release have finished
                if self._unloader is not None:
                    self._unloader(k, s.handle)
                s.handle = None
            try:
                slot.handle = self._loader(expert_id, compress.deserialize_artifact(_read(entry.source)))
            except BaseException as e:
                slot.error = e
                with self._lock:
                    if self._slots.get(expert_id) is slot:
                        del self._slots[expert_id]
                        self._current -= slot.nbytes
                        self._loads -= 1
                slot.ready.set()
                raise
            slot.ready.set()
        elif loading:
            slot.ready.wait()
            if slot.error is not None:
                raise slot.error
        return slot.handle

    def release(self, expert_id: str, stream=None) -> None:
        """Unpin.  For GPU handles, `stream` is the stream the caller's kernels that read
        the expert were queued on (default: the current stream): an event recorded there
        is what eviction waits for."""
        with self._lock:
            slot = self._slots.get(expert_id)
            if slot is None or slot.pins == 0:
                raise UnknownExpertError(f"expert {expert_id!r} is not acquired")
            if hasattr(slot.handle, "fence"):
                slot.handle.fence(stream)
            slot.pins -= 1

    def stats(self) -> ResidencyState:
        with self._lock:
            res = {k: (s.nbytes, s.tick, s.pins) for k, s in self._slots.items()}
            return ResidencyState(res, self._current, self._peak, self._loads, self._evicts)

    # ------------------------------------------------------------------ layout
    @classmethod
    def from_root(cls, root: str, budget_bytes: int, **kw) -> "ExpertRegistry":
        """Registry root layout: <root>/registry.json {base_digest,
        experts: [{id, domain, size_bytes}]} + <root>/<id>.mesw."""
        with open(os.path.join(root, "registry.json")) as f:
            man = json.load(f)
        reg = cls(budget_bytes, man["base_digest"], **kw)
        for e in man["experts"]:
            ent = reg.register(e["id"], os.path.join(root, f"{e['id']}.mesw"))
            if "size_bytes" in e and int(e["size_bytes"]) != ent.size_bytes:
                raise ValueError(f"registry.json size for {e['id']!r} does not match the artifact")
        return reg
