"""Unified Dynamic Cache on the device: paged KV storage owned by sequences, never by batches.

Mirrors the reference UnifiedDynamicCache API (reference model.py:266-337: register, has_handle,
can_admit, append/append_many, entries, count, evict_sequence, usage_bytes, recount_bytes) but
stores entries in fixed-size device pages:

  pool[l]  [n_pages, page_size, *row_shape]   one pool per layer (same page ids in every layer)
  pages[h] host list of page ids of sequence h; token position p lives at
           slot = pages[h][p // page_size] * page_size + p % page_size in every layer's pool

Appends are one qmoe_kv_append launch (row scatter by slot mapping); reads are a qmoe_kv_gather
(toy attention) or the page table handed to a paged attention kernel.  Changing batch
composition moves nothing.  The byte ledger is kept in the caller's units: the reference's
``2 * d * 8`` per entry for parity runs (model.py:277), real KV bytes for production models.
"""

from __future__ import annotations

from typing import Optional, Sequence as Seq

import torch

from . import kernels as K
from .core import CacheCapacityError, SimulationError, StateCorruptionError


class UnifiedDynamicCache:
    def __init__(self, num_layers: int, row_shape: Seq[int], dtype: torch.dtype, device: torch.device,
                 entry_bytes: int, capacity_bytes: float = 8 * 1024**3, page_size: int = 16,
                 initial_pages: int = 256, max_pages: Optional[int] = None):
        self.num_layers = num_layers
        self.row_shape = tuple(row_shape)
        self.dtype = dtype
        self.device = device
        self.entry_bytes = int(entry_bytes)
        self.capacity_bytes = capacity_bytes
        self.page_size = page_size
        self.max_pages = max_pages
        self._pools: list[torch.Tensor] = []
        self._n_pages = 0
        self._free: list[int] = []
        self._grow(initial_pages)
        self._pages: dict[int, list[int]] = {}
        self._counts: dict[int, list[int]] = {}
        self._ledger = 0

    # -- physical pages ------------------------------------------------------------------------
    def _grow(self, n_pages: int) -> None:
        if self.max_pages is not None and n_pages > self.max_pages:
            raise CacheCapacityError(f"paged KV pool cannot grow to {n_pages} pages (max {self.max_pages})")
        shape = (n_pages, self.page_size) + self.row_shape
        new = [torch.zeros(shape, dtype=self.dtype, device=self.device) for _ in range(self.num_layers)]
        for l, old in enumerate(self._pools):
            new[l][: old.shape[0]].copy_(old)
        self._free.extend(range(n_pages - 1, self._n_pages - 1, -1))
        self._pools = new
        self._n_pages = n_pages

    def pool(self, layer: int) -> torch.Tensor:
        return self._pools[layer]

    def _ensure_pages(self, handle: int, upto: int) -> None:
        pages = self._pages[handle]
        need = -(-upto // self.page_size)
        while len(pages) < need:
            if not self._free:
                # grow by half: the copy keeps old and new pools alive at once, and a doubling of
                # a multi-GB pool next to a 93 GB model runs out of HBM
                grow = self._n_pages + max(1, self._n_pages // 2)
                if self.max_pages is not None:  # a smaller step that still fits beats a refusal
                    grow = min(grow, max(self.max_pages, self._n_pages + 1))
                self._grow(grow)
            pages.append(self._free.pop())

    def slots(self, handle: int, start: int, n: int) -> list[int]:
        pages, ps = self._pages[handle], self.page_size
        return [pages[p // ps] * ps + p % ps for p in range(start, start + n)]

    def page_table(self, handle: int) -> list[int]:
        return list(self._pages[handle])

    # -- reference API -----------------------------------------------------------------------------
    def register(self, handle: int) -> None:
        if handle in self._pages:
            raise SimulationError(f"cache handle {handle} already registered")
        self._pages[handle] = []
        self._counts[handle] = [0] * self.num_layers

    def has_handle(self, handle: int) -> bool:
        return handle in self._pages

    def can_admit(self, new_entries: int) -> bool:
        return self._ledger + new_entries * self.entry_bytes <= self.capacity_bytes

    def reserve(self, handle: int, layer: int, n: int, want_slots: bool = True) -> list[int]:
        """Account n new entries of one sequence at one layer and return their slots (the same
        slots in every layer, so callers may skip recomputing them with want_slots=False)."""
        if handle not in self._pages:
            raise StateCorruptionError(f"unknown cache handle {handle}")
        if not self.can_admit(n):
            raise CacheCapacityError(
                f"cache capacity {self.capacity_bytes} bytes exceeded at {self._ledger} used")
        start = self._counts[handle][layer]
        self._ensure_pages(handle, start + n)
        self._counts[handle][layer] = start + n
        self._ledger += n * self.entry_bytes
        return self.slots(handle, start, n) if want_slots else []

    def counts_at(self, handles, layer: int) -> list[int]:
        """count(h, layer) for many handles (KeyError for an unknown one)."""
        counts = self._counts
        return [counts[h][layer] for h in handles]

    def reserve_batch(self, handles, layer: int, ns, want_slots: bool = True) -> list[int]:
        """reserve() for every member of a batch at one layer, one call per layer: same counts,
        pages, ledger and slots (concatenated in member order).  When the batch would not fit,
        or a handle is unknown, it falls back to member-by-member reserve() so the error is
        raised at the same member with the same partial accounting."""
        total = sum(ns)
        pages_d, counts_d = self._pages, self._counts
        if self._ledger + total * self.entry_bytes > self.capacity_bytes or any(h not in pages_d for h in handles):
            out: list[int] = []
            for h, n in zip(handles, ns):
                out += self.reserve(h, layer, n, want_slots)
            return out
        ps = self.page_size
        out = []
        for h, n in zip(handles, ns):
            cnt = counts_d[h]
            start = cnt[layer]
            pages = pages_d[h]
            if len(pages) * ps < start + n:
                self._ensure_pages(h, start + n)
            cnt[layer] = start + n
            if want_slots:
                out += [pages[p // ps] * ps + p % ps for p in range(start, start + n)]
        self._ledger += total * self.entry_bytes
        return out

    def unreserve_batch(self, handles, layer: int, ns) -> None:
        """Undo reserve_batch(handles, layer, ns) (the entries were never written: a layer a run-ahead
        host enqueued behind a device-side preemption point, whose guarded append was skipped).
        Pages stay with their sequences."""
        counts_d = self._counts
        for h, n in zip(handles, ns):
            counts_d[h][layer] -= n
        self._ledger -= sum(ns) * self.entry_bytes

    def append_many(self, handle: int, layer: int, rows: torch.Tensor) -> None:
        slots = self.reserve(handle, layer, rows.shape[0])
        K.kv_append(self._pools[layer], torch.tensor(slots, dtype=torch.int32, device=self.device),
                    rows.contiguous())

    def append(self, handle: int, layer: int, row: torch.Tensor) -> None:
        self.append_many(handle, layer, row.unsqueeze(0))

    def scatter(self, layer: int, slots, rows: torch.Tensor, guard: Optional[torch.Tensor] = None) -> None:
        """One launch for the new rows of many sequences (slots from ``reserve``: a list or an
        int32 device tensor).  guard: skip on the device if the iteration was preempted
        (kernels.kv_append)."""
        if len(slots):
            if not isinstance(slots, torch.Tensor):
                slots = torch.tensor(slots, dtype=torch.int32, device=self.device)
            K.kv_append(self._pools[layer], slots, rows if rows.is_cuda else rows.contiguous(), guard=guard)

    def entries(self, handle: int, layer: int) -> torch.Tensor:
        """All entries of one sequence at one layer, ascending entry order, gathered to [n, *row]."""
        n = self._counts[handle][layer]
        if n == 0:
            raise StateCorruptionError(f"no cache entries for handle {handle} layer {layer}")
        out = torch.empty((n,) + self.row_shape, dtype=self.dtype, device=self.device)
        return K.kv_gather(self._pools[layer], torch.tensor(self.slots(handle, 0, n), dtype=torch.int32,
                                                            device=self.device), out)

    def count(self, handle: int, layer: int) -> int:
        return self._counts[handle][layer]

    def evict_sequence(self, handle: int) -> None:
        pages = self._pages.pop(handle, None)
        if pages is None:
            return
        counts = self._counts.pop(handle)
        self._ledger -= sum(counts) * self.entry_bytes
        self._free.extend(reversed(pages))

    def usage_bytes(self) -> int:
        return self._ledger

    def recount_bytes(self) -> int:
        """Brute-force recount from the per-sequence counts (ledger test oracle)."""
        return sum(sum(c) for c in self._counts.values()) * self.entry_bytes

    def pages_in_use(self) -> int:
        return sum(len(p) for p in self._pages.values())
