"""Routing-replay device plugin — TEST DOUBLE for CPU-only tests of the host control path.

It stands in for the device model (paper_2503_09304_b200.model.MoEModel) so the REAL engine,
scheduler and driver can run on a CPU builder against the decision logs the reference produced
(tests/golden/logs).  Expert ids and emitted tokens are replayed in call order from the
reference's own route/route_many/emit_token records; the per-expert
queue construction is a plain torch restatement.  The product path never uses this module.
"""

from __future__ import annotations

import gzip
import json
from types import SimpleNamespace

import torch

from conftest import GOLDEN
from paper_2503_09304_b200.core import Phase, StateCorruptionError
from paper_2503_09304_b200.model import ModelConfig


def load_log(name: str) -> dict:
    with gzip.open(GOLDEN / "logs" / f"{name}.json.gz", "rt") as fh:
        return json.load(fh)


def trace_of(rec: dict):
    from paper_2503_09304_b200.core import Priority
    from paper_2503_09304_b200.workload import TraceRecord

    return [TraceRecord(i, a, Priority.from_tag(p), pl, mn, s) for i, a, p, pl, mn, s in rec["trace"]]


class ReplayModel:
    kv_dtype = torch.float32
    device = torch.device("cpu")
    kv_page_kwargs = {"initial_pages": 4}

    def __init__(self, rec: dict):
        self.config = ModelConfig(**rec["model"])
        self._routes = list(rec["routes"])
        self._emits = list(rec["emits"])
        self._r = 0
        self._e = 0

    def kv_row_shape(self):
        return (1,)

    def kv_entry_bytes(self):
        return 2 * self.config.hidden_dim * 8

    def embed_batch(self, tokens):
        return torch.zeros((len(tokens), 1))

    def attention_batch(self, layer, h, members, cache):
        for m in members:
            seq = m.seq
            have = cache.count(seq.cache_handle, layer)
            want = seq.tokens_fed() if seq.phase is Phase.DECODE else 0
            if have != want:
                raise StateCorruptionError(f"sequence {seq.id} layer {layer}: {have} entries, expected {want}")
            cache.reserve(seq.cache_handle, layer, m.n)
        x = torch.zeros((h.shape[0], 1))
        return x, x

    def route_batch(self, layer, x):
        T, rows = x.shape[0], []
        while len(rows) < T:
            rl, n, ids = self._routes[self._r]
            self._r += 1
            assert rl == layer and len(ids) == n, "replay diverged from the reference call order"
            rows += ids
        assert len(rows) == T, "replay diverged: batch token count"
        ids = torch.tensor(rows, dtype=torch.int32)
        return ids, torch.zeros(ids.shape)

    def new_expert_state(self, T):
        return torch.zeros((T * self.config.top_k, 1)), torch.zeros(T, dtype=torch.int32)

    def permute(self, ids, cursor, x):
        E, k = self.config.num_experts, self.config.top_k
        flat = ids.reshape(-1).long()
        pend = (ids >= cursor[:, None]).reshape(-1)
        key = torch.where(pend, flat, torch.full_like(flat, E))
        order = torch.sort(key, stable=True).indices
        counts = torch.bincount(flat[pend], minlength=E)[:E].tolist()
        perm = order[: int(pend.sum())].to(torch.int32)
        offsets = torch.tensor([0] + list(torch.tensor(counts).cumsum(0).tolist()), dtype=torch.int32)
        return perm, offsets, None

    def run_experts(self, layer, xp, offsets, perm, y, e_begin, e_end, preempt_flag=None, **_):
        return torch.tensor([e_end], dtype=torch.int32)

    def advance_cursor(self, cursor, stop):
        cursor.clamp_(min=int(stop[0]))

    def combine_batch(self, layer, y, w, res, x):
        return torch.zeros_like(res)

    def emit_batch(self, h, rows):
        out = self._emits[self._e:self._e + len(rows)]
        self._e += len(rows)
        return out

    @staticmethod
    def cat_rows(parts):
        return torch.cat(parts, 0)


class RandomPreempt:
    """Seeded coin per report, the reference's test policy (tests/test_sim.py:18-28)."""

    def __init__(self, seed, p=0.3):
        import numpy as np
        from paper_2503_09304_b200.core import SchedulerDirective

        self.rng = np.random.default_rng(seed)
        self.p = p
        self.D = SchedulerDirective

    def __call__(self, report, queues):
        return self.D.PREEMPT_AT_NEXT_BOUNDARY if self.rng.random() < self.p else self.D.CONTINUE


def policy_for(rec: dict):
    spec = rec["policy"]
    if spec.startswith("random:"):
        _, seed, p = spec.split(":")
        return RandomPreempt(int(seed), float(p))
    return None
