"""Expert-parallel serving (SURVEY.md §8(e) "preemption under EP"): the reference's scheduler,
engine and plugin API unchanged on every rank, the MoE experts sharded across the ranks of one
node.

Design (replicated attention, sharded experts):
  * every rank runs the same Simulation -- same trace, same scheduler, same clock values -- so
    every scheduling and preemption decision is replicated with no decision traffic: a report's
    timestamp is a function of the batch, the queue lengths and the clock, all identical on every
    rank (the permute runs over all E experts on every rank);
  * the attention stage, router, permute, combine and LM head run replicated on each rank's copy
    of the batch (attention + embeddings are ~3% of Mixtral's weights, the experts ~97%: what
    decode streams from HBM is sharded);
  * rank g holds experts [bounds[g], bounds[g+1]) and runs the grouped tcgen05 GEMM on those only
    (qmoe_expert_ffn on the local slice of the queue offsets);
  * the combine exchange is an all-gather of expert outputs over NVLink peer memory with no host
    round trip: each rank pushes its experts' output rows into the same slot of every peer's
    receive buffer (qmoe_ep_share_rows), a device flag barrier, and each rank copies the other
    ranks' rows into its slot-ordered y (qmoe_ep_collect_rows) before the replicated combine;
  * preemption: the engine's host-boundary mode decides the stop expert before the launch on
    every rank alike (virtual-clock exact mode, reference engine.py:204-219); each rank runs
    [lo, hi) ∩ [0, stop), exchanges, and the per-token cursors advance to the same global stop, so
    checkpoints, resumes and the decision log are identical to the single-GPU run.

Clock: a VirtualClock (exact decision-log parity) or a LockstepClock -- rank 0's wall clock,
broadcast at the top of every scheduler iteration, advanced between broadcasts by the engine's
cost-model charges, so the ranks agree on every timestamp while it tracks real time.

Next step (not built): data-parallel attention (members sharded across ranks, token dispatch
with qmoe_ep_dispatch_dev as in ep.PeerExpertParallelMoE) with the scheduler replicated the same
way.
"""

from __future__ import annotations

import time
from typing import Optional

import torch
import torch.distributed as dist

from . import kernels as K
from .ep import expert_bounds
from .mixtral import DecoderConfig, DecoderMoEModel


class LockstepClock:
    """Milliseconds shared by the ranks: rank 0's wall clock at every sync(), advanced in between
    by the engine's cost-model charges times a scale that tracks the ratio of wall time to charged
    time over the previous iterations (so any CostModel -- the reference's A100-era default or a
    fitted B200 one -- keeps report timestamps close to real time between syncs).  Every input of
    the clock (the broadcast wall time, the replicated charges) is the same on every rank, so the
    ranks read the same time.  virtual=True: the engine keeps the host-boundary (replicable) expert
    decisions and the driver starts no arrival watcher."""

    virtual = True

    def __init__(self, group=None, device: Optional[torch.device] = None):
        self.group = group
        backend = dist.get_backend(group)
        self._dev = torch.device("cpu") if backend == "gloo" else (device or torch.device("cuda"))
        self._buf = torch.zeros(1, dtype=torch.float64, device=self._dev)
        self._rank = dist.get_rank(group)
        dist.barrier(group=group)
        self._t0 = time.perf_counter()
        self.now = 0.0
        self.syncs = 0
        self.scale = 1.0        # wall ms per charged ms
        self._charged = 0.0     # charged (unscaled) since the last sync
        self._last_wall = 0.0

    def wall_ms(self) -> float:
        return (time.perf_counter() - self._t0) * 1000.0

    def sync(self) -> None:
        self._buf.fill_(self.wall_ms() if self._rank == 0 else 0.0)
        dist.broadcast(self._buf, 0, group=self.group)
        w = float(self._buf.item())
        if self._charged > 0.0 and w > self._last_wall:
            self.scale = 0.5 * self.scale + 0.5 * (w - self._last_wall) / self._charged
        self._charged, self._last_wall = 0.0, w
        self.now = max(self.now, w)
        self.syncs += 1

    def advance(self, delta_ms: float) -> None:
        if delta_ms < 0:
            raise ValueError(f"clock cannot move backwards (delta {delta_ms})")
        self._charged += delta_ms
        self.now += self.scale * delta_ms

    def advance_to(self, timestamp: float) -> None:
        wait = timestamp - self.wall_ms()
        if wait > 0:
            time.sleep(wait / 1000.0)
        self.now = max(self.now, timestamp)


class ExpertParallelDecoder(DecoderMoEModel):
    """DecoderMoEModel plugin whose experts are sharded over the process group (see module doc).
    Every rank must construct it with the same cfg / seed and drive the same Simulation."""

    def __init__(self, cfg: DecoderConfig, rank: int, world: int, group=None, device: Optional[torch.device] = None,
                 seed: int = 0, dtype: torch.dtype = torch.bfloat16, barrier_timeout_s: float = 30.0):
        from .moe_block import shared_sub_experts

        S = shared_sub_experts(cfg.shared_ffn_dim, cfg.ffn_dim) if cfg.shared_ffn_dim else 0
        self.bounds = expert_bounds(cfg.num_experts + S, world)
        self.rank, self.world, self.group = rank, world, group
        super().__init__(cfg, device=device, seed=seed, dtype=dtype,
                         expert_range=(self.bounds[rank], self.bounds[rank + 1]))
        self.timeout_s = barrier_timeout_s
        self._direct_shared = False  # the local slice of the queues reads gathered rows only
        self.flags = torch.zeros(world, dtype=torch.int32, device=self.device)
        self.error = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.epoch = 0
        self._recv = None      # two receive buffers [cap, d] (alternating per exchange)
        self._peers = None     # ([recv0 peers], [recv1 peers], flag peers) int64 device tables
        self._cap = 0
        self._parity = 0
        self.stats = {"exchanges": 0, "rows_pushed": 0}
        self.check_every = 256

    # ------------------------------------------------------------------ peer buffers
    def _connect(self, cap: int) -> None:
        """(Re)allocate the two receive buffers for cap slots and exchange IPC handles (collective:
        every rank reaches it at the same layer, since the batch is replicated)."""
        d = self.cfg.hidden_dim
        self._recv = [torch.empty((cap, d), dtype=self.dtype, device=self.device) for _ in range(2)]
        bufs = self._recv + [self.flags]
        mine = [K.ipc_export(t) for t in bufs]
        torch.cuda.synchronize(self.device)
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=self.group)
        self._peers = [torch.tensor([t.data_ptr() if g == self.rank else K.ipc_import(*allh[g][i])
                                     for g in range(self.world)], dtype=torch.int64, device=self.device)
                       for i, t in enumerate(bufs)]
        self._cap = cap
        dist.barrier(group=self.group)

    def _barrier(self) -> None:
        self.epoch += 1
        K.ep_barrier(self._peers[2], self.rank, self.world, self.epoch, self.error, self.timeout_s)

    # ------------------------------------------------------------------ engine interface
    def run_experts(self, layer: int, xp, offsets, perm, y, e_begin: int, e_end: int, preempt_flag=None,
                    progress=None, progress_seq: int = 0, cursor_out=None):
        """This rank's experts of the launch range on the tensor cores, then the output all-gather.
        Returns the global stop (device int32) the engine advances the cursors to."""
        if preempt_flag is not None or progress is not None:
            raise NotImplementedError("expert-parallel serving decides expert boundaries on the host "
                                      "(LockstepClock / VirtualClock), not with the device flag")
        lo, hi = self.e_lo, self.e_hi
        a, b = max(lo, e_begin), min(hi, e_end)
        L = self.layers[layer]
        if a < b:
            rows = xp.shape[0]
            F = self.cfg.ffn_dim
            act = K.workspace(rows * F * 2, "act", self.device).view(self.dtype)[: rows * F].view(rows, F)
            # the local slice of the global queue offsets (absolute queue positions into xp / perm)
            K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets[lo:hi + 1], perm, L.gate_up, L.down, y, e_begin=a - lo,
                         e_end=b - lo, act_ws=act)
        if self.world > 1:
            n = y.shape[0]
            if n > self._cap:
                self._connect(max(n, 2 * self._cap))
            p = self._parity
            self._parity ^= 1
            if a < b:
                K.ep_share_rows(y, perm, offsets, a, b, self._peers[p], self.rank, self.world)
            self._barrier()
            K.ep_collect_rows(self._recv[p], y, perm, offsets, e_begin, e_end, a if a < b else lo,
                              b if a < b else lo)
            self.stats["exchanges"] += 1
            if self.check_every and self.stats["exchanges"] % self.check_every == 0 and int(self.error.item()):
                raise RuntimeError(f"rank {self.rank}: an expert-parallel device barrier timed out")
        stop = self._stop if cursor_out is None else cursor_out
        stop.fill_(e_end)
        return stop
