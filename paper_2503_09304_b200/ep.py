"""Expert parallelism across the GPUs of one node: experts sharded in contiguous blocks, tokens
data-parallel, NCCL all-to-all-v dispatch and combine per MoE layer.

Per layer on every rank (T local tokens):
  1. router + permute on the local tokens over ALL E experts (libqmoe).  The permute's
     expert-major order makes the rows bound for rank g one contiguous block of Xp.
  2. one all_gather of the E per-expert queue lengths (the same counts the virtual-clock
     boundary decisions need, so every rank can replicate the scheduler's decisions).
  3. dispatch all-to-all-v of Xp rows (bf16, d each).
  4. a local regroup gather (qmoe_gather_rows) puts received rows in local-expert-major order;
     the grouped tcgen05 expert FFN runs on the local experts and, through its perm argument,
     writes each output straight back to its received position.
  5. combine all-to-all-v returns the rows; qmoe_scatter_rows puts them in token-slot order;
     qmoe_combine does the weighted sum (+ residual).
Expert ids, queue order and therefore outputs are identical to the single-GPU path (the local
expert FFN sees exactly the same rows in the same order per expert).

``ops`` is the kernel module (paper_2503_09304_b200.kernels); tests substitute a CPU double to
exercise the exchange logic under gloo.
"""

from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist

from . import kernels as K


def expert_bounds(num_experts: int, world: int) -> list[int]:
    """Contiguous expert blocks; uneven counts (60 over 8) get sizes differing by at most one."""
    return [(num_experts * g) // world for g in range(world + 1)]


def regroup_index(counts: list[list[int]], e_lo: int, e_hi: int) -> tuple[list[int], list[int]]:
    """Rows arrive ordered (source rank, local expert); return (index into the received buffer
    for local-expert-major order, local offsets [E_local + 1]).  counts[src][e] = rows of expert
    e that rank src sends."""
    world = len(counts)
    base, acc = [], 0
    for src in range(world):  # start of (src, e) block in the received buffer
        row = {}
        for e in range(e_lo, e_hi):
            row[e] = acc
            acc += counts[src][e]
        base.append(row)
    idx, offsets = [], [0]
    for e in range(e_lo, e_hi):
        for src in range(world):
            b = base[src][e]
            idx.extend(range(b, b + counts[src][e]))
        offsets.append(len(idx))
    return idx, offsets


def dispatch_tables(allc: list[list[int]], bounds: list[int], me: int) -> tuple[list[int], list[int]]:
    """Peer-memory dispatch: for source rank `me`'s rows of expert e, the owning rank and the first
    receive row there.  Owner g lays its receive buffer out by local expert (ascending), then source
    rank, then queue order -- the order regroup_index produces for the all-to-all transport -- so the
    grouped GEMM consumes it directly.  allc[s][e] = rows of expert e that rank s sends."""
    world = len(allc)
    E = bounds[-1]
    dest_rank, dest_base = [0] * E, [0] * E
    for g in range(world):
        base = 0
        for e in range(bounds[g], bounds[g + 1]):
            dest_rank[e] = g
            dest_base[e] = base + sum(allc[s][e] for s in range(me))
            base += sum(allc[s][e] for s in range(world))
    return dest_rank, dest_base


class ExpertParallelMoE(torch.nn.Module):
    """Mixtral-style sparse MoE block with experts sharded over the process group."""

    def __init__(self, hidden_size: int, intermediate_size: int, num_experts: int, top_k: int, rank: int,
                 world: int, device: Optional[torch.device] = None, dtype: torch.dtype = torch.bfloat16,
                 group=None, ops=K, route_mode: int = K.ROUTE_TOPK_SOFTMAX):
        super().__init__()
        self.d, self.F, self.E, self.k = hidden_size, intermediate_size, num_experts, top_k
        self.rank, self.world, self.group, self.ops = rank, world, group, ops
        self.route_mode = route_mode
        self.device = device or torch.device("cuda")
        self.dtype = dtype
        b = expert_bounds(num_experts, world)
        self.bounds = b
        self.e_lo, self.e_hi = b[rank], b[rank + 1]
        El = self.e_hi - self.e_lo
        self.w_router = torch.empty((num_experts, hidden_size), dtype=dtype, device=self.device)
        self.gate_up = torch.empty((El, 2 * intermediate_size, hidden_size), dtype=dtype, device=self.device)
        self.down = torch.empty((El, hidden_size, intermediate_size), dtype=dtype, device=self.device)

    @torch.no_grad()
    def init_random(self, seed: int = 0) -> "ExpertParallelMoE":
        """Same draws as SparseMoeBlock.init_random for the full layer, sliced to the local experts,
        so an EP run and a single-GPU run share weights."""
        g = torch.Generator(device=self.device).manual_seed(seed)
        d, F, E = self.d, self.F, self.E
        wr = torch.randn((E, d), generator=g, device=self.device, dtype=torch.float32) * d ** -0.5
        self.w_router.copy_(wr)
        gu = torch.randn((E, 2 * F, d), generator=g, device=self.device, dtype=torch.float32).mul_(d ** -0.5)
        self.gate_up.copy_(gu[self.e_lo:self.e_hi])
        del gu
        dn = torch.randn((E, d, F), generator=g, device=self.device, dtype=torch.float32).mul_(F ** -0.5)
        self.down.copy_(dn[self.e_lo:self.e_hi])
        del dn
        return self

    @torch.no_grad()
    def load_full(self, w_router, gate_up, down) -> "ExpertParallelMoE":
        self.w_router.copy_(w_router)
        self.gate_up.copy_(gate_up[self.e_lo:self.e_hi])
        self.down.copy_(down[self.e_lo:self.e_hi])
        return self

    def exchange_counts(self, counts: list[int]) -> list[list[int]]:
        t = torch.tensor(counts, dtype=torch.int64, device=self._comm_device())
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.group)
        return [o.tolist() for o in out]

    def _comm_device(self):
        return self.device

    @torch.no_grad()
    def forward(self, hidden_states: torch.Tensor, residual: Optional[torch.Tensor] = None) -> torch.Tensor:
        ops, E, k, d = self.ops, self.E, self.k, self.d
        shape = hidden_states.shape
        x = hidden_states.reshape(-1, d).contiguous()
        T = x.shape[0]
        ids, w = ops.router(x, self.w_router, k, self.route_mode)
        perm, offsets, xp = ops.permute(ids, E, x=x)
        self.last_routing = (ids, w, perm, offsets)
        off = offsets.tolist()
        counts = [off[e + 1] - off[e] for e in range(E)]
        allc = self.exchange_counts(counts)
        b = self.bounds
        send = [off[b[g + 1]] - off[b[g]] for g in range(self.world)]
        recv = [sum(allc[src][self.e_lo:self.e_hi]) for src in range(self.world)]
        R = off[E]
        x_in = torch.empty((sum(recv), d), dtype=x.dtype, device=x.device)
        dist.all_to_all_single(x_in, xp[:R], output_split_sizes=recv, input_split_sizes=send, group=self.group)
        idx, loc_off = regroup_index(allc, self.e_lo, self.e_hi)
        y_in = torch.empty_like(x_in)
        if idx:
            gidx = torch.tensor(idx, dtype=torch.int32, device=x.device)
            xg = ops.gather_rows(x_in, gidx)
            loc = torch.tensor(loc_off, dtype=torch.int32, device=x.device)
            act = torch.empty((len(idx), self.F), dtype=x.dtype, device=x.device)
            ops.expert_ffn(K.EXPERT_SWIGLU, xg, loc, gidx, self.gate_up, self.down, y_in, act_ws=act)
        y_back = torch.empty((R, d), dtype=x.dtype, device=x.device)
        dist.all_to_all_single(y_back, y_in, output_split_sizes=send, input_split_sizes=recv, group=self.group)
        y = torch.empty((T * k, d), dtype=x.dtype, device=x.device)
        if R:
            ops.scatter_rows(y_back, perm[:R].contiguous(), y)
        res = None if residual is None else residual.reshape(-1, d).contiguous()
        return ops.combine(y, w, res).reshape(shape)


class PeerExpertParallelMoE(ExpertParallelMoE):
    """The same expert-parallel block with the two all-to-alls replaced by peer-memory stores
    (csrc/ep.cu): a dispatch kernel writes every routed row straight into its owner's receive
    buffer in the owner's local-expert-major order, and the grouped GEMM's down-projection epilogue
    writes every output row straight into its source rank's slot buffer, tile by tile.  Device flag
    barriers over peer memory order the phases (no host round trip, no NCCL on the data path).
    Receive / slot / flag buffers are allocated once for `max_tokens` tokens per rank and exchanged
    through CUDA IPC (`connect`, collective)."""

    def __init__(self, hidden_size: int, intermediate_size: int, num_experts: int, top_k: int, rank: int,
                 world: int, max_tokens: int, device: Optional[torch.device] = None,
                 dtype: torch.dtype = torch.bfloat16, group=None, ops=K, route_mode: int = K.ROUTE_TOPK_SOFTMAX,
                 barrier_timeout_s: float = 30.0, host_barrier: bool = False):
        super().__init__(hidden_size, intermediate_size, num_experts, top_k, rank, world, device=device, dtype=dtype,
                         group=group, ops=ops, route_mode=route_mode)
        if dtype != torch.bfloat16:
            raise ValueError("the peer-memory transport runs the bf16 tcgen05 path")
        self.max_tokens = max_tokens
        cap = world * max_tokens * top_k  # worst case: every routed row of every rank lands here
        dev = self.device
        self.x_recv = torch.empty((cap, hidden_size), dtype=dtype, device=dev)
        self.ret = torch.empty(cap, dtype=torch.int32, device=dev)
        self.y = torch.empty((max_tokens * top_k, hidden_size), dtype=dtype, device=dev)
        self.flags = torch.zeros(world, dtype=torch.int32, device=dev)
        self.error = torch.zeros(1, dtype=torch.int32, device=dev)
        self.act = torch.empty((cap, intermediate_size), dtype=dtype, device=dev)
        # per-layer queue lengths of every rank ([world][E], filled by the peers' exchange kernels),
        # the expert ownership bounds and this rank's received row ranges, all on the device
        self.counts = torch.zeros(world * num_experts, dtype=torch.int32, device=dev)
        self.bounds_dev = torch.tensor(self.bounds, dtype=torch.int32, device=dev)
        self.loc_offsets = torch.zeros(self.e_hi - self.e_lo + 1, dtype=torch.int32, device=dev)
        self.epoch = 0
        self.timeout_s = barrier_timeout_s
        # host_barrier: order the phases with a stream sync + process-group barrier instead of the
        # device flag barrier (debugging aid: isolates the data path from the flag protocol)
        self.host_barrier = host_barrier
        self._peer_tables = None
        # the barrier kernels time out into self.error instead of hanging; it is read (one sync)
        # every check_every forward calls and raises (0 disables)
        self.check_every = 64
        self._calls = 0

    def _comm_device(self):
        backend = dist.get_backend(self.group)
        return torch.device("cpu") if backend == "gloo" else self.device

    def connect(self) -> None:
        """Exchange CUDA IPC handles of the receive / return / slot / flag buffers (collective)."""
        bufs = (self.x_recv, self.ret, self.y, self.flags, self.counts)
        mine = [K.ipc_export(t) for t in bufs]
        torch.cuda.synchronize(self.device)  # buffers (zeroed flags) materialised before peers map them
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=self.group)
        tables = []
        for i, t in enumerate(bufs):
            ptrs = [t.data_ptr() if g == self.rank else K.ipc_import(*allh[g][i]) for g in range(self.world)]
            tables.append(torch.tensor(ptrs, dtype=torch.int64, device=self.device))
        self._peer_tables = tables
        dist.barrier(group=self.group)

    def dispatch_tables(self, allc: list[list[int]]) -> tuple[list[int], list[int]]:
        return dispatch_tables(allc, self.bounds, self.rank)

    @torch.no_grad()
    def forward(self, hidden_states: torch.Tensor, residual: Optional[torch.Tensor] = None,
                preempt_flag: Optional[torch.Tensor] = None, cursor_out: Optional[torch.Tensor] = None,
                cursor: Optional[torch.Tensor] = None, routing=None) -> torch.Tensor:
        """One MoE layer with no host round trip: router + permute (local tokens), queue-length
        exchange over peer memory (every rank gets all ranks' counts), dispatch with device-built
        tables, barrier, grouped GEMM on the local experts whose epilogue returns rows to their
        source ranks, barrier, combine.

        Preemption (north_star item 4 under EP): preempt_flag (this rank's int32 device flag, in
        LOCAL expert ids: s > 0 stops the local launch at the first local boundary >= s) and
        cursor_out (local stop) as qmoe_expert_ffn; cursor (int32 [T], GLOBAL expert ids) keeps
        already-completed slots of this rank's tokens out of the dispatch on a resume, with routing
        = (ids, w) of the preempted layer so the resumed layer routes nothing anew."""
        ops, E, k, d = self.ops, self.E, self.k, self.d
        shape = hidden_states.shape
        x = hidden_states.reshape(-1, d).contiguous()
        T = x.shape[0]
        if T > self.max_tokens:
            raise ValueError(f"{T} tokens exceed max_tokens={self.max_tokens}")
        if self._peer_tables is None:
            self.connect()
        x_peers, ret_peers, y_peers, flag_peers, counts_peers = self._peer_tables
        ids, w = routing if routing is not None else ops.router(x, self.w_router, k, self.route_mode)
        perm, offsets, _ = ops.permute(ids, E, cursor=cursor)
        self.last_routing = (ids, w, perm, offsets)
        self.epoch += 1
        ops.ep_exchange_counts(offsets, self.rank, self.world, counts_peers, flag_peers, self.epoch, self.error,
                               self.timeout_s)
        ops.ep_dispatch_dev(x, perm, offsets, k, self.rank, self.world, self.counts, self.bounds_dev, x_peers,
                            ret_peers, self.loc_offsets)
        self._barrier(flag_peers)
        ops.expert_ffn_peer_ex(self.x_recv, self.loc_offsets, self.ret, self.gate_up, self.down, y_peers,
                               rows_hint=T * k, act_ws=self.act, preempt_flag=preempt_flag, cursor_out=cursor_out)
        self._barrier(flag_peers)
        res = None if residual is None else residual.reshape(-1, d).contiguous()
        out = ops.combine(self.y[: T * k], w, res).reshape(shape)
        self._calls += 1
        if self.check_every and self._calls % self.check_every == 0 and self.barrier_failed():
            # a peer never arrived: the layers since the last check ran on partial peer buffers
            raise RuntimeError(f"rank {self.rank}: an expert-parallel device barrier timed out "
                               f"(within the last {self.check_every} layers)")
        return out

    def _barrier(self, flag_peers) -> None:
        self.epoch += 1
        if self.host_barrier:
            torch.cuda.current_stream(self.device).synchronize()
            dist.barrier(group=self.group)
        else:
            self.ops.ep_barrier(flag_peers, self.rank, self.world, self.epoch, self.error, self.timeout_s)

    def barrier_failed(self) -> bool:
        """True if any device barrier timed out (syncs)."""
        return bool(int(self.error.item()))
