"""Inference engine: drives a batch through ATTENTION -> ROUTER -> EXPERTS per layer, reports
to the scheduler after attention, after the router and after each non-empty expert, honours
PREEMPT_AT_NEXT_BOUNDARY at those boundaries, and checkpoints/restores batch state on the device.

Same public surface as the reference engine (reference engine.py:31-226): VirtualClock,
CostModel, Completed, Preempted, InferenceEngine.execute / restore / next_batch_id,
max_stage_cost.  What changes is where state lives and how the expert stage runs:

* Batch state (expert input, residual, routing ids/weights, expert outputs in slot order, and a
  per-token expert cursor) is a handful of device tensors.  A checkpoint is a set of row views
  of them — preemption copies nothing (reference engine.py:401-423 copies every array).
* The expert stage is: one permute launch (stable expert-major queue order over the pending
  slots), one 4*(E+1)-byte D2H of the queue offsets, the report loop on the host (the virtual
  timestamps of all expert boundaries follow from the queue lengths: engine.py:215), and ONE
  grouped expert launch for experts [0, stop) where stop is the boundary the scheduler chose.
  On preemption the per-token cursors advance to `stop` on the device.
* Restore rebuilds a merged resume batch in the new member order by concatenating checkpoint
  rows (zero-copy when the resumed members are one contiguous run of a single preempted batch).

Device plugin interface (model.py implements it; tests may substitute a replay double):
  config.{num_layers, hidden_dim, num_experts, top_k}
  embed_batch(tokens) -> h[T,d]
  attention_batch(layer, h, members, cache) -> (x, residual)
  route_batch(layer, x) -> (ids[T,k], w[T,k])
  new_expert_state(T) -> (y[T*k,d], cursor[T])
  permute(ids, cursor, x) -> (perm, offsets, xp, counts: list[int])
  run_experts(layer, xp, offsets, perm, y, e_begin, e_end) -> stop (device int32[1])
  advance_cursor(cursor, stop)
  combine_batch(layer, y, w, residual, x) -> h_next[T,d]
  emit_batch(h, rows) -> list[int]
  cat_rows(list of tensors) -> tensor
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field
from typing import Callable, Optional, Union

from .core import (Batch, BatchProgress, Checkpoint, EngineReport, MemberProgress, Phase, SchedulerDirective, Sequence,
                   SimulationError, Stage, StateCorruptionError, batch_form)
from .model import MemberRows

PREEMPT = SchedulerDirective.PREEMPT_AT_NEXT_BOUNDARY


class VirtualClock:
    """Monotone virtual milliseconds (reference engine.py:31-45)."""

    virtual = True

    def __init__(self, start: float = 0.0):
        self.now = float(start)

    def advance(self, delta_ms: float) -> None:
        if delta_ms < 0:
            raise SimulationError(f"clock cannot move backwards (delta {delta_ms})")
        self.now += delta_ms

    def advance_to(self, timestamp: float) -> None:
        if timestamp < self.now:
            raise SimulationError(f"clock cannot jump back to {timestamp} from {self.now}")
        self.now = timestamp


class WallClock:
    """Real milliseconds since construction.  Charges are ignored (time passes by itself);
    advance_to sleeps until the target so idle periods last as long as in a real server."""

    virtual = False

    def __init__(self):
        self._t0 = time.perf_counter()

    @property
    def now(self) -> float:
        return (time.perf_counter() - self._t0) * 1000.0

    def advance(self, delta_ms: float) -> None:
        if delta_ms < 0:
            raise SimulationError(f"clock cannot move backwards (delta {delta_ms})")

    def advance_to(self, timestamp: float) -> None:
        wait = timestamp - self.now
        if wait > 0:
            time.sleep(wait / 1000.0)


@dataclass(frozen=True)
class CostModel:
    """Linear virtual-time charges per stage in ms (reference engine.py:48-88)."""

    attn_base: float = 1.2
    attn_per_token: float = 0.001
    attn_per_cached: float = 0.0003
    router_cost: float = 0.8
    expert_base: float = 0.85
    expert_per_entry: float = 0.0005
    checkpoint_cost: float = 2.0
    restore_cost: float = 2.0

    def validate(self) -> None:
        for name, value in self.__dict__.items():
            if value < 0:
                raise ValueError(f"cost parameter {name} must be >= 0, got {value}")

    def attention_cost(self, tokens: int, cached_entries: int) -> float:
        return self.attn_base + self.attn_per_token * tokens + self.attn_per_cached * cached_entries

    def expert_cost(self, entries: int) -> float:
        return self.expert_base + self.expert_per_entry * entries

    def stage_cost(self, stage: Stage, *, tokens: int = 0, cached_entries: int = 0, expert_entries: int = 0) -> float:
        if stage is Stage.ATTENTION:
            return self.attention_cost(tokens, cached_entries)
        if stage is Stage.ROUTER:
            return self.router_cost
        if stage is Stage.EXPERTS:
            return 0.0 if expert_entries == 0 else self.expert_cost(expert_entries)
        return 0.0

    def scaled(self, factor: float) -> "CostModel":
        return CostModel(**{k: v * factor for k, v in self.__dict__.items()})


@dataclass
class Completed:
    tokens: dict[int, int]


@dataclass
class Preempted:
    checkpoints: dict[int, Checkpoint]


IterationOutcome = Union[Completed, Preempted]
ReportCallback = Callable[[EngineReport], SchedulerDirective]


@dataclass
class _State:
    """Device state of one in-flight batch; rows are member-major, token order within a member."""

    seqs: list[Sequence]
    members: list[MemberRows]
    T: int
    h: object = None         # hidden entering the attention stage
    x: object = None         # expert input (attention-stage output)
    res: object = None       # residual for the combine
    ids: object = None
    w: object = None
    y: object = None
    cursor: object = None
    progress: tuple = ()     # MemberProgress of every member (constant within one execute)
    q: object = None         # (perm, offsets, xp) of the current expert launch
    resume_q: object = None  # queues a preempted expert stage resumes with (qmoe_resume_point)


class InferenceEngine:
    """Single-host-thread engine; all tensor work is enqueued on the current CUDA stream."""

    def __init__(self, model, cache, clock, cost_model: CostModel = CostModel(), max_batch_size: int = 32,
                 log: Optional[list] = None, device_preempt: Optional[bool] = None):
        cost_model.validate()
        self.model = model
        self.cache = cache
        self.clock = clock
        self.cost = cost_model
        self.max_batch_size = max_batch_size
        self.max_stage_cost = 0.0
        self.log = log  # decision log: per-expert queue contents ("Q" events) when not None
        self._batch_counter = 0
        self.stats = {"iterations": 0, "preemptions": 0, "expert_launches": 0, "zero_copy_restores": 0,
                      "copy_restores": 0}
        # Device-resident preemption (flag polled by the grouped kernel) is the wall-clock default;
        # virtual-clock runs decide the boundary before the launch so they replay the reference
        # decision log exactly.
        self._device_preempt = (not getattr(clock, "virtual", True)) if device_preempt is None else device_preempt
        self._pinned_off = None
        self._flags = None
        self._flag_slot = 0
        self._on_expert_report = None
        self._launch_seq = 0
        self._stop_marks: list = []
        self._preempt_at = {"ATTENTION": 0, "ROUTER": 0}
        self.stats["reports_at_drain"] = 0
        self._active = None   # the running iteration's preempt flag (device-preempt mode)
        self.in_rollback = False
        self._flag = None
        self._prev = None     # the previous layer's state within the running iteration
        self._ring_i = 0
        self._last_hit: list = []
        # wall clock: the reports of the experts holding the last report_tail of a launch's rows
        # are answered without waiting for their drain (1.0: none waits; see
        # _experts_device_preempt)
        self.report_tail = float(os.environ.get("QMOE_REPORT_TAIL", "1.0"))
        # Report elision (set by the driver, wall clock only): when every answer within an iteration
        # is provably the answer of its first report -- a built-in policy reads only the queues and
        # the batch's priorities, and the driver admits no request inside an iteration (the arrival
        # watcher defers admission to the iteration start and stops the GPU through the device flag)
        # -- the reports after a CONTINUE first report are answered CONTINUE without the callback
        # round trip (Qwen: 66 reports per layer).  Rollback reports are always delivered.
        self.elide_reports = False
        self._elide = False
        self.stats["reports_elided"] = 0

    def next_batch_id(self) -> int:
        self._batch_counter += 1
        return self._batch_counter

    def restore(self, sequences: list[Sequence]) -> Batch:
        """Rebuild a batch from checkpoints at one position; charges restore_cost per member."""
        if not sequences:
            raise ValueError("nothing to restore")
        positions = set()
        for seq in sequences:
            if seq.checkpoint is None:
                raise ValueError(f"sequence {seq.id} has no checkpoint to restore")
            positions.add(seq.checkpoint.position)
        if len(positions) != 1:
            raise ValueError(f"checkpoints at mixed positions {sorted(positions)}; group them first")
        batch = batch_form(sequences, sequences[0].phase, self.max_batch_size, self.next_batch_id())
        self.clock.advance(self.cost.restore_cost * len(sequences))
        return batch

    # ------------------------------------------------------------------------------------------
    def execute(self, batch: Batch, sequences: list[Sequence], on_report: ReportCallback,
                on_expert_report: Optional[Callable[[EngineReport, Optional[SchedulerDirective]],
                                                    SchedulerDirective]] = None) -> IterationOutcome:
        """on_expert_report (optional, wall-clock device-preempt path): answers one expert-boundary
        report given the previous expert report's answer in the same launch (None for the first),
        so a driver may skip re-running a pure policy when nothing changed in between."""
        self._on_expert_report = on_expert_report
        if [s.id for s in sequences] != batch.members:
            raise SimulationError("sequence list does not match batch members")
        if hasattr(self.model, "pass_serial"):
            self.model.pass_serial += 1  # per-pass buffers of the plugin (DecoderMoEModel.new_expert_state)
        st = self._init_state(sequences)
        layer, stage = batch.layer_cursor, batch.stage_cursor
        if stage not in (Stage.ATTENTION, Stage.ROUTER, Stage.EXPERTS):
            raise SimulationError(f"batch cursor at non-executable stage {stage}")
        self.stats["iterations"] += 1
        if not self._device_preempt:
            return self._run(batch, st, layer, stage, on_report)
        self._begin_iteration()
        try:
            return self._run(batch, st, layer, stage, on_report)
        finally:
            self._end_iteration()

    def _ask(self, on_report: ReportCallback, report_fn):
        """Deliver one report (report_fn builds it) unless this iteration's reports are elided."""
        if self._elide:
            self.stats["reports_elided"] += 1
            return SchedulerDirective.CONTINUE
        d = on_report(report_fn())
        if self.elide_reports and d is not PREEMPT:
            self._elide = True
        return d

    def _run(self, batch: Batch, st: _State, layer: int, stage: Stage, on_report: ReportCallback) -> IterationOutcome:
        m = self.model
        L = m.config.num_layers
        dev = self._device_preempt
        self._elide = False
        while layer < L:
            if stage is Stage.ATTENTION:
                st.x, st.res = m.attention_batch(layer, st.h, st.members, self.cache)
                st.h = None
                if not self._elide:
                    scanned = sum(self.cache.count(s.cache_handle, layer) for s in st.seqs)
                    self._charge(self.cost.attention_cost(st.T, scanned))
                if self._ask(on_report, lambda: self._report(batch, Stage.ATTENTION, layer, st)) is PREEMPT:
                    if dev and self._prev_voided(sync=True):
                        return self._preempt_void(batch, on_report, layer)
                    self._preempt_at["ATTENTION"] += 1
                    return self._preempt(st, layer, Stage.ROUTER)
                stage = Stage.ROUTER

            if stage is Stage.ROUTER:
                st.ids, st.w = m.route_batch(layer, st.x)
                st.y, st.cursor = m.new_expert_state(st.T)
                self._charge(self.cost.router_cost)
                if self._ask(on_report, lambda: self._report(batch, Stage.ROUTER, layer, st)) is PREEMPT:
                    if dev and self._prev_voided(sync=True):
                        return self._preempt_void(batch, on_report, layer)
                    self._preempt_at["ROUTER"] += 1
                    return self._preempt(st, layer, Stage.EXPERTS)
                stage = Stage.EXPERTS

            # EXPERTS: queue build for the pending slots (or, resuming a whole preempted batch, the
            # preempted launch's queues with the completed experts emptied), boundary decisions,
            # one grouped launch.
            if st.resume_q is not None:
                perm, offsets, xp = st.resume_q
                st.resume_q = None
            else:
                perm, offsets, xp = m.permute(st.ids, st.cursor, st.x)
            st.q = (perm, offsets, xp)
            if dev:
                stop_dev, preempted = self._experts_device_preempt(batch, st, layer, perm, offsets, xp, on_report)
                if preempted is None:  # the previous layer's launch was stopped by the device flag
                    return self._preempt_void(batch, on_report, layer)
            else:
                stop_dev, preempted = self._experts_host_boundary(batch, st, layer, perm, offsets, xp, on_report)
            if preempted:
                self._resume_point(st, stop_dev)
                return self._preempt(st, layer, Stage.EXPERTS)
            st.h = m.combine_batch(layer, st.y, st.w, st.res, st.x)
            if dev:
                self._prev = _State(st.seqs, st.members, st.T, None, st.x, st.res, st.ids, st.w, st.y, st.cursor,
                                    st.progress)
                self._prev.layer, self._prev.ring, self._prev.hit = layer, self._ring_i, self._last_hit
                self._prev.q = st.q
            st.q = None
            st.x = st.res = st.ids = st.w = st.y = st.cursor = None
            layer += 1
            stage = Stage.ATTENTION

        rows = [mr.row0 + mr.n - 1 for mr in st.members]
        tokens = m.emit_batch(st.h, rows)  # synchronises: the last expert launch's stop is in
        if dev and self._prev_voided(sync=True):
            return self._preempt_void(batch, on_report, L)
        return Completed({s.id: int(t) for s, t in zip(st.seqs, tokens)})

    # ------------------------------------------------------------------------------------------
    # Device-resident preemption (wall clock).  One preempt flag per iteration, polled by every
    # grouped expert launch of the iteration at each expert boundary: 0 = run; s > 0 = stop at the
    # first boundary >= s; -1 = a launch of this iteration stopped early, so everything enqueued
    # behind it is void (later launches claim nothing, guarded K/V appends skip).  It is raised
    # either by the host at an expert report (PREEMPT answer) or, with no host round trip, by
    # raise_arrival_flag() -- the serving driver's arrival watcher, the moment an LS request
    # arrives (qllm_policy preempts for a fresh LS prefill, reference sched.py:57-70).  The host
    # keeps running ahead of the GPU (it enqueues layer l+1 while layer l's experts run) and learns
    # that layer l stopped one layer later, at layer l+1's queue-length read; it then rolls the
    # iteration back to layer l's expert boundary (_preempt_void).
    def _begin_iteration(self) -> None:
        import torch

        m = self.model
        if self._flags is None:
            dev = m.device
            # Flags live in DEVICE memory (an L2 hit for the polling SMs; host-mapped memory polled
            # by every CTA serialises on PCIe).  A ring of slots, one per iteration; slot i+512 is
            # zeroed in stream order so a slot is clean long before reuse.
            self._flags = torch.zeros(1024, dtype=torch.int32, device=dev)
            self._sig_src = torch.zeros(1024, dtype=torch.int32, pin_memory=True)
            self._sig_stream = torch.cuda.Stream(device=dev)
            self._one = torch.ones(1, dtype=torch.int32, pin_memory=True)
            self._watch_stream = torch.cuda.Stream(device=dev)
            # per launch: where it stopped (device copy for the cursor advance, pinned copy + event
            # for the host), a ring of 256
            # where each launch stopped: the kernel's cursor_out points into this pinned ring (the
            # last CTA out stores it through UVA), read by the host after the next queue-length
            # sync and by the resume-point kernel -- no extra launch or copy per layer
            self._stop_pinned = torch.zeros(256, dtype=torch.int32, pin_memory=True)
            # progress words: written by the GPU (system-scope stores), read here through numpy
            self._progress = torch.zeros(64, dtype=torch.int32, pin_memory=True)
            self._progress_np = self._progress.numpy()
        if self._stop_marks and self._stop_marks[-1][4] is None:
            self._resolve_stop_marks()  # before the launches of this iteration reuse ring slots
        slot = self._flag_slot = (self._flag_slot + 1) % 1024
        self._flags[(slot + 512) % 1024].zero_()
        self._flag = self._flags[slot:slot + 1]
        self._prev = None
        if hasattr(m, "preempt_guard"):
            m.preempt_guard = self._flag
        self._active = self._flag  # visible to raise_arrival_flag (another thread)

    def _end_iteration(self) -> None:
        self._active = None
        self._prev = None
        if hasattr(self.model, "preempt_guard"):
            self.model.preempt_guard = None

    def raise_arrival_flag(self) -> bool:
        """Thread-safe: ask the running iteration's expert launches to stop at their next expert
        boundary (flag := 1, an async H2D write on this thread's own stream).  Returns False when no
        iteration is running (the arrival is then seen at the next report).  A write landing on an
        iteration that already ended, or on a flag already at -1, is harmless: slots are reused 512
        iterations later, and a void iteration is rolled back by the host regardless."""
        import torch

        flag = self._active
        if flag is None:
            return False
        with torch.cuda.stream(self._watch_stream):
            flag.copy_(self._one, non_blocking=True)
        self.stats["arrival_flags"] = self.stats.get("arrival_flags", 0) + 1
        return True

    def _prev_voided(self, sync: bool) -> bool:
        """Did the previous layer's expert launch of this iteration stop before its last expert?"""
        p = self._prev
        if p is None:
            return False
        if sync:  # a host-side PREEMPT answer: the iteration ends here anyway
            import torch

            torch.cuda.current_stream().synchronize()
        return int(self._stop_pinned[p.ring]) < self.model.config.num_experts

    def _preempt_void(self, batch: Batch, on_report: ReportCallback, layer: int) -> Preempted:
        """Roll back to the expert boundary where the previous layer's launch stopped: undo the
        K/V reservation of the layer enqueued behind it (its guarded append was skipped), deliver
        the report of the last expert that completed (the policy admits the arrival that raised
        the flag and answers PREEMPT), advance that layer's cursors on the device, checkpoint."""
        p = self._prev
        m = self.model
        if layer < m.config.num_layers:
            self.cache.unreserve_batch([mr.seq.cache_handle for mr in p.members], layer, [mr.n for mr in p.members])
        stop = int(self._stop_pinned[p.ring])
        done = [e for e in p.hit if e < stop]
        rep = (self._report(batch, Stage.EXPERTS, p.layer, p, expert_id=done[-1]) if done
               else self._report(batch, Stage.ROUTER, p.layer, p))
        self.in_rollback = True  # the driver admits arrivals up to this report (Simulation._admission_time)
        try:
            if on_report(rep) is not PREEMPT:
                self.stats["flag_policy_disagree"] = self.stats.get("flag_policy_disagree", 0) + 1
        finally:
            self.in_rollback = False
        self._resume_point(p, self._stop_pinned[p.ring:p.ring + 1])
        self._preempt_at["EXPERT_DEVICE_FLAG"] = self._preempt_at.get("EXPERT_DEVICE_FLAG", 0) + 1
        return self._preempt(p, p.layer, Stage.EXPERTS)

    # ------------------------------------------------------------------------------------------
    def _experts_host_boundary(self, batch, st, layer, perm, offsets, xp, on_report):
        """Virtual-clock / exact mode: read the queue lengths (one small D2H), answer every
        expert-boundary report on the host, then ONE launch for experts [0, stop)."""
        m = self.model
        E = m.config.num_experts
        off = offsets.tolist()
        counts = [off[e + 1] - off[e] for e in range(E)]
        slots = perm[: off[E]].tolist() if (self.log is not None and off[E]) else None
        stop, preempted = E, False
        for e in range(E):
            n = counts[e]
            if n == 0:
                continue
            if slots is not None:
                self._log_queue(st, layer, e, slots[off[e]:off[e] + n])
            self._charge(self.cost.expert_cost(n))
            if self._on_report(batch, st, layer, e, on_report) is PREEMPT:
                stop, preempted = e + 1, True
                break
        stop_dev = None
        if off[E]:
            stop_dev = m.run_experts(layer, xp, offsets, perm, st.y, 0, stop)
            self.stats["expert_launches"] += 1
        return stop_dev, preempted

    def _experts_device_preempt(self, batch, st, layer, perm, offsets, xp, on_report):
        """Device-resident preemption: launch ALL experts at once under the iteration's preempt
        flag (polled by the kernel whenever a CTA moves to a new expert) with per-expert progress
        words in pinned host memory (the kernel publishes a launch sequence number into
        progress[e] when expert e's last output row is stored).  Returns (stop_dev, preempted),
        preempted None when the PREVIOUS layer's launch turned out to have stopped early.

        Wall clock: the expert reports are answered right after the queue lengths arrive, while
        the grouped GEMM runs; with report_tail < 1 the report of expert e instead waits until the
        GPU has drained expert e (the host polls progress[e]; arrivals are admitted up to that
        moment, as in the reference where the report follows the drain, engine.py:204-219,
        sim.py:135-142) -- measured to cost ~30% of decode throughput, because the host then
        stops running ahead of the GPU.  An LS arrival needs neither: the serving driver raises
        the flag itself (raise_arrival_flag).  A PREEMPT answer raises the flag to "stop at the
        first boundary >= e+1": the kernel stops there and writes where it stopped (cursor_out),
        from which the per-token cursors advance on the device.

        Virtual clock (tests): reports are answered right after the launch, one by one."""
        import torch

        m = self.model
        E = m.config.num_experts
        if self._pinned_off is None or self._pinned_off.numel() != E + 1:
            self._pinned_off = torch.empty(E + 1, dtype=torch.int32, pin_memory=True)
            self._off_ready = torch.cuda.Event()
        self._pinned_off.copy_(offsets, non_blocking=True)
        self._off_ready.record()
        flag = self._flag
        self._launch_seq += 1
        seq = self._launch_seq
        ring = self._ring_i = (self._ring_i + 1) % 256
        stop_dev = m.run_experts(layer, xp, offsets, perm, st.y, 0, E, preempt_flag=flag, progress=self._progress,
                                 progress_seq=seq, cursor_out=self._stop_pinned[ring:ring + 1])
        self.stats["expert_launches"] += 1
        self._off_ready.synchronize()  # waits for the permute only; the GEMM keeps running
        if self._prev_voided(sync=False):  # the permute ran after the previous launch: its stop is in
            return stop_dev, None
        off = self._pinned_off.tolist()
        hit = self._last_hit = [e for e in range(E) if off[e + 1] > off[e]]
        stop = None
        wall = not getattr(self.clock, "virtual", True)
        if self._elide:
            self.stats["reports_elided"] += len(hit)
        elif self._on_expert_report is not None and wall:
            prog = self._progress_np
            tail_rows = self.report_tail * off[E]
            last = None
            for i, e in enumerate(hit):
                if off[E] - off[e + 1] >= tail_rows and prog[e] != seq:
                    self._await_progress(prog, e, seq)
                    self.stats["reports_at_drain"] += 1
                d = self._on_expert_report(self._report(batch, Stage.EXPERTS, layer, st, expert_id=e), last)
                if d is PREEMPT:
                    stop = e + 1
                    break
                last = d
        else:
            for e in hit:
                self._charge(self.cost.expert_cost(off[e + 1] - off[e]))
                if self._on_report(batch, st, layer, e, on_report) is PREEMPT:
                    stop = e + 1
                    break
        if stop is not None:
            # raise "stop at the first boundary >= stop" while the kernel runs: an async H2D write
            # on a side stream (copy engine), so the reported expert always completes
            running = self._progress_np[hit[-1]] != seq
            slot = self._flag_slot
            self._sig_src[slot] = stop
            with torch.cuda.stream(self._sig_stream):
                flag.copy_(self._sig_src[slot:slot + 1], non_blocking=True)
            # where the kernel really stopped: its ring slot, read once the launch is done (the next
            # iterations' _begin_iteration, or preemption_positions)
            ev = torch.cuda.Event()
            ev.record()
            self._stop_marks.append([self._ring_i, hit[-1] + 1, running, ev, None])
            return stop_dev, True
        return stop_dev, False

    def _resume_point(self, st: _State, stop_dev) -> None:
        """Cursors advance to the stop on the device.  With a model exposing resume_point, the
        preempted launch's perm / Xp are kept with the completed experts' queues emptied, so a
        restore of the whole batch resumes without a re-permute (engine.py:312-328 re-enqueues
        only pending experts; the pending slots of each expert are the same rows, same order)."""
        rp = getattr(self.model, "resume_point", None)
        if rp is None or st.q is None:
            self.model.advance_cursor(st.cursor, stop_dev)
            return
        perm, offsets, xp = st.q
        st.resume_q = (perm, rp(st.cursor, stop_dev, offsets), xp)

    def _resolve_stop_marks(self) -> None:
        for mark in self._stop_marks:
            if mark[4] is None and mark[3].query():
                mark[4] = int(self._stop_pinned[mark[0]])
                mark[3] = None

    def _await_progress(self, prog, e: int, seq: int, timeout_s: float = 30.0) -> None:
        """Spin on the pinned progress word of expert e (a plain host read, ~100 ns)."""
        if prog[e] == seq:
            return
        t_end = time.perf_counter() + timeout_s
        n = 0
        while prog[e] != seq:
            n += 1
            if (n & 0xFFFF) == 0 and time.perf_counter() > t_end:
                raise SimulationError(f"expert {e} never reported completion (launch {seq})")

    def preemption_positions(self) -> dict:
        """Where preemptions landed: ATTENTION / ROUTER reports, or an expert report -- and for those,
        whether the device flag stopped the grouped kernel before its last hit expert
        (EXPERT_MID_LAUNCH) or the kernel had already covered every hit expert (EXPERT_END_OF_LAUNCH).
        Synchronises the device once."""
        import torch

        torch.cuda.synchronize()
        self._resolve_stop_marks()
        out = dict(self._preempt_at)
        for (_, end, running, _, got) in self._stop_marks:
            key = "EXPERT_MID_LAUNCH" if got < end else "EXPERT_END_OF_LAUNCH"
            out[key] = out.get(key, 0) + 1
            out["flag_raised_while_running"] = out.get("flag_raised_while_running", 0) + int(running)
        out["expert_reports_answered_at_drain"] = self.stats["reports_at_drain"]
        return out

    def _on_report(self, batch, st, layer, expert, on_report):
        return on_report(self._report(batch, Stage.EXPERTS, layer, st, expert_id=expert))

    def _init_state(self, sequences: list[Sequence]) -> _State:
        members, row = [], 0
        inputs = []
        for seq in sequences:
            if seq.cache_handle is None or not self.cache.has_handle(seq.cache_handle):
                raise StateCorruptionError(f"sequence {seq.id} has no registered cache handle")
            toks = seq.iteration_input()
            if seq.checkpoint is not None and seq.checkpoint.num_tokens != len(toks):
                raise StateCorruptionError(f"sequence {seq.id}: checkpoint does not match iteration input")
            inputs.append(toks)
            members.append(MemberRows(seq, row, len(toks)))
            row += len(toks)
        st = _State(list(sequences), members, row)
        st.progress = BatchProgress(MemberProgress(s.id, s.priority, s.phase, len(s.generated)) for s in sequences)
        ckpts = [s.checkpoint for s in sequences]
        if ckpts[0] is None:
            st.h = self.model.embed_batch([t for toks in inputs for t in toks])
            return st
        st.x, st.res = self._gather(ckpts, "hidden"), self._gather(ckpts, "residual")
        if ckpts[0].ids is not None:
            st.ids, st.w = self._gather(ckpts, "ids"), self._gather(ckpts, "weights")
            st.y, st.cursor = self._gather(ckpts, "y"), self._gather(ckpts, "cursor")
            o = ckpts[0].origin if self._contiguous(ckpts) else None
            if o is not None and o[1] == 0 and ckpts[-1].origin[2] == o[0].T and o[0].resume_q is not None:
                st.resume_q = o[0].resume_q  # the whole preempted batch, in its order: reuse its queues
                self.stats["queue_reuse_resumes"] = self.stats.get("queue_reuse_resumes", 0) + 1
        self.stats["zero_copy_restores" if self._contiguous(ckpts) else "copy_restores"] += 1
        for s in sequences:
            s.checkpoint = None  # checkpoints live only while preempted
        return st

    @staticmethod
    def _contiguous(ckpts: list[Checkpoint]) -> bool:
        o = [getattr(c, "origin", None) for c in ckpts]
        if any(x is None for x in o) or any(x[0] is not o[0][0] for x in o):
            return False
        return all(o[i][2] == o[i + 1][1] for i in range(len(o) - 1))

    def _gather(self, ckpts: list[Checkpoint], name: str):
        if self._contiguous(ckpts):
            st, r0, r1 = ckpts[0].origin[0], ckpts[0].origin[1], ckpts[-1].origin[2]
            k = self.model.config.top_k
            full = getattr(st, {"hidden": "x", "residual": "res", "weights": "w"}.get(name, name))
            return full[r0 * k:r1 * k] if name == "y" else full[r0:r1]
        return self.model.cat_rows([getattr(c, name) for c in ckpts])

    def _charge(self, cost_ms: float) -> None:
        self.clock.advance(cost_ms)
        if cost_ms > self.max_stage_cost:
            self.max_stage_cost = cost_ms

    def _report(self, batch: Batch, stage: Stage, layer: int, st: _State,
                expert_id: Optional[int] = None) -> EngineReport:
        return EngineReport(batch.batch_id, stage, layer, self.clock.now, st.progress, expert_id)

    def _log_queue(self, st: _State, layer: int, expert: int, slots: list[int]) -> None:
        k = self.model.config.top_k
        owner = []
        for mr in st.members:
            owner += [(mr.seq.id, t) for t in range(mr.n)]
        self.log.append(["Q", layer, expert, [list(owner[s // k]) for s in slots]])

    def _preempt(self, st: _State, layer: int, resume_stage: Stage) -> Preempted:
        k = self.model.config.top_k
        routed = resume_stage > Stage.ROUTER
        out: dict[int, Checkpoint] = {}
        for mr in st.members:
            r = slice(mr.row0, mr.row0 + mr.n)
            ck = Checkpoint(layer_index=layer, stage=resume_stage, hidden=st.x[r], residual=st.res[r],
                            ids=st.ids[r] if routed else None, weights=st.w[r] if routed else None,
                            y=st.y[mr.row0 * k:(mr.row0 + mr.n) * k] if routed else None,
                            cursor=st.cursor[r] if routed else None)
            ck.origin = (st, mr.row0, mr.row0 + mr.n)
            ck.validate()
            mr.seq.checkpoint = ck
            out[mr.seq.id] = ck
        self.stats["preemptions"] += 1
        self._charge(self.cost.checkpoint_cost)
        return Preempted(out)
