"""Expert-parallel serving (ep_serving.py) host logic under gloo on CPU, world 2 and 3: every rank
runs the REAL engine + scheduler + driver on the same trace, holds a contiguous block of experts,
runs only those experts of each launch and all-gathers the output rows, exactly as
ExpertParallelDecoder does on the GPU.  Checked:
  * each rank's decision log equals the reference's single-process log bit for bit (replicated
    decisions: no decision traffic is needed), preemption traces included;
  * at every combine, every slot of every token holds the output of its own expert (no slot
    missed or filled twice across preemptions, partial launches and merged resumes);
  * LockstepClock: all ranks read the same time at every sync.
The device plugin is the routing-replay double (tests/replay.py) -- test infrastructure only."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

TRACES = ["traceA_qllm", "traceB_qllm", "random0_qllm", "random3_qllm", "random6_qllm"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ep_replay_model(rec, rank, world):
    from replay import ReplayModel
    from paper_2503_09304_b200.ep import expert_bounds

    class EPReplayModel(ReplayModel):
        """Replay double with the expert stage of ExpertParallelDecoder: y[slot] = 1 + the slot's
        expert, computed only by the expert's owner, then all-gathered."""

        def __init__(self):
            super().__init__(rec)
            b = expert_bounds(self.config.num_experts, world)
            self.lo, self.hi = b[rank], b[rank + 1]
            self.exchanges = 0
            self.combines = 0

        def route_batch(self, layer, x):
            ids, w = super().route_batch(layer, x)
            self._ids = ids
            return ids, w

        def new_expert_state(self, T):
            return torch.zeros((T * self.config.top_k, 1)), torch.zeros(T, dtype=torch.int32)

        def run_experts(self, layer, xp, offsets, perm, y, e_begin, e_end, preempt_flag=None, **_):
            off = offsets.tolist()
            a, b = max(self.lo, e_begin), min(self.hi, e_end)
            for e in range(a, b):
                for r in range(off[e], off[e + 1]):
                    assert y[perm[r], 0] == 0, "slot computed twice"
                    y[perm[r], 0] = e + 1
            # all-gather of the rows (the GPU path pushes them over peer memory)
            parts = [torch.zeros_like(y) for _ in range(world)]
            dist.all_gather(parts, y)
            for e in range(e_begin, e_end):
                if a <= e < b:
                    continue
                for r in range(off[e], off[e + 1]):
                    y[perm[r], 0] = parts[next(g for g in range(world)
                                               if expert_bounds(self.config.num_experts, world)[g] <= e
                                               < expert_bounds(self.config.num_experts, world)[g + 1])][perm[r], 0]
            self.exchanges += 1
            return torch.tensor([e_end], dtype=torch.int32)

        def combine_batch(self, layer, y, w, res, x):
            assert bool((y[:, 0] > 0).all()), "combine reached with a slot never computed"
            self.combines += 1
            return super().combine_batch(layer, y, w, res, x)

    return EPReplayModel()


def _worker(rank, world, port, names, q):
    import sys

    sys.path.insert(0, os.path.dirname(__file__))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from replay import load_log, policy_for, trace_of
        from paper_2503_09304_b200.ep_serving import LockstepClock
        from paper_2503_09304_b200.sim import Simulation

        out = {}
        for name in names:
            rec = load_log(name)
            model = _ep_replay_model(rec, rank, world)
            sim = Simulation(trace_of(rec), model=model, scheduler=rec["scheduler"],
                             max_batch_size=rec["max_batch_size"], policy=policy_for(rec), record_log=True)
            res = sim.run()
            out[name] = {"same_as_reference": [list(e) for e in res.log] == [list(e) for e in rec["log"]],
                         "makespan": res.makespan_ms == rec["makespan_ms"], "exchanges": model.exchanges,
                         "combines": model.combines, "log_len": len(res.log)}
        clk = LockstepClock()
        reads = []
        for i in range(5):
            clk.advance(0.25)  # replicated engines charge the same cost-model ms between syncs
            clk.sync()
            reads.append(clk.now)
        t = torch.tensor(reads, dtype=torch.float64)
        allr = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allr, t)
        out["clock_syncs_monotone"] = all(reads[i] <= reads[i + 1] for i in range(4))
        out["clock_same_as_rank0"] = allr[0].tolist() == reads
        q.put((rank, out))
    except Exception as exc:  # noqa: BLE001 - report to the parent
        import traceback

        q.put((rank, {"error": f"{exc!r}\n{traceback.format_exc()}"}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ep_serving_replicates_the_reference_decision_log(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, TRACES, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for rank in range(world):
        assert "error" not in got[rank], got[rank].get("error")
        for name in TRACES:
            r = got[rank][name]
            assert r["same_as_reference"] and r["makespan"], (rank, name)
            assert r["exchanges"] == got[0][name]["exchanges"] > 0 and r["combines"] > 0
        assert got[rank]["clock_syncs_monotone"]
        assert got[rank]["clock_same_as_rank0"]
    for p in procs:
        assert p.exitcode == 0
