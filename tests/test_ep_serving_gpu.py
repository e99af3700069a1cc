"""Expert-parallel serving on the GPU path (ep_serving.ExpertParallelDecoder), world size 2 on ONE
B200: two processes share cuda:0, each holds half of the experts (tcgen05 grouped GEMM on its own
experts only), and the output rows are all-gathered through CUDA-IPC-mapped receive buffers with
device flag barriers -- the NVLink data path of an 8-GPU box, exercised between two contexts.
Every rank drives the real engine + scheduler + driver on the same trace with a virtual clock and
a seeded random preemption policy (preemptions at every kind of boundary, partial launches,
merged resumes).  Checked: each rank's decision log, tokens and job records equal the
single-process DecoderMoEModel run on the same weights, bit for bit; a Qwen-like config puts the
shared expert's sub-experts on the second rank."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _cfg(kind):
    from paper_2503_09304_b200 import kernels as K
    from paper_2503_09304_b200.mixtral import DecoderConfig

    if kind == "mixtral":
        return DecoderConfig("tiny-mixtral", 2, 512, 1024, 8, 2, 4, 2, 128, 1024, 1e6, 1e-5)
    return DecoderConfig("tiny-qwen", 2, 512, 512, 6, 2, 4, 4, 128, 1024, 1e6, 1e-6,
                         route_mode=K.ROUTE_SOFTMAX_TOPK, shared_ffn_dim=1024)


def _trace():
    from paper_2503_09304_b200.workload import WorkloadSpec, trace_for_rate

    spec = WorkloadSpec(duration_s=1.5, ls_fraction=0.3, prompt_mean=24, prompt_sigma=0.7, prompt_bounds=(2, 96),
                        output_mean=6, output_sigma=0.5, output_bounds=(1, 12))
    return trace_for_rate(spec, 12.0, seed=4)


def _run(model, clock=None):
    import numpy as np

    from paper_2503_09304_b200.core import SchedulerDirective
    from paper_2503_09304_b200.sim import Simulation

    rng = np.random.default_rng(17)

    def policy(report, queues):  # seeded coin per report (the reference's test policy)
        return (SchedulerDirective.PREEMPT_AT_NEXT_BOUNDARY if rng.random() < 0.15
                else SchedulerDirective.CONTINUE)

    sim = Simulation(_trace(), model=model, scheduler="qllm", max_batch_size=6, policy=policy, record_log=True,
                     clock=clock)
    res = sim.run()
    return {"log": [list(e) for e in res.log], "tokens": {k: s.generated for k, s in sorted(res.sequences.items())},
            "records": [[r.seq_id, r.first_token_ms, r.finish_ms] for r in res.records],
            "preemptions": res.probes.preemptions}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, kind, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2503_09304_b200.ep_serving import ExpertParallelDecoder

        model = ExpertParallelDecoder(_cfg(kind), rank, world, device=torch.device("cuda", 0), seed=5,
                                      barrier_timeout_s=60.0)
        out = _run(model)
        # the same trace on the ranks' shared wall clock: timing-dependent decisions, but every rank
        # must take the same ones (replicated state, one clock)
        from paper_2503_09304_b200.ep_serving import LockstepClock

        lock = _run(model, clock=LockstepClock())
        out["lockstep_log"] = lock["log"]
        out["lockstep_tokens"] = lock["tokens"]
        torch.cuda.synchronize()
        out["barrier_error"] = int(model.error.item())
        out["exchanges"] = model.stats["exchanges"]
        q.put((rank, out, None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # noqa: BLE001 - report to the parent instead of hanging it
        import traceback

        q.put((rank, None, f"{exc!r}\n{traceback.format_exc()}"))


@pytest.mark.parametrize("kind", ["mixtral", "qwen"])
def test_expert_parallel_serving_equals_single_gpu(cuda, kind):
    from paper_2503_09304_b200.mixtral import DecoderMoEModel

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        rank, out, err = q.get(timeout=600)
        assert err is None, f"rank {rank}: {err}"
        got[rank] = out
    for p in procs:
        p.join(timeout=120)
    want = _run(DecoderMoEModel(_cfg(kind), device=torch.device("cuda", 0), seed=5))
    assert want["preemptions"] > 0
    for rank in range(world):
        g = got[rank]
        assert g["barrier_error"] == 0 and g["exchanges"] > 0
        assert g["log"] == want["log"], f"rank {rank}: decision log differs from the single-GPU run"
        assert g["tokens"] == want["tokens"]
        assert g["records"] == want["records"]
    assert got[0]["lockstep_log"] == got[1]["lockstep_log"] and len(got[0]["lockstep_log"]) > 0
    assert got[0]["lockstep_tokens"] == got[1]["lockstep_tokens"]
