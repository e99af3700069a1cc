"""Expert parallelism over peer memory (csrc/ep.cu), world size 2, on ONE B200: two processes share
cuda:0 and map each other's receive / slot / flag buffers through CUDA IPC exactly as two GPUs of
an NVSwitch box would: the dispatch kernel stores rows into the peer's receive buffer, the expert
GEMM epilogue stores outputs into the peer's slot buffer, and stream-ordered device flag barriers
(system-scope release/acquire on the peer's flags) order the phases.  gloo carries only the
host-side handle exchange and the per-layer counts all-gather.  Every rank's layer output must
match the single-process SparseMoeBlock on the same weights bit for bit: ids, routing weights,
per-expert queue order and the layer output.
The large case (> 512 received rows, 128/256-row tcgen05 tiles, several buffers in separate
allocations) is the one that caught an IPC-handle cache keyed on a handle prefix."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

D, F, E, K, SEED = 512, 1024, 8, 2, 11
TOKENS = {0: [24, 7, 40], 1: [31, 0, 9]}  # per rank, per forward call (uneven; one empty batch)
BIG = {0: [700, 64], 1: [513, 600]}      # > 512 received rows: the 128/256-row tcgen05 tiles


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs(rank, call, T):
    g = torch.Generator().manual_seed(1000 * rank + call)
    return torch.randn((T, D), generator=g).bfloat16()


def _worker(rank, world, port, q, transport):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2503_09304_b200.ep import ExpertParallelMoE, PeerExpertParallelMoE

        tokens = BIG if transport == "p2p-big" else TOKENS
        if transport.startswith("p2p"):
            blk = PeerExpertParallelMoE(D, F, E, K, rank, world, max_tokens=1024, device=torch.device("cuda", 0),
                                        barrier_timeout_s=60.0).init_random(SEED)
        else:  # the all-to-all-v transport; gloo stands in for NCCL (two ranks cannot share a GPU in NCCL)
            blk = ExpertParallelMoE(D, F, E, K, rank, world, device=torch.device("cuda", 0)).init_random(SEED)
            blk.barrier_failed = lambda: False
        outs = []
        for call, T in enumerate(tokens[rank]):
            x = _inputs(rank, call, T).cuda()
            o = blk(x, residual=x)
            ids, w, perm, offsets = blk.last_routing
            R = int(offsets[-1])
            outs.append((o.view(torch.int16).cpu().numpy(), ids.cpu().numpy(), w.cpu().numpy(),
                         perm[:R].cpu().numpy(), offsets.cpu().numpy()))
        torch.cuda.synchronize()
        q.put((rank, outs, blk.barrier_failed(), None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # noqa: BLE001 - report to the parent instead of hanging it
        q.put((rank, None, None, repr(exc)))


@pytest.mark.parametrize("transport", ["p2p", "p2p-big", "alltoall"])
def test_expert_parallel_matches_single_process(cuda, transport):
    from paper_2503_09304_b200 import kernels as Kn
    from paper_2503_09304_b200.moe_block import SparseMoeBlock

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, transport)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    errors = [e for (_, _, _, e) in got if e]
    assert not errors, errors
    ref_blk = SparseMoeBlock(D, F, E, K, device=cuda).init_random(SEED)
    tokens = BIG if transport == "p2p-big" else TOKENS
    for rank, outs, failed, _ in got:
        assert not failed, f"rank {rank}: a device barrier timed out"
        for call, T in enumerate(tokens[rank]):
            x = _inputs(rank, call, T).cuda()
            if T == 0:
                assert outs[call][0].shape == (0, D)
                continue
            o, ids, w, perm, offsets = outs[call]
            ref = ref_blk(x.view(1, T, D), residual=x.view(1, T, D)).view(T, D)
            rids, rw = ref_blk.last_routing
            rperm, roff, _ = Kn.permute(rids, E)
            R = int(roff[-1])
            # expert ids and per-expert queue order bit-exact under EP; the
            # outputs too (each expert sees the same rows; every row's K order and roundings are
            # those of the single-GPU launch)
            assert np.array_equal(ids, rids.cpu().numpy()), (rank, call)
            assert np.array_equal(w, rw.cpu().numpy()), (rank, call)
            assert np.array_equal(offsets, roff.cpu().numpy()) and np.array_equal(perm, rperm[:R].cpu().numpy())
            assert np.array_equal(o, ref.view(torch.int16).cpu().numpy()), (rank, call)


def test_device_flag_barrier_two_concurrent_ranks(cuda):
    """qmoe_ep_barrier with two 'ranks' on two streams of one process (both resident at once):
    60 epochs complete with no timeout and every flag ends at the last epoch; a rank whose peer
    never arrives times out into the error word instead of hanging."""
    from paper_2503_09304_b200 import kernels as Kn

    flags = [torch.zeros(2, dtype=torch.int32, device=cuda) for _ in range(2)]
    table = torch.tensor([f.data_ptr() for f in flags], dtype=torch.int64, device=cuda)
    err = torch.zeros(1, dtype=torch.int32, device=cuda)
    streams = [torch.cuda.Stream() for _ in range(2)]
    torch.cuda.synchronize()
    for epoch in range(1, 61):
        for me in range(2):
            with torch.cuda.stream(streams[me]):
                Kn.ep_barrier(table, me, 2, epoch, err, timeout_s=20.0)
    torch.cuda.synchronize()
    assert int(err) == 0
    assert [f.tolist() for f in flags] == [[60, 60], [60, 60]]
    Kn.ep_barrier(table, 0, 2, 61, err, timeout_s=0.2)  # rank 1 never arrives
    torch.cuda.synchronize()
    assert int(err) == 1


def _preempt_worker(rank, world, port, q, T, stop_local):
    """Each rank runs one layer with its local launch stopped at local boundary stop_local (the
    device flag preset), agrees on the global resume cursor with its peer, resumes the layer with
    that cursor (same routing, pending slots only), and returns the output bits plus an
    uninterrupted layer's for comparison."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2503_09304_b200.ep import PeerExpertParallelMoE

        dev = torch.device("cuda", 0)
        blk = PeerExpertParallelMoE(D, F, E, K, rank, world, max_tokens=1024, device=dev,
                                    barrier_timeout_s=60.0).init_random(SEED)
        x = _inputs(rank, 7, T).cuda()
        full = blk(x, residual=x).clone()
        ids, w = blk.last_routing[:2]
        blk.y.fill_(float("nan"))  # every slot must be rewritten by the preempted launch or the resume
        flag = torch.full((1,), stop_local, dtype=torch.int32, device=dev)
        stop = torch.zeros(1, dtype=torch.int32, device=dev)
        blk(x, residual=x, preempt_flag=flag, cursor_out=stop, routing=(ids, w))
        torch.cuda.synchronize()
        # global resume point: experts below it completed on every rank (a rank that ran past it
        # recomputes the rest -- same bits); the ranks' local stops are exchanged on the host here
        lo, hi = blk.e_lo, blk.e_hi
        mine = lo + int(stop) if int(stop) < hi - lo else E
        allst = [None] * world
        dist.all_gather_object(allst, mine)
        c = min(allst)
        cursor = torch.full((T,), c, dtype=torch.int32, device=dev)
        out = blk(x, residual=x, cursor=cursor, routing=(ids, w))
        torch.cuda.synchronize()
        q.put((rank, int(stop), c, torch.equal(out.view(torch.int16), full.view(torch.int16)), blk.barrier_failed(),
               None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # noqa: BLE001
        q.put((rank, None, None, None, None, repr(exc)))


@pytest.mark.parametrize("T,stop_local", [(40, 1), (700, 2), (600, 1)])
def test_expert_parallel_preemption_resume_is_bit_identical(cuda, T, stop_local):
    """Preemption under EP: each rank's grouped launch over its local experts stops
    at an expert boundary (device flag), the ranks resume from the common global cursor, and the
    layer output equals an uninterrupted layer's bit for bit on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_preempt_worker, args=(r, 2, port, q, T, stop_local)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    errors = [g[-1] for g in got if g[-1]]
    assert not errors, errors
    for rank, stop, c, same, failed, _ in got:
        assert not failed
        assert stop is not None and stop <= E // 2
        assert same, (rank, stop, c)
    assert any(g[2] < E for g in got)  # the launch really stopped before the last expert somewhere
