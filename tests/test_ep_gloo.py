"""Expert-parallel exchange logic under gloo, world_size 2, on CPU: the EP block's dispatch /
regroup / combine must reproduce the single-process MoE layer exactly (same rows per expert in
the same order).  Kernels are replaced by a CPU double built on the oracle (test-only)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_09304_b200.ep import ExpertParallelMoE, dispatch_tables, expert_bounds, regroup_index


class CpuOps:
    """CPU stand-ins for the libqmoe wrappers (same signatures), oracle-backed."""

    @staticmethod
    def router(x, wr, k, mode=0):
        from oracle import moe_oracle as om

        ids, w = om.route_many(wr.double().numpy(), x.double().numpy(), k)
        return torch.tensor(ids, dtype=torch.int32), torch.tensor(w, dtype=torch.float32)

    @staticmethod
    def permute(ids, E, cursor=None, x=None):
        from oracle import moe_oracle as om

        perm, offsets = om.permute(ids.numpy(), None, E)
        T, k = ids.shape
        p = torch.zeros(T * k, dtype=torch.int32)
        p[: len(perm)] = torch.tensor(perm, dtype=torch.int32)
        xp = torch.zeros((T * k, x.shape[1]), dtype=x.dtype)
        xp[: len(perm)] = x[torch.tensor(perm, dtype=torch.long) // k]
        return p, torch.tensor(offsets, dtype=torch.int32), xp

    @staticmethod
    def gather_rows(src, idx):
        return src[idx.long()]

    @staticmethod
    def scatter_rows(src, idx, out):
        out[idx.long()] = src
        return out

    @staticmethod
    def expert_ffn(variant, xp, offsets, perm, w1, w2, y, act_ws=None, **kw):
        from oracle import moe_oracle as om

        off = offsets.tolist()
        for e in range(w1.shape[0]):
            a, b = off[e], off[e + 1]
            if a < b:
                out = om.expert_swiglu(w1[e].double().numpy(), w2[e].double().numpy(), xp[a:b].double().numpy())
                y[perm[a:b].long()] = torch.tensor(out, dtype=y.dtype)

    @staticmethod
    def combine(y, w, res):
        T, k = w.shape
        out = (w[:, :, None].double() * y.double().reshape(T, k, -1)).sum(1)
        if res is not None:
            out = out + res.double()
        return out.to(y.dtype)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


D, F, E, K = 32, 48, 6, 2


def _weights():
    g = torch.Generator().manual_seed(7)
    return (torch.randn((E, D), generator=g) / D ** 0.5, torch.randn((E, 2 * F, D), generator=g) / D ** 0.5,
            torch.randn((E, D, F), generator=g) / F ** 0.5)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wr, gu, dn = _weights()
    blk = ExpertParallelMoE(D, F, E, K, rank, world, device=torch.device("cpu"), dtype=torch.float32, ops=CpuOps)
    blk.load_full(wr, gu, dn)
    x = torch.randn((20 + 7 * rank, D), generator=torch.Generator().manual_seed(100 + rank))
    out = blk(x, residual=x)
    q.put((rank, x.numpy(), out.numpy()))
    dist.destroy_process_group()


def _single(x):
    wr, gu, dn = _weights()
    ids, w = CpuOps.router(x, wr, K)
    perm, offsets, xp = CpuOps.permute(ids, E, x=x)
    y = torch.zeros((x.shape[0] * K, D))
    CpuOps.expert_ffn(1, xp, offsets, perm, gu, dn, y)
    return CpuOps.combine(y, w, x).numpy()


@pytest.mark.parametrize("world", [2])
def test_ep_matches_single_process_under_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, x, out in got:
        np.testing.assert_allclose(out, _single(torch.tensor(x)), rtol=0, atol=1e-6)


def test_expert_bounds_uneven():
    assert expert_bounds(8, 2) == [0, 4, 8]
    b = expert_bounds(60, 8)
    assert b[0] == 0 and b[-1] == 60 and {b[i + 1] - b[i] for i in range(8)} == {7, 8}


def test_regroup_index_orders_by_local_expert_then_source():
    counts = [[1, 2, 0, 3], [2, 0, 1, 1]]  # counts[src][e]
    idx, off = regroup_index(counts, 2, 4)
    # received: src0 -> e2:0 rows, e3:3 rows [0,1,2]; src1 -> e2:1 row [3], e3:1 row [4]
    assert idx == [3, 0, 1, 2, 4]
    assert off == [0, 1, 5]


@pytest.mark.parametrize("world,E", [(2, 8), (4, 8), (8, 60), (3, 5)])
def test_peer_dispatch_tables_match_regroup_order(world, E):
    """The peer-memory transport writes rows straight to their final receive position: for every
    owner, the (source, expert) blocks tile [0, received rows) exactly, in the same local-expert-major
    then source-rank order that regroup_index gives the all-to-all transport."""
    rng = np.random.default_rng(world * 100 + E)
    counts = rng.integers(0, 9, size=(world, E)).tolist()
    counts[0][0] = 0  # an empty (source, expert) block
    b = expert_bounds(E, world)
    for g in range(world):
        # position of every received row, keyed (expert, source, i)
        pos = {}
        for s in range(world):
            dest_rank, dest_base = dispatch_tables(counts, b, s)
            for e in range(b[g], b[g + 1]):
                assert dest_rank[e] == g
                for i in range(counts[s][e]):
                    pos[(e, s, i)] = dest_base[e] + i
        total = sum(counts[s][e] for s in range(world) for e in range(b[g], b[g + 1]))
        assert sorted(pos.values()) == list(range(total))
        order = [key for key, _ in sorted(pos.items(), key=lambda kv: kv[1])]
        assert order == sorted(order)  # expert, then source, then queue order
        idx, off = regroup_index(counts, b[g], b[g + 1])
        assert off[-1] == total
