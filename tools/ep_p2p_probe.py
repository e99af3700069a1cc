"""Diagnostic: two processes on cuda:0 run the peer-memory EP block (Mixtral shape) for a few
calls at a given T and report per-call wall time and barrier status."""
import os, sys, time, socket
import torch, torch.distributed as dist, torch.multiprocessing as mp
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(rank, world, port, T, d, F, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2503_09304_b200.ep import PeerExpertParallelMoE
    blk = PeerExpertParallelMoE(d, F, 8, 2, rank, world, max_tokens=T, device=torch.device("cuda", 0),
                                barrier_timeout_s=float(os.environ.get("TMO", "10")),
                                host_barrier=os.environ.get("BARRIER") == "host").init_random(1)
    x = torch.randn((T, d), device="cuda").bfloat16()
    log = []
    for i in range(4):
        t0 = time.time()
        blk(x)
        torch.cuda.synchronize()
        log.append((round(time.time() - t0, 3), blk.barrier_failed()))
    q.put((rank, log))
    dist.destroy_process_group()


if __name__ == "__main__":
    T, d, F = (int(a) for a in sys.argv[1:4])
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn"); q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, port, T, d, F, q)) for r in range(2)]
    [p.start() for p in ps]
    print([q.get(timeout=600) for _ in range(2)], flush=True)
    [p.join() for p in ps]
