import os, sys, socket
import torch, torch.distributed as dist, torch.multiprocessing as mp
sys.path.insert(0, "/root/repo") if os.path.exists("/root/repo") else None
sys.path.insert(0, os.getcwd())
D, F, E, K, SEED = 512, 1024, 8, 2, 11

def worker(rank, world, port, q, hb, mt):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2503_09304_b200.ep import PeerExpertParallelMoE
    from paper_2503_09304_b200 import kernels as Kn
    blk = PeerExpertParallelMoE(D, F, E, K, rank, world, max_tokens=mt, device=torch.device("cuda", 0), host_barrier=hb).init_random(SEED)
    g = torch.Generator().manual_seed(1000 * rank)
    T = [24, 31][rank]
    x = torch.randn((T, D), generator=g).bfloat16().cuda()
    out = blk(x, residual=x)
    torch.cuda.synchronize()
    ids, w = Kn.router(x, blk.w_router, K)
    q.put((rank, x.float().cpu().numpy(), out.float().cpu().numpy(), ids.cpu().numpy(), None))
    dist.barrier(); dist.destroy_process_group()

if __name__ == "__main__":
    from paper_2503_09304_b200.moe_block import SparseMoeBlock
    hb = sys.argv[1] == "host"; mt = int(sys.argv[2])
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn"); q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, port, q, hb, mt)) for r in range(2)]
    [p.start() for p in ps]
    res = [q.get(timeout=120) for _ in range(2)]
    [p.join() for p in ps]
    ref = SparseMoeBlock(D, F, E, K, device="cuda").init_random(SEED)
    for rank, x, out, ids, y in res:
        x, out, ids = torch.tensor(x).bfloat16(), torch.tensor(out), torch.tensor(ids)
        T = x.shape[0]
        r = (ref(x.cuda().view(1, T, D)).view(T, D).float() + x.cuda().float()).cpu()
        bad = ((out - r).norm(dim=1) / r.norm(dim=1)) > 1e-2
        print("rank", rank, "bad tokens", bad.nonzero().flatten().tolist(), "ids of bad", ids[bad].tolist()[:8])
