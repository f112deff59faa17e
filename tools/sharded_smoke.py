"""Two ranks sharing one GPU over gloo (the box has 1 GPU): ShardedIndexer.run / .decode
must equal the single-GPU engine.  Dev check for the multi-GPU host path."""
import os, sys, socket
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_07363_b200 import IndexerEngine
    from paper_2605_07363_b200.sharded import ShardedIndexer
    g = torch.Generator(device="cuda").manual_seed(0)
    L, H, d, k, B = 20000, 64, 128, 512, 1024
    K = torch.randn(L, d, device="cuda", generator=g).bfloat16()
    Q = torch.randn(L, H, d, device="cuda", generator=g).bfloat16()
    W = torch.softmax(torch.randn(L, H, device="cuda", generator=g), -1).float()
    ok = {}
    for m in (("misa", "dsa", "misa_hier") if world == 2 else ("misa",)):
        kw = dict(budget_k=k, active_heads_h=8, block_size=B, candidate_kprime=2048)
        ref = IndexerEngine(m, **kw).run(K, Q, W).topk
        sh = ShardedIndexer(m, world=world, rank=rank, **kw)
        Kbuf = K.clone()
        got = sh.run(Kbuf, Q, W, gather=True)
        ok[m + "_prefill"] = bool(torch.equal(got, ref))
        # the same key buffer rewritten in place (next layer) through the same sharded indexer
        Kbuf.copy_(torch.randn(L, d, device="cuda", generator=g).bfloat16())
        ref2 = IndexerEngine(m, **kw).run(Kbuf, Q, W).topk
        ok[m + "_prefill_rewritten_keys"] = bool(torch.equal(sh.run(Kbuf, Q, W, gather=True), ref2))
        del Kbuf
        Qd, Wd = Q[-8:].contiguous(), W[-8:].contiguous()
        refd = IndexerEngine(m, **kw).decode(K, Qd, Wd).topk
        gotd = ShardedIndexer(m, world=world, rank=rank, **kw).decode(K, Qd, Wd)
        ok[m + "_decode"] = bool(torch.equal(gotd, refd))
    # MISA-dagger at k' = 8192: pruned coarse lists (m = 4096, cap 6152 per rank), full-list
    # re-exchange of the early rows, merge of 2 x 8192 at the merge capacity
    kw = dict(budget_k=2048, active_heads_h=8, block_size=B, candidate_kprime=8192)
    ref = IndexerEngine("misa_hier", **kw).run(K, Q, W).topk
    sh = ShardedIndexer("misa_hier", world=world, rank=rank, **kw)
    ok["misa_hier_k8192_prefill"] = bool(torch.equal(sh.run(K, Q, W, gather=True), ref))
    ok["pruned"] = sh.exchange.last.get("cols", 8192) < 8192
    if world > 2:  # G * k' = 32768 > 16384: the global merge runs in rounds of list groups
        ok["misa_hier_k8192_decode"] = bool(torch.equal(sh.decode(K, Q[-8:].contiguous(), W[-8:].contiguous()),
                                                        IndexerEngine("misa_hier", **kw).decode(
                                                            K, Q[-8:].contiguous(), W[-8:].contiguous()).topk))
    q.put((rank, ok))
    dist.destroy_process_group()


if __name__ == "__main__":
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    [p.start() for p in ps]
    res = dict(q.get(timeout=900) for _ in range(world))
    [p.join() for p in ps]
    print(res)
    assert all(all(v.values()) for v in res.values()), res
    print("sharded smoke ok")
