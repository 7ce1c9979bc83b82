"""The N>1 product path on the GPU: two ranks (gloo, both on cuda:0 -- the only
GPU this build has) run bench.py's exact step through the C-ABI.

* replicated_store (north_star, BASELINE C3): rank 0 stores + seals, its packed
  rows Wb are broadcast, rank 1 ORs them into its cleared W8 and seals;
* sharded_store (u8 MAX all-reduce merge), sharded_store_bits
  (all-gather of packed partials + gb_or_bits, §8.f N3) and sharded_store_upper
  (all-gather of the upper-triangle blocks only + gb_or_upper, N3);
all four give both ranks W8 / Wb byte-identical to a single-rank store of all
messages.  Probe shards (weak: K per rank from the global stream; strong: a
fixed batch split) decoded on the ranks and gathered equal the single-rank
decode of the whole batch (Eq.(11) column independence) and
the oracle.  seal_status_all agrees over the ranks (a rank whose shard held an
invalid message makes every rank raise, none hangs)."""
import os
import socket

import numpy as np
import pytest

import gbgen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

C, L, M, K = 8, 128, 6000, 2500


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        import paper_1303_7032_b200 as gb
        from paper_1303_7032_b200 import dist as gdist
        torch.cuda.set_device(0)
        msgs = gbgen.messages(71, M, C, L)
        to_dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda()
        net = gb.Net(C, L, device=0)
        res = {}

        def snap(tag):
            torch.cuda.synchronize()
            res[tag + "_w8"] = net.weights().cpu().numpy()
            net.seal()
            res[tag + "_wb"] = net.bits().cpu().numpy()

        gdist.replicated_store(net, to_dev(msgs) if rank == 0 else None)
        gdist.seal_status_all(net)
        snap("bcast")
        gdist.sharded_store(net, to_dev(gdist.message_shard(msgs, rank, ws)))
        gdist.seal_status_all(net)
        snap("max")
        gdist.sharded_store_bits(net, to_dev(gdist.message_shard(msgs, rank, ws)))
        gdist.seal_status_all(net)
        snap("bits")
        gdist.sharded_store_upper(net, to_dev(gdist.message_shard(msgs, rank, ws)))
        gdist.seal_status_all(net)
        snap("upper")
        # weak shards of the global probe stream, decoded on the broadcast W (the bench's step)
        gdist.replicated_store(net, to_dev(msgs) if rank == 0 else None)
        lo, hi = gdist.weak_bounds(K, rank)
        pr, _ = gbgen.probes(72, msgs, K, 4, L, start=lo, random_count=K // 10)
        st, it, ss = net.decode(to_dev(pr), gb.HYBRID, gamma=2, max_iters=20)
        # strong shards of a fixed batch, all three rules
        allpr, _ = gbgen.probes(73, msgs, 3001, 4, L, random_count=300)
        a, b = gdist.strong_bounds(3001, rank, ws)
        strong = [net.decode(to_dev(allpr[a:b]), r, gamma=2, max_iters=20) for r in (0, 1, 2)]
        torch.cuda.synchronize()
        res["weak"] = np.concatenate([st.cpu().numpy().view(np.uint32), it.cpu().numpy()[:, None].view(np.uint16)
                                      .astype(np.uint32), ss.cpu().numpy()[:, None].astype(np.uint32)], axis=1)
        for r, (s2, i2, t2) in zip((0, 1, 2), strong):
            res[f"strong{r}"] = np.concatenate([s2.cpu().numpy().view(np.uint32),
                                                i2.cpu().numpy()[:, None].view(np.uint16).astype(np.uint32),
                                                t2.cpu().numpy()[:, None].astype(np.uint32)], axis=1)
        # a rank whose shard holds an invalid message: every rank raises in seal_status_all
        shard = gdist.message_shard(msgs, rank, ws)[:100].copy()
        if rank == 1:
            shard[0, 0] = L
        gdist.sharded_store_bits(net, to_dev(shard))
        raised = False
        try:
            gdist.seal_status_all(net)
        except gb.GBError:
            raised = True
        res["raised"] = np.array([raised])
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
        net.close()
    finally:
        dist.destroy_process_group()


def test_two_ranks_bench_step_on_gpu(tmp_path):
    import torch.multiprocessing as mp
    import paper_1303_7032_b200 as gb
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    ws = 2
    mp.spawn(_worker, args=(ws, _free_port(), str(tmp_path)), nprocs=ws, join=True)
    got = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(ws)]
    msgs = gbgen.messages(71, M, C, L)
    net = gb.Net(C, L)
    net.store(torch.from_numpy(msgs.view(np.int16)).cuda())
    net.seal()
    w8 = net.weights().cpu().numpy()
    net.seal()
    wb = net.bits().cpu().numpy()
    w, _ = oracle.store(msgs, C, L)
    assert np.array_equal(w8, w)
    for r in range(ws):
        for tag in ("bcast", "max", "bits", "upper"):
            assert np.array_equal(got[r][tag + "_w8"], w8), (r, tag)
            assert np.array_equal(got[r][tag + "_wb"], wb), (r, tag)
        assert got[r]["raised"][0]
    # weak: concatenated rank shards == the global stream [0, 2K) decoded at once (and the oracle)
    pr0 = np.concatenate([gbgen.probes(72, msgs, K, 4, L, start=r * K, random_count=K // 10)[0] for r in range(ws)])
    st, it, ss = net.decode(torch.from_numpy(pr0.view(np.int16)).cuda(), gb.HYBRID, gamma=2, max_iters=20)
    torch.cuda.synchronize()
    whole = np.concatenate([st.cpu().numpy().view(np.uint32), it.cpu().numpy()[:, None].view(np.uint16)
                            .astype(np.uint32), ss.cpu().numpy()[:, None].astype(np.uint32)], axis=1)
    assert np.array_equal(np.concatenate([g["weak"] for g in got]), whole)
    ost, oit, oss = oracle.decode(w, C, L, pr0, oracle.HYBRID, gamma=2, max_iters=20)
    assert np.array_equal(whole[:, :-2], ost) and np.array_equal(whole[:, -2], oit) and np.array_equal(whole[:, -1], oss)
    allpr, _ = gbgen.probes(73, msgs, 3001, 4, L, random_count=300)
    for r in (0, 1, 2):
        ost, oit, oss = oracle.decode(w, C, L, allpr, r, gamma=2, max_iters=20)
        cat = np.concatenate([g[f"strong{r}"] for g in got])
        assert np.array_equal(cat[:, :-2], ost) and np.array_equal(cat[:, -2], oit) and np.array_equal(cat[:, -1], oss), r
    net.close()
