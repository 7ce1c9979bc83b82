"""Multi-process (world_size 2, gloo, CPU) checks of the N>1 plumbing.

The GPU store/decode are replaced by the CPU oracle (test-only), so what is
tested is the sharding and merge logic of paper_1303_7032_b200.dist:
  * the MAX all-reduce of per-rank partial W (uint8) equals the single-store
    W byte for byte (Eq.(1) OR semantics), and so does the OR of
    the all-gathered packed partials (gather_bits);
  * decoding per-rank probe shards and gathering equals decoding the whole
    batch (Eq.(11) column independence), for the weak
    (per-rank K) and strong (split K) shardings;
  * max/sum over ranks; MAX on packed bit words is rejected.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gbgen
import oracle
from paper_1303_7032_b200 import dist as gdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        c, l, m = 8, 32, 400
        msgs = gbgen.messages(7, m, c, l)
        part, _ = oracle.store(np.ascontiguousarray(gdist.message_shard(msgs, rank, ws)), c, l)
        w8 = torch.from_numpy(part.copy())
        gdist.merge_weights_(w8)
        full, _ = oracle.store(msgs, c, l)
        assert np.array_equal(w8.numpy(), full), "MAX merge != single store"
        with pytest.raises(TypeError):
            gdist.merge_weights_(torch.zeros(4, dtype=torch.int32))
        # N3 packed merge: all-gather of the packed partials, OR == single store
        packed = np.packbits(part, axis=1, bitorder="little").view(np.int32)   # Wb layout (n = 256)
        allb = gdist.gather_bits(torch.from_numpy(packed.copy()))
        assert tuple(allb.shape) == (ws,) + packed.shape
        ored = np.bitwise_or.reduce(allb.numpy().view(np.uint32), axis=0)
        unpacked = np.unpackbits(ored.view(np.uint8), axis=1, bitorder="little")
        assert np.array_equal(unpacked, full), "OR of gathered packed partials != single store"
        # weak sharding: each rank decodes k probes of the global stream
        k = 64
        lo, hi = gdist.weak_bounds(k, rank)
        pr, _ = gbgen.probes(8, msgs, k, 3, l, start=lo)
        st, it, ss = oracle.decode(w8.numpy(), c, l, pr, oracle.HYBRID, gamma=1)
        gath = [torch.zeros((k, st.shape[1]), dtype=torch.int64) for _ in range(ws)]
        dist.all_gather(gath, torch.from_numpy(st.astype(np.int64)))
        # strong sharding of a fixed batch
        K = 101
        allpr, _ = gbgen.probes(9, msgs, K, 3, l)
        a, b = gdist.strong_bounds(K, rank, ws)
        st2, it2, _ = oracle.decode(w8.numpy(), c, l, allpr[a:b], oracle.SOM, gamma=1)
        sizes = [gdist.strong_bounds(K, r, ws) for r in range(ws)]
        buf = torch.zeros((max(h - g for g, h in sizes), st2.shape[1] + 1), dtype=torch.int64)
        buf[:b - a, :-1] = torch.from_numpy(st2.astype(np.int64))
        buf[:b - a, -1] = torch.from_numpy(it2.astype(np.int64))
        gath2 = [torch.zeros_like(buf) for _ in range(ws)]
        dist.all_gather(gath2, buf)
        tmax = gdist.max_over_ranks([float(rank), 10.0 - rank])
        tsum = gdist.sum_over_ranks([1, rank])
        if rank == 0:
            np.save(os.path.join(out_dir, "weak.npy"), torch.cat(gath).numpy())
            np.save(os.path.join(out_dir, "strong.npy"),
                    torch.cat([g[:h - lo_] for g, (lo_, h) in zip(gath2, sizes)]).numpy())
            np.save(os.path.join(out_dir, "red.npy"), np.array(tmax + [float(x) for x in tsum]))
    finally:
        dist.destroy_process_group()


def test_two_rank_store_merge_and_shard_invariance(tmp_path):
    ws = 2
    mp.spawn(_worker, args=(ws, _free_port(), str(tmp_path)), nprocs=ws, join=True)
    c, l, m = 8, 32, 400
    msgs = gbgen.messages(7, m, c, l)
    full, _ = oracle.store(msgs, c, l)
    # weak: the concatenation of the rank shards is the global stream [0, 2k)
    pr, _ = gbgen.probes(8, msgs, 128, 3, l)
    st, _, _ = oracle.decode(full, c, l, pr, oracle.HYBRID, gamma=1)
    np.testing.assert_array_equal(np.load(tmp_path / "weak.npy"), st.astype(np.int64))
    allpr, _ = gbgen.probes(9, msgs, 101, 3, l)
    st2, it2, _ = oracle.decode(full, c, l, allpr, oracle.SOM, gamma=1)
    got = np.load(tmp_path / "strong.npy")
    np.testing.assert_array_equal(got[:, :-1], st2.astype(np.int64))
    np.testing.assert_array_equal(got[:, -1], it2.astype(np.int64))
    np.testing.assert_array_equal(np.load(tmp_path / "red.npy"), [1.0, 10.0, 2.0, 1.0])


def test_max_on_packed_bits_is_not_or():
    """Why the merge is on u8: MAX of packed words loses bits."""
    a, b = np.uint32(0b01), np.uint32(0b10)
    assert max(a, b) != (a | b)
    assert max(np.uint8(1), np.uint8(0)) == (np.uint8(1) | np.uint8(0))
